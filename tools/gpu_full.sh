#!/bin/bash
# full GPU check: gpu tests, smoke, bench (plain), phase probe
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 300 python -m paper_1712_05878_b200.diag > gpurun_out/diag.json 2>&1; echo "diag rc $?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print({k: d[k] for k in ['value','ms_per_step','clocks','gpu_launches']}, 'e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'], 'upd', d['update_kernel']['frac'])"
