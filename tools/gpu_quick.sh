#!/bin/bash
# quick GPU iteration: parity tests + phase probe + short bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -m paper_1712_05878_b200.diag > gpurun_out/diag.json 2>&1; echo "diag rc $?"
cat gpurun_out/diag.json
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print({k: d[k] for k in ['value','ms_per_step','e2e','clocks','gpu_launches']}, d['roofline']['frac'], d['update_kernel']['frac'])"
