#!/bin/bash
# full GPU tests + bench (no CPU baseline) with the streaming e2e
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --steps 20000 --e2e-steps 1000 > gpurun_out/bench.log 2>&1; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print({k: d[k] for k in ['value','ms_per_step','clocks','gpu_launches']}); print('e2e', json.dumps(d['e2e']))"
