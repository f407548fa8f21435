#!/bin/bash
# tensor-core round kernel: parity, phase probe for both variants, short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_parity.log 2>&1; echo "parity rc $?"
tail -15 gpurun_out/pytest_parity.log
timeout 300 python -m paper_1712_05878_b200.diag > gpurun_out/diag_simt.json 2>&1; echo "diag simt rc $?"
GHC_STEP=tc timeout 300 python -m paper_1712_05878_b200.diag > gpurun_out/diag_tc.json 2>&1; echo "diag tc rc $?"
timeout 600 python bench.py --no-cpu --steps 20000 > gpurun_out/bench.log 2>&1; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print({k: d[k] for k in ['value','ms_per_step','clocks','gpu_launches']}, 'e2e', d['e2e']['value'], d['config'], d['roofline'].get('kernel'))"
