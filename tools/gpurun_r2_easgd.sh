# sync EASGD with one gradient launch per round: role parity vs the oracle,
# session bench (c3 et al.)
timeout 900 python -m pytest tests/test_gpu_roles.py tests/test_gpu_wide.py tests/test_gpu_parity.py -q -x -m gpu -k "easgd or EASGD or roles or wide or worker_grads or replay or async" 2>&1 | tail -2
python tools/session_bench.py > gpurun_out/session_bench.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/session_bench.json')); print({k: (round(v.get('samples_per_s', 0)/1e6, 2), round(v.get('us_per_update', 0), 1)) for k, v in d.items() if isinstance(v, dict)})"
