python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2.py tests/test_gpu_resident.py tests/test_gpu_e2e*.py -x -q -m gpu 2>&1 | tail -2
python tools/e2e_anatomy.py > gpurun_out/e2e_anatomy2.json 2>&1; cat gpurun_out/e2e_anatomy2.json | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v['us_per_round'],3) for k,v in d.items()})"
python tools/launch_anatomy.py > gpurun_out/launch_anatomy2.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/launch_anatomy2.json')); print({k: d[k]['entry_to_round0_us'] for k in ('R1','R2','R20')}, d['gated_event_us'])"
