# prologue (both master buffers loaded with the flag) + relaxed final cluster
# barrier: fixed cost per launch and driver-shaped bench vs the previous build
python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2.py tests/test_gpu_resident.py tests/test_gpu_roles.py -x -q -m gpu 2>&1 | tail -2
python tools/ab_bits.py; GHC_LIB_PATH=_ab/libghc_head.so python tools/ab_bits.py
for i in 1 2; do
python tools/launch_anatomy.py > gpurun_out/la_new.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/la_new.json')); print('new ', {k: (d[k]['entry_to_round0_us'], d[k]['last_commit_to_exit_us']) for k in ('R1','R2','R20')}, {k: round(v,1) for k,v in d['gated_event_us'].items()})"
GHC_LIB_PATH=_ab/libghc_head.so python tools/launch_anatomy.py > gpurun_out/la_head.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/la_head.json')); print('head', {k: (d[k]['entry_to_round0_us'], d[k]['last_commit_to_exit_us']) for k in ('R1','R2','R20')}, {k: round(v,1) for k,v in d['gated_event_us'].items()})"
done
