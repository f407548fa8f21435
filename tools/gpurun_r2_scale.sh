# gradient scale hoisted out of the round loop (fixed n): bit identity vs the
# previous build, parity, per-phase probe and driver-shaped bench A/B
python tools/ab_bits.py; GHC_LIB_PATH=_ab/libghc_head.so python tools/ab_bits.py
python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2.py tests/test_gpu_resident.py -x -q -m gpu 2>&1 | tail -1
for i in 1 2 3; do
for L in "" _ab/libghc_head.so; do
GHC_LIB_PATH=$L python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag_sc.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/diag_sc.json')); print('${L:-new}', 'us/round %.3f' % d['us_per_round'], 'gap', d['phases_ns']['next_round_gap']['median'], 'xwait', d['phases_ns']['sample0_x_wait']['median'])"
done; done
