# FFMA2 gate pairs in the weight-gradient pass: bit-identity vs the previous
# build (_ab/libghc_head.so), parity tests, per-phase probe, bench
python tools/ab_bits.py; GHC_LIB_PATH=_ab/libghc_head.so python tools/ab_bits.py
python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag_dw2.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/diag_dw2.json')); print('new us/round %.2f' % d['us_per_round'], {k: v['median'] for k, v in d['phases_ns'].items() if k.startswith('sample')})"
GHC_LIB_PATH=_ab/libghc_head.so python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag_head.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/diag_head.json')); print('head us/round %.2f' % d['us_per_round'], {k: v['median'] for k, v in d['phases_ns'].items() if k.startswith('sample')})"
done
