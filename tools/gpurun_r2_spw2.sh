# Two samples interleaved per warp (GHC_SPW=2 build, _ab/libghc_spw2.so):
# 4 warps x 2 samples per CTA instead of 8 x 1 — per-phase probe and parity
for i in 1 2; do
GHC_LIB_PATH=_ab/libghc_spw2.so GHC_SPW_DIAG=2 python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag_spw2.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/diag_spw2.json')); print('spw2 us/round %.2f' % d['us_per_round'], d['ctas'], d['warps'], {k: v['median'] for k, v in d['phases_ns'].items()})"
python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag_spw1.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/diag_spw1.json')); print('spw1 us/round %.2f' % d['us_per_round'], d['ctas'], d['warps'], {k: v['median'] for k, v in d['phases_ns'].items()})"
done
GHC_LIB_PATH=_ab/libghc_spw2.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
