# staggered second poll in exchange steps (c) / (d): GHC_POLL_STAGGER = 0
# (default build), 300, 600 SM cycles — bit-identity, parity, per-phase probe
for L in "" _ab/libghc_ps300.so _ab/libghc_ps600.so; do
  echo "== ${L:-default}"
  GHC_LIB_PATH=$L python tools/ab_bits.py
  GHC_LIB_PATH=$L timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
done
for i in 1 2; do for L in "" _ab/libghc_ps300.so _ab/libghc_ps600.so; do
  GHC_LIB_PATH=$L python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag_ps.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/diag_ps.json')); print('${L:-default}', 'us/round %.2f' % d['us_per_round'], {k: v['median'] for k, v in d['phases_ns'].items() if not k.startswith('sample0')})"
done; done
