# A/B of the single-GPU exchange: reduce-scatter (two L2 hops, clusters of 4)
# vs one hop over clusters of 8 / 16 (GHC_CS, GHC_XCHG=onehop)
for cfg in "" "GHC_CS=8" "GHC_CS=8 GHC_XCHG=onehop" "GHC_CS=16 GHC_XCHG=onehop"; do
  echo "== $cfg"
  env $cfg timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2.py -x -q -m gpu 2>&1 | tail -2
  env $cfg timeout 120 python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag_hop.json 2>&1
  python - <<'PY'
import json
d = json.load(open('gpurun_out/diag_hop.json'))
print(d['kernel'], d['ctas'], d['warps'], 'us/round %.2f' % d['us_per_round'],
      {k: v['median'] for k, v in d['phases_ns'].items()})
PY
done
