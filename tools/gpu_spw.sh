#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m paper_1712_05878_b200.diag > gpurun_out/diag_spw2.json 2>&1; echo "diag2 rc $?"
cp paper_1712_05878_b200/_build/alt/libghc.so paper_1712_05878_b200/_build/libghc.so
GHC_SPW_DIAG=1 timeout 300 python -m paper_1712_05878_b200.diag > gpurun_out/diag_spw1.json 2>&1; echo "diag1 rc $?"
python - <<'PY'
import json
for f in ['gpurun_out/diag_spw2.json','gpurun_out/diag_spw1.json']:
    d=json.load(open(f)); print(f, d['us_per_round'], d['warps'], {k: v['median'] for k,v in d['phases_ns'].items()})
PY
