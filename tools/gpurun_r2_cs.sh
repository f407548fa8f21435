for cs in 4 2; do
  GHC_CS=$cs python -c "
import sys; sys.path.insert(0,'.')
import paper_1712_05878_b200 as g
ctx=g.Context(0); a=g.Architecture(ctx,'lstm(5,20,10),softmax(20,3)'); print('$cs', a.kernel_name, ctx.lib.ghc_plan_max_clusters(a.h))"
  GHC_CS=$cs python tools/fixed_cost.py > gpurun_out/fc_$cs.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/fc_$cs.json'));print('cs $cs', d['fit_round_us'], d['fit_fixed_us'], d['call_us_by_rounds']['20']/20)"
  GHC_CS=$cs python -m paper_1712_05878_b200.diag --rounds 200 > gpurun_out/ph_$cs.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ph_$cs.json')); print(d['us_per_round'], d['ctas'], d['warps'], {k:v['median'] for k,v in d['phases_ns'].items()})"
done
