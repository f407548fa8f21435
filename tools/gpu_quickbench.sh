#!/bin/bash
# Quick A/B on the GPU box: the sync-round parity subset + a short bench.
# usage: tools/gpu_quickbench.sh TAG
T=${1:-q}
python -m pytest tests -m gpu -x -q -k "simt and (master or worker_grad)" > gpurun_out/t_$T.log 2>&1; tail -1 gpurun_out/t_$T.log
for i in 1 2; do
python bench.py --steps 30000 --warmup 50 --e2e-steps 500 --no-cpu > gpurun_out/b_$T.json 2>gpurun_out/b_$T.err
python -c "import json;d=json.loads(open('gpurun_out/b_$T.json').read().splitlines()[-1]);print('value',d['value'],'us',d['ms_per_step']*1e3,'e2e',d['e2e']['value'],d['clocks'])"
done
python -m paper_1712_05878_b200.diag > gpurun_out/p_$T.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/p_$T.json'));print(d['us_per_round'],{k:v['median'] for k,v in d['phases_ns'].items()})"
