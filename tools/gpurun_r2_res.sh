timeout 300 python -m pytest tests/test_gpu_resident.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench20.json 2>gpurun_out/bench20.err; tail -2 gpurun_out/bench20.err
python -c "
import json;d=json.loads(open('gpurun_out/bench20.json').read().splitlines()[-1])
e=d['e2e']; print('value', d['value'], 'us/round', d['ms_per_step']*1e3); print({k:(round(v['ms_per_step']*1e3,2) if isinstance(v,dict) and 'ms_per_step' in v else v) for k,v in e.items() if k not in ('path',)})
print(e.get('per_call_cxx'))"
