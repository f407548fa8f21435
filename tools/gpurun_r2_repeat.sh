# repeatability of the driver-shaped bench: 5 separate processes
for i in 1 2 3 4 5; do
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/rep_$i.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/rep_$i.json').read().splitlines()[-1])
print(json.dumps({'run': $i, 'value': d['value'], 'us_per_round': d['ms_per_step']*1e3, 'e2e': d['e2e']['value'], 'e2e_us_per_round': d['e2e']['ms_per_step']*1e3, 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))"
done
