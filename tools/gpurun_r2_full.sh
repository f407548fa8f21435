# full validation: GPU suite, smoke, driver-shaped bench, resident anatomy
python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench20.json 2>gpurun_out/bench20.err; tail -2 gpurun_out/bench20.err
python -c "
import json;d=json.loads(open('gpurun_out/bench20.json').read().splitlines()[-1]);print(d['value'], d['ms_per_step']*1e3, d['timing']['resident']['ms_per_step']*1e3, d['e2e']['value'], d['e2e']['ms_per_step']*1e3, d['roofline']['latency']['frac'], d['clocks']['sm_mhz'])"
python tools/resident_anatomy.py > gpurun_out/resident_anatomy.json 2>&1; tail -3 gpurun_out/resident_anatomy.json
