# A/B of a kernel change: parity of the fused kernels, per-phase probe, driver-shaped bench
python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2.py -x -q -m gpu 2>&1 | tail -3
python -m paper_1712_05878_b200.diag --rounds 400 > gpurun_out/diag.json 2>&1; cat gpurun_out/diag.json | head -40
python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench20.json 2>gpurun_out/bench20.err
python -c "
import json;d=json.loads(open('gpurun_out/bench20.json').read().splitlines()[-1]);print('value',d['value'],'us/round',d['ms_per_step']*1e3,'steady',d['timing'].get('steady_us_per_round'),'e2e',d['e2e']['value'])"
