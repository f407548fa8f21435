# update kernels: parity (in-place vs one-pass, oracle), adapter drop-in, roles; HBM roofline
python -m pytest tests/test_gpu_parity.py tests/test_gpu_adapter.py tests/test_gpu_roles.py -x -q -m gpu -k "sgd or easgd or adapter or roles" 2>&1 | tail -3
python tools/update_bench.py > gpurun_out/update_bench.jsonl 2>gpurun_out/update_bench.err; cat gpurun_out/update_bench.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['kernel']:26s} {d['api'][:48]:48s} {d['ms']*1e3:7.1f} us {d['frac']*100:5.1f} %\")"
python tools/update_bench.py --once > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"sgd_out|easgd_worker_out" --csv python tools/update_bench.py --once > gpurun_out/ncu_upd2.csv 2>gpurun_out/ncu_upd2.err; grep -v "^==" gpurun_out/ncu_upd2.csv | tail -8
