python tools/update_bench.py > gpurun_out/upd.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/upd.jsonl'):
    d=json.loads(l); print(d['kernel'], d['api'][:30], round(d['ms']*1e3,1),'us', round(d['frac'],3))"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv -k regex:"sgd|easgd|elastic|weighted|fixup" python tools/update_bench.py --once > gpurun_out/ncu_upd.csv 2> gpurun_out/ncu_upd.err; tail -40 gpurun_out/ncu_upd.csv | cut -c1-200
