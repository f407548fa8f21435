# bench (driver shape), then the headline kernel's launch list + one ncu --set full capture
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench20.json 2>gpurun_out/bench20.err; tail -2 gpurun_out/bench20.err
python -c "
import json;d=json.loads(open('gpurun_out/bench20.json').read().splitlines()[-1]);print(d['value'], d['ms_per_step']*1e3, d['timing']['resident']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['roofline']['latency']['frac'])"
export GHC_NO_COOP=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --e2e-steps 20 > gpurun_out/ncu_l.log 2>&1; echo "launch list rc $?"
ncu --set full --clock-control none --import-source on -k regex:lstm_round_kernel -s 2 -c 1 -o gpurun_out/r02_round python bench.py --gpus 1 --steps 200 --warmup 5 --no-cpu --e2e-steps 20 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
ncu -i gpurun_out/r02_round.ncu-rep --page raw --csv > gpurun_out/r02_round_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/r02_round_raw.csv')))
h = rows[0]
want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__grid_size','launch__registers_per_thread','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__inst_executed.sum']
for r in rows[2:3]:
    for w in want:
        if w in h: print(w, r[h.index(w)], rows[1][h.index(w)])
PY
