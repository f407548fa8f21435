export GHC_NO_COOP=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/ncu_l.log 2>&1; echo "launch list rc $?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/r02_launches.csv')))
hdr = [i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0,0.0])
for r in rows[hdr+1:]:
    try: v = float(r[vi].replace(',',''))
    except: continue
    agg[r[ki][:60]][0] += 1; agg[r[ki][:60]][1] += v
tot = sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:12]: print(f"{v[1]/tot*100:5.1f}% {v[0]:4d} {v[1]/1e3:9.1f}us {k}")
PY
