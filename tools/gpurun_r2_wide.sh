python -m pytest tests/test_gpu_wide.py tests/test_gpu_generic.py tests/test_gpu_dense.py -q -x > gpurun_out/tw.log 2>&1; tail -3 gpurun_out/tw.log
python tools/wide_bench.py > gpurun_out/wide.json 2>&1; cat gpurun_out/wide.json
ROUNDS=5 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/wide_bench.py > gpurun_out/wide_launches.csv 2>gpurun_out/wide_ncu.err
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/wide_launches.csv')))
hdr = [i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0,0.0])
for r in rows[hdr+1:]:
    try: v = float(r[vi].replace(',',''))
    except: continue
    agg[r[ki][:50]][0] += 1; agg[r[ki][:50]][1] += v
tot = sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{v[1]/tot*100:5.1f}% {v[0]:4d} {v[1]/1e3:9.1f}us {k}")
PY
