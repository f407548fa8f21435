# wide variant launch list with warm caches (ncu --cache-control none): per-kernel time and DRAM bytes
ROUNDS=3 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv python tools/wide_bench.py > gpurun_out/wide_launches_warm.csv 2>gpurun_out/wide_ncu_warm.err
python - <<'PY'
import csv, collections, re
lines = [l for l in open('gpurun_out/wide_launches_warm.csv') if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]; ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value'); ii = h.index('ID')
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[(r[ii], re.sub(r'\(.*', '', r[ki])[:48])][r[mi]] = float(r[vi].replace(',', ''))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, k), m in per.items():
    a = agg[k]; a[0] += 1; a[1] += m.get('gpu__time_duration.sum', 0); a[2] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e3/3:.1f} us per round (3 rounds, ncu serialised)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]/tot*100:5.1f}% {v[0]:4d} {v[1]/1e3/3:8.1f} us/round  DRAM {v[2]/max(v[1],1):7.1f} GB/s ({v[2]/max(v[1],1)/6547.5*100:4.0f}% of 6.55 TB/s)  {k}")
PY
