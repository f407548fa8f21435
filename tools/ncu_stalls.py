"""Aggregate ncu source-page (SASS) warp-stall samples into address ranges.

usage: ncu -i rep --page source --csv --print-source sass > src.csv
       python tools/ncu_stalls.py src.csv [--top 40] [--ranges a0-a1,...]
Prints the hottest instructions with their dominant stall reasons, and the
sample totals per range (phase) when --ranges is given (hex SASS addresses).
"""
import argparse
import csv
import collections

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--ranges", default="")
args = ap.parse_args()
rows = list(csv.reader(open(args.csv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        addr = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    tot = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    rs = {k: int(r[ix[k]] or 0) for k in reasons}
    data.append((addr, r[ix["Source"]], tot, rs))
total = sum(d[2] for d in data)
print("total samples", total)
agg = collections.Counter()
for d in data:
    agg.update(d[3])
print("by reason:", ", ".join(f"{k[6:]}={v}" for k, v in agg.most_common(10)))
for d in sorted(data, key=lambda d: -d[2])[: args.top]:
    top = sorted(d[3].items(), key=lambda kv: -kv[1])[:3]
    print(f"{d[0]:#06x} {d[2]:6d} {d[1][:60]:60s} " + " ".join(f"{k[6:]}={v}" for k, v in top if v))
if args.ranges:
    for rg in args.ranges.split(","):
        name, span = rg.split("=") if "=" in rg else (rg, rg)
        a0, a1 = (int(x, 16) for x in span.split("-"))
        sel = [d for d in data if a0 <= d[0] < a1]
        c = collections.Counter()
        for d in sel:
            c.update(d[3])
        s = sum(d[2] for d in sel)
        print(f"{name:12s} {s:7d} ({100.0 * s / max(total, 1):5.1f}%) "
              + " ".join(f"{k[6:]}={v}" for k, v in c.most_common(4)))
