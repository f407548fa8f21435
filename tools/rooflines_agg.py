"""Aggregate ncu launch lists (--metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,
launch__registers_per_thread; --csv) into one markdown table per path:
launches, mean µs per launch, DRAM bytes per launch, DRAM GB/s and its
fraction of the measured HBM copy peak (MEASURED_PEAKS.json), tensor-pipe
activity.  ncu serialises launches and flushes caches between them: the
DRAM figures are cold-cache, the fractions say how close a launch runs to
the HBM roof, not its share of a warm step.

    python tools/rooflines_agg.py path=file.csv [path=file.csv ...]"""
import collections
import csv
import json
import re
import sys

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
print(f"| path | kernel | launches | µs / launch | DRAM MB / launch | DRAM GB/s | % of measured HBM ({peak:.0f} GB/s) | tensor pipe active % | regs |")
print("|---|---|---|---|---|---|---|---|---|")
for arg in sys.argv[1:]:
    path, fn = arg.split("=", 1)
    lines = [l for l in open(fn) if l.startswith('"')]
    if not lines:
        print(f"| {path} | (no launches captured) | | | | | | | |")
        continue
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        try:
            per[(r[ii], re.sub(r"\(.*", "", r[ki])[:60])][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for (_, k), mm in per.items():
        a = agg[k]
        a["n"] += 1
        a["t"] += mm.get("gpu__time_duration.sum", 0.0)
        a["b"] += mm.get("dram__bytes_read.sum", 0.0) + mm.get("dram__bytes_write.sum", 0.0)
        a["tp"] += mm.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
        a["regs"] = max(a["regs"], mm.get("launch__registers_per_thread", 0.0))
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        n, t_ns, b = a["n"], a["t"], a["b"]
        gbs = b / t_ns if t_ns else 0.0  # bytes per ns = GB/s
        print(f"| {path} | `{k.strip()}` | {int(n)} | {t_ns / n / 1e3:.1f} | {b / n / 1e6:.2f} | {gbs:.0f} | "
              f"{100 * gbs / peak:.0f} | {a['tp'] / n:.1f} | {int(a['regs'])} |")
