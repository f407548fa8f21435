"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export per
source line: warp-stall samples (all) and the top stall reasons.  SASS rows
(empty 'Line No') are attributed to the preceding source line.
usage: python tools/ncu_src_agg.py export.csv [top_n] [file_filter]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
flt = sys.argv[3] if len(sys.argv) > 3 else ""
hdr = next(r for r in rows if r and r[0] == "Line No")
stall_cols = [(i, c) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
n_hdr = len(hdr)
cur_file, cur_line = None, None
tot = collections.Counter()
why = collections.defaultdict(collections.Counter)
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0].strip():
        cur_line = (cur_file, int(r[0]))
        text[cur_line] = ",".join(r[1:len(r) - n_hdr + 2]).strip()[:80]
        continue
    if len(r) != n_hdr:
        continue
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    tot[cur_line] += s
    for i, c in stall_cols:
        why[cur_line][c[6:]] += int(r[i] or 0)
T = sum(tot.values())
print("total samples", T)
for ln, s in tot.most_common():
    if flt and flt not in ln[0]:
        continue
    top_n -= 1
    if top_n < 0:
        break
    w = why[ln]
    ws = sum(w.values()) or 1
    tops = " ".join(f"{k}:{v * 100 // ws}" for k, v in w.most_common(3))
    print(f"{s * 100 / T:5.1f}% {ln[0]}:{ln[1]:<4} [{tops}]  {text.get(ln, '')}")
