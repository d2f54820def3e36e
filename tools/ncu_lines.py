"""Per-source-line stall samples / instructions from `ncu --page source --csv
--print-source cuda,sass` output (stdin).  Usage: python tools/ncu_lines.py < mix.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
fname = None
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if r[0] == "Function Name" or hdr is None:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        agg[cur][2] = r[1][:90]
    try:
        s = float(r[4] or 0)
        ins = float(r[7] or 0)
    except (ValueError, IndexError):
        continue
    if cur:
        agg[cur][0] += s
        agg[cur][1] += ins
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot:.0f}, instructions {toti:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[1]) if len(sys.argv) > 1 else 40]:
    print(f"{k[0]:>22}:{k[1]:<4} {100 * v[0] / tot:5.1f}% samp {100 * v[1] / toti:5.1f}% inst  {v[2]}")
