"""Aggregate `ncu --page source --csv --print-source cuda,sass` instruction
counts / stall samples per enclosing source function (heuristic: nearest
preceding function-looking line).  Usage: ncu_funcs.py src.csv [csrc_dir]"""
import csv
import re
import sys
from collections import defaultdict
from pathlib import Path

src_dir = Path(sys.argv[2] if len(sys.argv) > 2 else Path(__file__).resolve().parents[1] / "paper_1912_01059_b200/csrc")
FUN = re.compile(r"^\s*(template\s*<.*>\s*)?(__device__|__global__|__host__).*?(\w+)\s*\(")
funcs = {}
for p in src_dir.glob("*.cu*"):
    starts = []
    for i, line in enumerate(p.read_text().splitlines(), 1):
        m = FUN.match(line)
        if m:
            starts.append((i, m.group(3)))
    funcs[p.name] = starts


def owner(fname, ln):
    best = "?"
    for i, n in funcs.get(fname, []):
        if i <= ln:
            best = n
    return f"{fname}:{best}"


rows = list(csv.reader(open(sys.argv[1])))
fname, hdr = None, None
agg = defaultdict(lambda: [0.0, 0.0])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        agg[owner(fname, int(r[0]))][0] += float(r[6] or 0)
        agg[owner(fname, int(r[0]))][1] += float(r[7] or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"instructions {ti:.3e}  samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{k:55s} {100 * v[1] / ti:5.1f}% inst {100 * v[0] / ts:5.1f}% samp")
