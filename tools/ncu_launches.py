"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count and total device time.  Usage:
python tools/ncu_launches.py gpurun_out/launches.csv [--last N]"""
import csv
import sys
from collections import defaultdict

MULT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = {k: j for j, k in enumerate(rows[start])}
    out = []
    for r in rows[start + 1:]:
        if len(r) < len(h) or r[h["Metric Name"]] != "gpu__time_duration.sum":
            continue
        us = float(r[h["Metric Value"]].replace(",", "")) * MULT[r[h["Metric Unit"]]]
        out.append((r[h["Kernel Name"]].split("(")[0], us))
    return out


if __name__ == "__main__":
    launches = load(sys.argv[1])
    if "--last" in sys.argv:
        launches = launches[-int(sys.argv[sys.argv.index("--last") + 1]):]
    agg = defaultdict(lambda: [0, 0.0])
    for name, us in launches:
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{len(launches)} launches, {tot / 1e3:.2f} ms device time")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{k[:72]:72s} {v[0]:6d} {v[1] / 1e3:10.3f} ms {100 * v[1] / tot:5.1f}%")
