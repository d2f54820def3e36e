"""Summarise an ncu --set full capture of ONE scheduled query batch
(tools/ncu_sched.py under `ncu --profile-from-start off`): per-kernel table +
the per-batch DRAM traffic JSON bench.py reads as roofline.traffic.
Usage: python tools/ncu_sched_summary.py REPORT.ncu-rep OUT_PREFIX [note]
writes OUT_PREFIX.txt and profiles/query_kernel_ncu_sift1m.json"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, out = sys.argv[1], Path(sys.argv[2])
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
units = rows[1]
M = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "lts__t_sector_hit_rate.pct", "launch__registers_per_thread"]
ix = {m: h.index(m) for m in M}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def val(r, m):
    v = float(r[ix[m]].replace(",", ""))
    return v * scale.get(units[ix[m]], 1)


lines = [f"ncu --set full --clock-control none of one scheduled 10k-query batch ({note})",
         f"{'kernel':44s} {'us':>9s} {'DRAM MB':>9s} {'warp inst':>12s} {'issue%':>7s} {'warps%':>7s} {'L2hit%':>7s} regs"]
tot = {"t": 0.0, "b": 0.0, "i": 0.0}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    t = val(r, "gpu__time_duration.sum")
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    i = val(r, "smsp__inst_executed.sum")
    tot["t"] += t
    tot["b"] += b
    tot["i"] += i
    lines.append(f"{name[:44]:44s} {t:9.1f} {b / 1e6:9.1f} {i:12.0f} "
                 f"{val(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):7.1f} "
                 f"{val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):7.1f} "
                 f"{val(r, 'lts__t_sector_hit_rate.pct'):7.1f} {int(val(r, 'launch__registers_per_thread'))}")
lines.append(f"{'batch total':44s} {tot['t']:9.1f} {tot['b'] / 1e6:9.1f} {tot['i']:12.0f}")
out.with_suffix(".txt").write_text("\n".join(lines) + "\n")
print("\n".join(lines))
js = {"kernel": "one scheduled query batch: query_kernel<u8,u8,8> pilot + park_order + resume_kernel rounds "
                f"(sift1m: C2 latent16 1M x 128 u8, 10k queries of a fresh batch; {note})",
      "dram_bytes_per_launch": tot["b"], "duration_ms_under_ncu": tot["t"] / 1e3, "warp_instructions": tot["i"],
      "source": f"ncu --set full --clock-control none --profile-from-start off python tools/ncu_sched.py; "
                f"{out.with_suffix('.txt').name}"}
Path("profiles/query_kernel_ncu_sift1m.json").write_text(json.dumps(js, indent=1) + "\n")
