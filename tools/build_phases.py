"""Per-phase build times at 1M (host perf_counter around each phase)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

base, _ = make_latent16(n=1_000_000, d=128, m=1, seed=1234)
ds = ga.Dataset(base)
ga.build(ga.Dataset(base[:50_000].copy()), ga.BuildConfig(seed=7))  # warm-up (module load, first launches)
h, st = ga.build(ds, ga.BuildConfig(seed=7))
ph = st.phase_seconds
print("total %.2f s, sum of phases %.2f s" % (st.build_seconds, sum(ph.values())))
groups = {}
for k, v in ph.items():
    kind = k.split("/")[-1].rstrip("0123456789.").replace("refine", "refine").replace("merge", "merge")
    kind = "sym" if k.endswith("/sym") else ("refine" if "refine" in k else ("merge" if "merge" in k else kind))
    groups[kind] = groups.get(kind, 0.0) + v
for k, v in sorted(groups.items(), key=lambda kv: -kv[1]):
    print(f"{k:10s} {v:7.3f} s")
by_layer = {}
for k, v in ph.items():
    parts = k.split("/")
    j = None
    for p_ in parts[1:]:
        if p_.startswith("merge") or p_.startswith("refine"):
            j = int(p_.replace("merge", "").replace("refine", "").split(".")[0])
    key = f"layer {j}" if j is not None else parts[-1]
    by_layer[key] = by_layer.get(key, 0.0) + v
for k, v in sorted(by_layer.items(), key=lambda kv: -kv[1]):
    print(f"{k:10s} {v:7.3f} s")
