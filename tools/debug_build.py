"""Debug helper: one small multi-level GPU build (run under compute-sanitizer)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1912_01059_b200 as ga  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
ds = ga.gen_synthetic(n, 4, seed=1, law="uniform")
h, st = ga.build(ds, ga.BuildConfig(k=6, k_nn=3, k_sym=3, s=32, g=4, refinements=0, seed=0))
print("layers", [L.node_count for L in h.layers], "stats", h.stats, "dropped", st.dropped_sym_links)
