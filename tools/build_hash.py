"""Hash of a GPU-built graph (determinism across processes).
Usage: python tools/build_hash.py [latent|deep] [n]"""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_deep_like, make_latent16  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "deep"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
base = make_deep_like(n, 1)[0] if kind == "deep" else make_latent16(n=n, d=128, m=1)[0]
h, st = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
hs = hashlib.sha256()
for L in h.layers:
    hs.update(L.adjacency.tobytes())
    hs.update(L.sym_count.tobytes())
print(kind, n, "graph sha256", hs.hexdigest()[:16], f"build {st.build_seconds:.1f} s")
