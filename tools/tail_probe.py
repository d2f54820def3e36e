"""Does per-query search length correlate with cheap pre-search features?"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
r = ga.query_arrays(h, Q, ga.QueryConfig(k_out=10, tau=0.6))
T = r.counters[:, 1].astype(float)
V = r.counters[:, 0].astype(float)
top = h.to_bottom[-1]
Xt = base[top].astype(np.float64)
d = ((Q.astype(np.float64)[:, None, :] - Xt[None]) ** 2).sum(-1)
ds = np.sort(d, axis=1)
feats = {"d_top1": ds[:, 0], "d_top10": ds[:, 9], "ratio": ds[:, 0] / ds[:, 9], "final_d1": r.dists[:, 0],
         "final_d10": r.dists[:, 9]}
print("T: mean %.1f p50 %.0f p90 %.0f p99 %.0f max %.0f" % (T.mean(), *np.percentile(T, [50, 90, 99]), T.max()))
for k, f in feats.items():
    print(f"corr(T, {k}) = {np.corrcoef(T, f)[0, 1]:+.3f}   spearman {np.corrcoef(np.argsort(np.argsort(T)), np.argsort(np.argsort(f)))[0, 1]:+.3f}")
