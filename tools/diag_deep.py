"""Compare GPU-built vs reference-built graphs on the deep3k / gist3k fixtures."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "oracle")]
import paper_1912_01059_b200 as ga  # noqa: E402
from conftest import golden_hierarchy, load_golden  # noqa: E402
from test_shapes import _data  # noqa: E402


def c10(h, ds, sample):
    knn, _ = ga.search.exact_knn_rows(ds, sample, 11)
    adj = h.layers[0].adjacency
    return np.mean([len(set(adj[x, :10]) & set([v for v in knn[i] if v != x][:10])) / 10 for i, x in enumerate(sample)])


for name in sys.argv[1:] or ["deep3k", "gist3k"]:
    g = load_golden(f"{name}.npz")
    base, q = _data(name)
    ds = ga.Dataset(base)
    href = golden_hierarchy(g, base)
    h, st = ga.build(ds, ga.BuildConfig(seed=7))
    gt = ga.brute_force_oracle(ds, q, 10).ids[:, 0]
    sample = np.arange(0, 3000, 3, dtype=np.int32)
    print(name, "layers", [L.node_count for L in h.layers], [L.node_count for L in href.layers])
    print(" C@10 gpu %.4f ref %.4f" % (c10(h, ds, sample), c10(href, ds, sample)))
    print(" sym used gpu %.3f ref %.3f dropped %d" % (h.layers[0].sym_count.mean(), href.layers[0].sym_count.mean(),
                                                     st.dropped_sym_links))
    print(" d_nn1_max gpu %.5g ref %.5g" % (h.stats.d_nn1_max, href.stats.d_nn1_max))
    for tau in (0.3, 0.6, 1.0, 2.0):
        for lab, hh in (("gpu", h), ("ref-graph", href)):
            r = ga.query_arrays(hh, q, ga.QueryConfig(k_out=10, tau=tau))
            rec1 = np.mean(r.ids[:, 0] == gt)
            rec10 = np.mean([gt[i] in r.ids[i] for i in range(len(gt))])
            print(f"  tau {tau} {lab:10s} R@1 {rec1:.3f} R@10 {rec10:.3f} V {r.counters[:, 0].mean():.0f} T {r.counters[:, 1].mean():.1f}")
