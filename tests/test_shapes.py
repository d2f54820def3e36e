"""The float benchmark shapes (BASELINE.json configs C3 and C4) at sizes the
reference builds in seconds: GIST-like latent16 d=960 floats and Deep-like
L2-normalised clustered d=96 floats (tests/golden/make_golden.py).

* CPU: the checker reproduces the reference's query() on the reference's
  graph bit for bit (pins the oracle on float data).
* GPU, same graph: ids identical except distance near-ties within 1e-5
  relative, distances within 1e-4 relative (north star); in fact the
  returned distances are the sequential FP64 sums, equal to the reference's.
* GPU-built graph: recall within 3 queries of the reference-built graph's
  on 200 queries (the 1M-scale 0.5-point comparison is bench.py's job).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle as O
import paper_1912_01059_b200 as ga
from conftest import golden_hierarchy, load_golden

SHAPES = ("gist3k", "deep3k")


def _data(name):
    from paper_1912_01059_b200.synthetic import make_latent16

    if name == "gist3k":
        base, q = make_latent16(n=3000, d=960, m=200, seed=1234, as_float=True)
    else:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
        from make_golden import deep_like

        base, q = deep_like(3000, 200)
    return base, q


def _golden(name):
    g = load_golden(f"{name}.npz")
    base, q = _data(name)
    assert hashlib.sha256(base.tobytes() + q.tobytes()).hexdigest() == str(g["data_sha256"])
    return g, base, q


@pytest.mark.parametrize("name", SHAPES)
def test_checker_matches_reference_float_queries(name):
    g, base, q = _golden(name)
    h = golden_hierarchy(g, base)
    layers = [(L.adjacency, L.k_nn, L.sym_count) for L in h.layers]
    for i in range(0, len(q), 4):
        ids, dd, v, t, term, _, _ = O.query(layers, h.to_bottom, base, q[i], 10, 0.6, h.stats.d_nn1_max)
        nh = len(ids)
        np.testing.assert_array_equal(ids, g["q_ids"][i, :nh])
        np.testing.assert_array_equal(dd, g["q_dists"][i, :nh])
        assert (v, t, term) == tuple(int(c) for c in g["q_cnt"][i, :3])


def _near_tie_equal(ids, dists, ref_ids, ref_dists, rel=1e-5):
    """ids equal, or every mismatching position is a distance near-tie."""
    if np.array_equal(ids, ref_ids):
        return True
    bad = ids != ref_ids
    a, b = dists[bad], ref_dists[bad]
    return bool(np.all(np.abs(a - b) <= rel * np.maximum(np.abs(b), 1e-30)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", SHAPES)
def test_same_graph_float_parity(name):
    g, base, q = _golden(name)
    h = golden_hierarchy(g, base)
    res = ga.query_arrays(h, q, ga.QueryConfig(k_out=10, tau=0.6))
    exact = 0
    for i in range(len(q)):
        ok = _near_tie_equal(res.ids[i], res.dists[i], g["q_ids"][i], g["q_dists"][i])
        assert ok, (i, res.ids[i], g["q_ids"][i])
        exact += int(np.array_equal(res.ids[i], g["q_ids"][i]))
        m = g["q_ids"][i] >= 0
        np.testing.assert_allclose(res.dists[i][m], g["q_dists"][i][m], rtol=1e-4)
    assert exact >= 0.95 * len(q)


def _recall(ids, first, k):
    return float(np.mean([first[i] in ids[i, :k] for i in range(len(first))]))


# On the tiny, strongly clustered Deep-like instance (64 well-separated
# clusters of ~47 points) every cross-cluster link is an inverse link created
# by symmetrize, so the graph depends on the order in which the reference
# merges and symmetrizes nodes in place: a single snapshot pass loses 3.5
# points (the reference itself, patched to merge from one snapshot, drops
# from 0.98 to 0.93).  The GPU build's node windows (64 merge / 128 sym for
# layers <= 20k nodes, build._merge_windows / _sym_windows) bring both
# shapes to within one query of the reference at every tau.
RECALL_SLACK = {"gist3k": 2 / 200, "deep3k": 2 / 200}


@pytest.mark.gpu
@pytest.mark.parametrize("name", SHAPES)
def test_gpu_built_float_recall_vs_reference(name):
    g, base, q = _golden(name)
    ds = ga.Dataset(base)
    h, stats = ga.build(ds, ga.BuildConfig(seed=7))
    href = golden_hierarchy(g, base)
    for j in range(1, h.num_layers):  # same RNG stream, same weights -> same layer members
        np.testing.assert_array_equal(np.sort(h.to_bottom[j]), np.sort(href.to_bottom[j]))
    gt = ga.brute_force_oracle(ds, q, 10)
    mine = ga.query_arrays(h, q, ga.QueryConfig(k_out=10, tau=0.6)).ids
    for k in (1, 10):
        r_mine, r_ref = _recall(mine, gt.ids[:, 0], k), _recall(g["q_ids"], gt.ids[:, 0], k)
        assert r_mine >= r_ref - RECALL_SLACK[name], (k, r_mine, r_ref)


@pytest.mark.gpu
def test_gpu_built_latent20k_recall_within_half_point():
    """North-star build parity on the benchmark generator (latent16, 20k x 128,
    2000 fresh queries): R@1 and R@10 of the GPU-built graph are within 0.5
    points of the reference-built graph's at tau 0.3 / 0.45 / 0.6, same
    BuildConfig(seed=7), ground truth from the GPU brute force."""
    from paper_1912_01059_b200.synthetic import make_latent16

    g = load_golden("latent20k.npz")
    base, q = make_latent16(n=20000, d=128, m=2000, seed=1234)
    assert hashlib.sha256(base.tobytes() + q.tobytes()).hexdigest() == str(g["data_sha256"])
    ds = ga.Dataset(base)
    h, _ = ga.build(ds, ga.BuildConfig(seed=7))
    first = ga.brute_force_oracle(ds, q, 1).ids[:, 0]
    report = []
    for tau in (0.3, 0.45, 0.6):
        t = f"{int(round(tau * 100)):03d}"
        mine = ga.query_arrays(h, q, ga.QueryConfig(k_out=10, tau=tau)).ids
        for k in (1, 10):
            r_mine, r_ref = _recall(mine, first, k), _recall(g[f"q{t}_ids"], first, k)
            report.append((tau, k, r_mine, r_ref))
    print(report)
    for tau, k, r_mine, r_ref in report:
        assert r_mine >= r_ref - 0.005, report


@pytest.mark.gpu
def test_gpu_built_latent200k_recall_within_half_point():
    """Build parity one order of magnitude closer to C2 (the benchmark's
    latent16 generator at 200k x 128, 5000 fresh queries; the reference's
    own build took 2155 s on one core): R@1 and R@10 of the GPU-built graph
    within 0.5 points of the reference-built graph at tau 0.3 / 0.45 / 0.6,
    same BuildConfig(seed=7), ground truth from the GPU brute force."""
    from paper_1912_01059_b200.synthetic import make_latent16

    g = load_golden("latent200k.npz")
    base, q = make_latent16(n=200_000, d=128, m=5000, seed=1234)
    assert hashlib.sha256(base.tobytes() + q.tobytes()).hexdigest() == str(g["data_sha256"])
    ds = ga.Dataset(base)
    h, _ = ga.build(ds, ga.BuildConfig(seed=7))
    first = ga.brute_force_oracle(ds, q, 1).ids[:, 0]
    report = []
    for tau in (0.3, 0.45, 0.6):
        t = f"{int(round(tau * 100)):03d}"
        mine = ga.query_arrays(h, q, ga.QueryConfig(k_out=10, tau=tau)).ids
        for k in (1, 10):
            report.append((tau, k, _recall(mine, first, k), _recall(g[f"q{t}_ids"], first, k)))
    print(report)
    for tau, k, r_mine, r_ref in report:
        assert r_mine >= r_ref - 0.005, report


@pytest.mark.gpu
def test_gpu_built_deep100k_recall():
    """Medium-scale build parity on the C4 generator (1024 clusters, rows
    L2-normalised, 100k x 96, 1000 held-out queries): R@10 of the GPU-built
    graph vs the reference-built graph at tau 0.3 / 0.6 / 1.0 / 2.0."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_golden import deep_c4

    g = load_golden("deep100k.npz")
    base, q = deep_c4(100_000, 1000)
    assert hashlib.sha256(base.tobytes() + q.tobytes()).hexdigest() == str(g["data_sha256"])
    ds = ga.Dataset(base)
    h, _ = ga.build(ds, ga.BuildConfig(seed=7))
    first = ga.brute_force_oracle(ds, q, 1).ids[:, 0]
    report = []
    for tau in (0.3, 0.6, 1.0, 2.0):
        t = f"{int(round(tau * 100)):03d}"
        mine = ga.query_arrays(h, q, ga.QueryConfig(k_out=10, tau=tau)).ids
        report.append((tau, _recall(mine, first, 10), _recall(g[f"q{t}_ids"], first, 10)))
    print(report)
    for tau, r_mine, r_ref in report:
        assert r_mine >= r_ref - DEEP100K_SLACK, report


DEEP100K_SLACK = 0.01  # 1000 queries: one point is ~one standard error of a recall estimate
