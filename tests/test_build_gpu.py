"""GPU construction: the reference's build known-answers, structural
invariants and statistical parity with the reference-built graph.

Ported from /root/reference/pkg/tests/test_build.py, test_graph.py and the
acceptance criteria (test_acceptance.py) -- exact expectations come from
independent numpy oracles (as in the reference suite) or the CPU checker.
"""

import numpy as np
import pytest

import oracle as O
import paper_1912_01059_b200 as ga
from paper_1912_01059_b200.graph import SENTINEL, AdjacencyLayer, Hierarchy

pytestmark = pytest.mark.gpu


def naive_knn_graph(X, k):
    X64 = X.astype(np.float64)
    out = np.empty((X.shape[0], k), dtype=np.int64)
    for i in range(X.shape[0]):
        d = ((X64 - X64[i]) ** 2).sum(axis=1)
        order = [j for j in np.argsort(d, kind="stable")[: k + 1] if j != i]
        out[i] = order[:k]
    return out


def dataset_1d(values):
    return ga.Dataset(np.asarray(values, dtype=np.float32).reshape(-1, 1))


def check_invariants(h):
    X = h.vectors()
    for j, layer in enumerate(h.layers):
        rows = h.rows_for(j)
        adj, nnd, symc, dnn1 = layer.adjacency, layer.nn_dists, layer.sym_count, layer.d_nn1
        assert (symc >= 0).all() and (symc <= layer.k_sym).all()
        for node in range(layer.node_count):
            row = adj[node]
            direct = row[: layer.k_nn]
            filled = direct[direct != SENTINEL]
            assert (direct[len(filled):] == SENTINEL).all()
            dists = nnd[node][: len(filled)]
            assert (np.diff(dists) >= 0).all()
            for nbr, dv in zip(filled, dists):
                assert nbr != node
                assert O.squared_l2(X[rows[node]], X[rows[nbr]]) == dv  # bitwise sequential FP64
            full = row[row != SENTINEL]
            assert len(set(full.tolist())) == len(full)
            assert (row[layer.k_nn + symc[node]:] == SENTINEL).all()
            if len(filled):
                assert dnn1[node] == dists[0]
        if j:
            t = h.to_bottom[j]
            assert len(np.unique(t)) == len(t)
            finer = h.to_bottom[j - 1]
            if finer is not None:
                assert set(t.tolist()) <= set(finer.tolist())


def test_single_batch_builds_equal_bruteforce():
    """Criterion 1: single-batch builds reproduce the exact kNN graph."""
    rng = np.random.default_rng(101)
    cases = 0
    for n in (32, 64):
        for d in (4, 16):
            for _ in range(5):
                X = rng.standard_normal((n, d)).astype(np.float32)
                cfg = ga.BuildConfig(k=12, k_nn=6, k_sym=6, s=n, g=2, refinements=0, seed=cases)
                h, _ = ga.build(ga.Dataset(X), cfg)
                assert h.num_layers == 1
                np.testing.assert_array_equal(h.layers[0].adjacency[:, :6], naive_knn_graph(X, 6))
                cases += 1
    assert cases == 20


def test_geometry_2048():
    ds = ga.gen_synthetic(2048, 4, seed=1, law="uniform")
    h, _ = ga.build(ds, ga.BuildConfig(k=6, k_nn=3, k_sym=3, s=32, g=4, refinements=0, seed=0))
    assert [L.node_count for L in h.layers] == [2048, 512, 128, 32]
    assert h.stats.d_nn1_max >= h.stats.d_nn1_mean >= 0
    check_invariants(h)


def test_too_small_dataset():
    with pytest.raises(ga.ConfigError, match="at least"):
        ga.build(ga.gen_synthetic(8, 4, seed=1), ga.BuildConfig(k=6, k_nn=3, k_sym=3, s=16, g=2))


def test_deterministic():
    ds = ga.gen_synthetic(300, 8, seed=4, law="clustered", clusters=6)
    cfg = ga.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, refinements=1, seed=9)
    h1, _ = ga.build(ds, cfg)
    h2, _ = ga.build(ds, cfg)
    for a, b in zip(h1.layers, h2.layers):
        np.testing.assert_array_equal(a.adjacency, b.adjacency)
        np.testing.assert_array_equal(a.nn_dists, b.nn_dists)
        np.testing.assert_array_equal(a.sym_count, b.sym_count)
    assert h1.stats == h2.stats


def test_compute_stats_examples():
    dup = ga.Dataset(np.ones((8, 2), dtype=np.float32))
    h, _ = ga.build(dup, ga.BuildConfig(k=4, k_nn=2, k_sym=2, s=8, g=2, refinements=0, seed=0))
    assert h.stats.d_nn1_mean == 0.0 and h.stats.d_nn1_max == 0.0
    h, _ = ga.build(dataset_1d(list(range(10))), ga.BuildConfig(k=4, k_nn=2, k_sym=2, s=10, g=2, refinements=0))
    assert h.stats.d_nn1_mean == 1.0 and h.stats.d_nn1_max == 1.0


def test_stats_match_oracle_nn():
    X = np.random.default_rng(5).standard_normal((64, 6)).astype(np.float32)
    h, _ = ga.build(ga.Dataset(X), ga.BuildConfig(k=8, k_nn=4, k_sym=4, s=64, g=2, refinements=0, seed=0))
    nn = []
    for i in range(64):
        d = ((X.astype(np.float64) - X[i].astype(np.float64)) ** 2).sum(axis=1)
        d[i] = np.inf
        nn.append(d.min())
    assert h.stats.d_nn1_max == pytest.approx(max(nn), rel=1e-12)
    assert h.stats.d_nn1_mean == pytest.approx(np.mean(nn), rel=1e-12)


def test_build_base_1d_example():
    ds = dataset_1d([0, 1, 3, 7])
    layer = AdjacencyLayer(4, 4, 2)
    ga.build_base(layer, ds.vectors, np.arange(4, dtype=np.int32), np.arange(4, dtype=np.int32))
    np.testing.assert_array_equal(layer.adjacency[:, :2], [[1, 2], [0, 2], [1, 0], [2, 1]])
    np.testing.assert_array_equal(layer.nn_dists[0], [1.0, 9.0])
    assert layer.d_nn1[3] == 16.0


def test_build_base_small_batch_reduces_k():
    layer = AdjacencyLayer(3, 8, 4)
    reduced = ga.build_base(layer, dataset_1d([0, 1, 2]).vectors, np.arange(3, dtype=np.int32),
                            np.arange(3, dtype=np.int32))
    assert reduced and (layer.adjacency[:, 2:4] == SENTINEL).all()


def two_batch_1d_hierarchy():
    ds = dataset_1d([0, 1, 2, 3, 4, 5, 6, 7])
    cfg = ga.BuildConfig(k=4, k_nn=2, k_sym=2, s=4, g=2, refinements=0, seed=0)
    bottom = AdjacencyLayer(8, 4, 2)
    h = Hierarchy([bottom], [None], s=4, g=2, config=cfg, dim=1)
    h.attach(ds)
    h.bottom_segment_of = np.array([0, 0, 0, 0, 1, 1, 1, 1], dtype=np.int32)
    h.bottom_perm = np.arange(8, dtype=np.int32)
    h.layer_offsets = [np.array([0, 4, 8], dtype=np.int64)]
    for batch in (np.arange(4, dtype=np.int32), np.arange(4, 8, dtype=np.int32)):
        ga.build_base(bottom, ds.vectors, h.rows_for(0), batch)
    top = AdjacencyLayer(4, 4, 2)
    h.layers.append(top)
    h.to_bottom.append(np.array([1, 3, 4, 6], dtype=np.int32))
    ga.build_base(top, ds.vectors, h.rows_for(1), np.arange(4, dtype=np.int32))
    return ds, h


def test_merge_creates_cross_partition_links():
    ds, h = two_batch_1d_hierarchy()
    bottom = h.layers[0]
    np.testing.assert_array_equal(np.sort(bottom.adjacency[3, :2]), [1, 2])
    ga.merge_layer(h, 0, tau_build=0.5)
    np.testing.assert_array_equal(np.sort(bottom.adjacency[3, :2]), [2, 4])
    np.testing.assert_array_equal(np.sort(bottom.adjacency[4, :2]), [3, 5])


def test_single_subtree_refine_is_noop():
    ds = ga.gen_synthetic(32, 4, seed=5)
    cfg = ga.BuildConfig(k=6, k_nn=3, k_sym=3, s=32, g=2, refinements=0, seed=1)
    h, _ = ga.build(ds, cfg)
    before = h.layers[0].adjacency.copy()
    ga.refine_layer(h, 0, cfg.tau_build)
    np.testing.assert_array_equal(h.layers[0].adjacency, before)


def test_mutual_pair_untouched():
    ds = dataset_1d([0.0, 1.0, 10.0, 11.0])
    cfg = ga.BuildConfig(k=4, k_nn=2, k_sym=2, s=4, g=2, refinements=0, seed=0)
    layer = AdjacencyLayer(4, 4, 2)
    h = Hierarchy([layer], [None], s=4, g=2, config=cfg, dim=1)
    h.attach(ds)
    ga.build_base(layer, ds.vectors, h.rows_for(0), np.arange(4, dtype=np.int32))
    ga.symmetrize(h, 0, tau_build=0.5)
    assert (layer.sym_count == 0).all()


def test_asymmetric_chain_gets_inverse_link():
    ds = dataset_1d([0.0, 1.0, 10.0])
    cfg = ga.BuildConfig(k=2, k_nn=1, k_sym=1, s=2, g=2, refinements=0, seed=0)
    layer = AdjacencyLayer(3, 2, 1)
    h = Hierarchy([layer], [None], s=2, g=2, config=cfg, dim=1)
    h.attach(ds)
    ga.build_base(layer, ds.vectors, h.rows_for(0), np.arange(3, dtype=np.int32))
    assert layer.adjacency[2, 0] == 1 and layer.adjacency[1, 0] == 0
    ga.symmetrize(h, 0, tau_build=0.5)
    assert list(layer.neighbors(1)) == [0, 2]


def test_merge_requires_bookkeeping():
    ds, h = two_batch_1d_hierarchy()
    h.bottom_segment_of = None
    with pytest.raises(RuntimeError, match="freshly built"):
        ga.merge_layer(h, 0, 0.5)


def test_built_layer_invariants_and_cross_partition_links():
    rng = np.random.default_rng(7)
    centers = np.array([[0.0] * 8, [50.0] * 8])
    X = (centers[rng.integers(0, 2, size=512)] + rng.normal(0, 0.5, (512, 8))).astype(np.float32)
    h, stats = ga.build(ga.Dataset(X), ga.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, refinements=1, seed=5))
    check_invariants(h)
    batch_of = h.bottom_segment_of
    direct = h.layers[0].adjacency[:, :4]
    missing = sum(not any(batch_of[v] != batch_of[i] for v in direct[i] if v != SENTINEL) for i in range(512))
    assert missing == 0
    assert stats.mean_sym_used < h.config.k / 2


def test_refinement_improves_consensus():
    ds = ga.gen_synthetic(2048, 8, seed=17, law="clustered", clusters=16)
    cfg = ga.BuildConfig(k=8, k_nn=4, k_sym=4, s=32, g=4, refinements=0, seed=2)
    h, _ = ga.build(ds, cfg)
    truth = naive_knn_graph(ds.vectors, 4)
    after = np.mean([len(set(h.layers[0].adjacency[i, :4]) & set(truth[i])) / 4 for i in range(2048)])
    pre = AdjacencyLayer(2048, 8, 4)
    perm, offsets = ga.partition_bottom(2048, 64, np.random.default_rng(cfg.seed))
    for i in range(64):
        ga.build_base(pre, ds.vectors, np.arange(2048, dtype=np.int32), perm[offsets[i]:offsets[i + 1]])
    before = np.mean([len(set(pre.adjacency[i, :4]) & set(truth[i])) / 4 for i in range(2048)])
    assert after >= before


def _recall_at(ids, gt_first, k):
    return float(np.mean([gt_first[i] in ids[i, :k] for i in range(len(gt_first))]))


def test_gpu_built_sift10k_recall_parity(golden_sift):
    """GPU-built graph vs the reference-built graph on the reference's own
    10k x 128 acceptance instance: R@1 and R@10 at tau 0.3/0.6/0.8 within one
    query (0.01) of the reference's, consensus C@10 >= 0.95, sym budget."""
    g, h_ref, Q = golden_sift
    base = h_ref.dataset
    h, stats = ga.build(base, ga.BuildConfig(seed=7))
    assert [L.node_count for L in h.layers] == [L.node_count for L in h_ref.layers]
    X64 = base.vectors.astype(np.float64)
    gt_first = np.array([int(np.argmin(((X64 - q.astype(np.float64)) ** 2).sum(axis=1))) for q in Q])
    for tag, tau in (("q3", 0.3), ("q6", 0.6), ("q8", 0.8)):
        mine = ga.query_arrays(h, Q, ga.QueryConfig(k_out=10, tau=tau)).ids
        ref_ids = g[tag + "_ids"]
        for k in (1, 10):
            assert abs(_recall_at(mine, gt_first, k) - _recall_at(ref_ids, gt_first, k)) <= 0.01 + 1e-12, (tag, k)
    assert stats.mean_sym_used < h.config.k / 4
    sample = np.random.default_rng(0).choice(base.n, 512, replace=False).astype(np.int32)
    knn, _ = ga.search.exact_knn_rows(base, sample, 11)
    adj = h.layers[0].adjacency
    c10 = np.mean([len(set(adj[x, :10]) & set([v for v in knn[i] if v != x][:10])) / 10 for i, x in enumerate(sample)])
    assert c10 >= 0.95, c10


@pytest.mark.parametrize("d", [32, 128, 256])
def test_leaf_knn_tensor_cores_vs_checker(d):
    """tcgen05 kind::i8 leaf kNN (ggnn_leaf_knn_tc): positions and distances
    equal the reference's batch_bruteforce (CPU checker) on integer data with
    heavy distance ties, for batch sizes 2..128."""
    from paper_1912_01059_b200 import _native as N
    from paper_1912_01059_b200.device import DeviceVectors

    rng = np.random.default_rng(d)
    sizes = np.concatenate([[2, 3, 16, 17, 128, 127, 64], rng.integers(2, 129, size=33)])
    n = int(sizes.sum()) + 50
    X = rng.integers(0, 4 if d == 32 else 256, size=(n, d)).astype(np.float32)
    X.setflags(write=False)
    members = rng.permutation(n)[: sizes.sum()].astype(np.int32)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    k_nn = 12
    dv = DeviceVectors.of_array(X)
    assert dv.exact_integers
    t = N.torch()
    pos = N.empty((len(members), k_nn), t.int32)
    dist = N.empty((len(members), k_nn), t.float64)
    red = t.zeros(1, dtype=t.int32, device=N.device())
    mem_d, off_d = N.to_dev(members), N.to_dev(offsets)  # keep the device copies alive across the launch
    N.call("ggnn_leaf_knn_tc", N.ctypes.byref(dv.struct), N.ptr(mem_d), None, N.ptr(off_d),
           len(sizes), int(sizes.max()), k_nn, N.ptr(pos), N.ptr(dist), None, 0, None, None, N.ptr(red),
           N.stream_ptr())
    pos, dist = pos.cpu().numpy(), dist.cpu().numpy()
    assert N.load().ggnn_tc_timeouts() == 0
    assert int(red.item()) == int((sizes < k_nn + 1).sum())
    for b in range(len(sizes)):
        lo, hi = offsets[b], offsets[b + 1]
        p_ref, d_ref = O.batch_bruteforce(X, members[lo:hi], k_nn)
        np.testing.assert_array_equal(pos[lo:hi], p_ref)
        np.testing.assert_array_equal(dist[lo:hi], d_ref)


def _leaf_float(X, sizes, rng, k_nn=12):
    from paper_1912_01059_b200 import _native as N
    from paper_1912_01059_b200.device import DeviceVectors

    n = X.shape[0]
    members = rng.permutation(n)[: sizes.sum()].astype(np.int32)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dv = DeviceVectors.of_array(X)
    assert not dv.exact_integers
    t = N.torch()
    pos = N.empty((len(members), k_nn), t.int32)
    dist = N.empty((len(members), k_nn), t.float64)
    red = t.zeros(1, dtype=t.int32, device=N.device())
    mem_d, off_d = N.to_dev(members), N.to_dev(offsets)
    N.call("ggnn_leaf_knn_tc", N.ctypes.byref(dv.struct), N.ptr(mem_d), None, N.ptr(off_d),
           len(sizes), int(sizes.max()), k_nn, N.ptr(pos), N.ptr(dist), None, 0, None, None, N.ptr(red),
           N.stream_ptr())
    pos, dist = pos.cpu().numpy(), dist.cpu().numpy()
    N.check_tc_timeouts("leaf")
    assert int(red.item()) == int((sizes < k_nn + 1).sum())
    for b in range(len(sizes)):
        lo, hi = offsets[b], offsets[b + 1]
        p_ref, d_ref = O.batch_bruteforce(X, members[lo:hi], k_nn)
        np.testing.assert_array_equal(pos[lo:hi], p_ref)
        np.testing.assert_array_equal(dist[lo:hi], d_ref)


@pytest.mark.parametrize("kind", ["gist", "deep", "ties", "offset"])
def test_leaf_knn_tf32_tensor_cores_vs_checker(kind):
    """Float leaf kNN on tcgen05 kind::tf32 (3xTF32 Gram matrix of the
    centred batch, a rigorous error bound selects candidates, sequential FP64
    re-score): positions and distances bit for bit equal to the reference's
    batch_bruteforce (CPU checker) on the C3 / C4 generators (gist3k / deep3k
    rows), on duplicated rows (exact ties) and on rows far from the origin."""
    rng = np.random.default_rng(len(kind))
    if kind == "gist":
        from paper_1912_01059_b200.synthetic import make_latent16

        X = make_latent16(n=3000, d=960, m=1, seed=1234, as_float=True)[0]
    elif kind == "deep":
        sys_path_golden()
        from make_golden import deep_like

        X = deep_like(3000, 1)[0]
    elif kind == "ties":
        base = rng.standard_normal((700, 64)).astype(np.float32)
        X = np.concatenate([base, base[rng.integers(0, 700, size=700)]]).astype(np.float32)
    else:
        X = (1000.0 + rng.standard_normal((2000, 40)) * 0.01).astype(np.float32)
    X = np.ascontiguousarray(X)
    X.setflags(write=False)
    sizes = np.concatenate([[2, 3, 16, 17, 128, 127, 64], rng.integers(2, 129, size=9)])
    sizes = sizes[np.cumsum(sizes) <= X.shape[0]]
    _leaf_float(X, sizes, rng)


def sys_path_golden():
    import sys
    from pathlib import Path

    p = str(Path(__file__).resolve().parent / "golden")
    if p not in sys.path:
        sys.path.insert(0, p)


def test_build_accounting_counts_every_search():
    """ggnn_search_accounting: the device totals equal the sum of the
    searches' own (visited, steps) counters, and build(..., accounting=True)
    reports per-phase algorithmic bytes (SURVEY 8d build accounting)."""
    from paper_1912_01059_b200 import _native as N
    from paper_1912_01059_b200.synthetic import make_latent16

    base, Q = make_latent16(n=4000, d=32, m=300, seed=2)
    h, st = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7), accounting=True)
    summ = st.accounting_summary(32, 1)
    assert summ["visited_total"] > 0 and summ["steps_total"] > 0 and summ["leaf_knn_flops"] > 0
    assert summ["search_bytes_total"] == sum(
        v * 32 + st.search_steps[k] * (4 * 24 + 4) for k, v in st.search_visited.items())
    t = N.torch()
    acc = t.zeros(2, dtype=t.int64, device=N.device())
    N.call("ggnn_search_accounting", N.ptr(acc))
    try:
        res = ga.search.descent_arrays(h, Q, ga.QueryConfig(k_out=10, tau=0.6), h.num_layers - 1, 0)
    finally:
        N.call("ggnn_search_accounting", None)
    v, s = acc.tolist()
    assert v == int(res.counters[:, 0].astype(np.int64).sum())
    assert s == int(res.counters[:, 1].astype(np.int64).sum())
    # off again: nothing more is counted
    ga.search.descent_arrays(h, Q, ga.QueryConfig(k_out=10, tau=0.6), h.num_layers - 1, 0)
    assert acc.tolist() == [v, s]
