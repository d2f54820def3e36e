"""Acceptance criteria of the reference suite (tests/test_acceptance.py) on
the GPU path: recall level and monotonicity over tau (criterion 2), two
shards vs one index (criterion 6), and >= 10^4 randomized queries with
invariant checks on adversarial data (criterion 7: all-identical and
duplicate-heavy tables, tiny caches, a single-node layer)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1912_01059_b200 as ga
from paper_1912_01059_b200.synthetic import make_sift_shaped

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bench():
    base, queries = make_sift_shaped()  # the reference's synthetic bench_data (conftest.py:79-87)
    ds = ga.Dataset(base)
    gt = ga.brute_force_oracle(ds, queries, 10).ids
    h, _ = ga.build(ds, ga.BuildConfig(seed=7))
    return ds, queries, gt, h


def test_criterion2_recall_and_monotone_sweep(bench):
    ds, Q, gt, h = bench
    r1 = [ga.recall_at(ga.query_arrays(h, Q, ga.QueryConfig(k_out=10, tau=t)).ids, gt[:, 0], 1)
          for t in (0.3, 0.4, 0.5, 0.6, 0.7, 0.8)]
    assert r1[3] >= 0.95, r1
    assert all(b >= a - 1e-12 for a, b in zip(r1, r1[1:])), r1


def test_criterion6_two_shards_close_to_one(bench):
    ds, Q, gt, h = bench
    cfg = ga.QueryConfig(k_out=10, tau=0.6)
    single = ga.recall_at(ga.query_arrays(h, Q, cfg).ids, gt[:, 0], 1)
    si, _ = ga.build_sharded(ds, ds.n // 2, ga.BuildConfig(seed=7))
    sharded = ga.recall_at(ga.query_sharded_arrays(si, Q, cfg).ids, gt[:, 0], 1)
    assert abs(single - sharded) <= 0.02, (single, sharded)


def test_criterion7_randomized_invariants():
    rng = np.random.default_rng(707)
    datasets = [
        ga.gen_synthetic(512, 8, seed=1, law="uniform"),
        ga.gen_synthetic(512, 8, seed=2, law="clustered", clusters=6),
        ga.Dataset(np.ones((128, 8), dtype=np.float32)),
        ga.Dataset(np.repeat(np.random.default_rng(3).standard_normal((16, 8)), 8, axis=0).astype(np.float32)),
    ]
    cfgs = (ga.QueryConfig(k_out=4, tau=0.6, max_iterations=50, prioq_size=8, visited_size=8),
            ga.QueryConfig(k_out=4, tau=0.6))
    checked = 0
    for ds in datasets:
        h, _ = ga.build(ds, ga.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, refinements=1, seed=5))
        X = ds.vectors
        layers = [(L.adjacency, L.k_nn, L.sym_count) for L in h.layers]
        for cfg in cfgs:
            Q = (X[rng.integers(0, ds.n, size=1300)] + rng.standard_normal((1300, 8)).astype(np.float32) * 0.3)
            Q = Q.astype(np.float32)
            res = ga.batch_query(h, Q, cfg)
            for i, r in enumerate(res):
                assert r.steps <= cfg.max_iterations
                assert r.terminated_by in ("stopping-rule", "queue-empty", "iteration-cap")
                for node, dist in r.hits:
                    assert O.squared_l2(Q[i], X[node]) == dist  # exact sequential FP64
                assert len(set(r.ids.tolist())) == len(r.ids)
                assert r.visited_count <= r.distinct_touched + r.forgotten
                checked += 1
            # and the same graph through the CPU checker: identical ids on float data
            # except distance near-ties (rel 1e-5)
            for i in range(0, 1300, 97):
                ids, dd, *_ = O.query(layers, h.to_bottom, X, Q[i], cfg.k_out, cfg.tau, h.stats.d_nn1_max,
                                      cfg.max_iterations, cfg.prioq_size, cfg.visited_size)
                if not np.array_equal(res[i].ids, ids):
                    np.testing.assert_allclose(res[i].dists, dd, rtol=1e-5)
    # single-node layer: the only point is expanded, then the queue is empty
    one = ga.Dataset(np.zeros((1, 4), dtype=np.float32))
    h1 = ga.Hierarchy([ga.AdjacencyLayer(1, 4, 2)], [None], 4, 2, ga.BuildConfig(k=4, k_nn=2, k_sym=2, s=4, g=2),
                      dim=4)
    h1.attach(one)
    r = ga.query(h1, np.zeros(4, dtype=np.float32), ga.QueryConfig(k_out=2, tau=0.6))
    assert r.hits[0] == (0, 0.0) and r.terminated_by == "queue-empty"
    checked += 1
    assert checked >= 10_000
