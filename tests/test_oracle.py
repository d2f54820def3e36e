"""Pin the CPU checker (oracle/ggnn_oracle.c) to the reference's own outputs.

Every expectation comes from the unmodified compiled reference (golden
fixtures, tests/golden/make_golden.py).  On the reference's arithmetic the
oracle must agree bitwise -- ids, float64 distances and every counter -- on
integer AND float data, because it restates the same sequential FP64 loops.
"""

import numpy as np
import pytest

import oracle as O
from conftest import TERM_CODE, oracle_layers


def test_exhaustive_topk(golden_int):
    g, _ = golden_int
    for i, q in enumerate(g["Q"]):
        ids, d = O.exhaustive_topk(g["X"], q, 9)
        np.testing.assert_array_equal(ids, g["topk_ids"][i])
        np.testing.assert_array_equal(d, g["topk_d"][i])


def test_batch_bruteforce(golden_int):
    g, _ = golden_int
    for b in range(4):
        pos, dist = O.batch_bruteforce(g["X"], g[f"bb_mem{b}"], 6)
        np.testing.assert_array_equal(pos, g[f"bb_pos{b}"])
        np.testing.assert_array_equal(dist, g[f"bb_dist{b}"])


def test_greedy_search_from_seeds(golden_int):
    g, h = golden_int
    L = h.layers[0]
    X = g["X"]
    for i in range(len(g["Q"])):
        seeds = g["gs_seeds"][i]
        sd = np.array([O.squared_l2(g["Q"][i], X[s]) for s in seeds])
        r = O.greedy_search(X, h.rows_for(0), L.adjacency, L.k_nn, L.sym_count, g["Q"][i], seeds, sd, 6, 0.4,
                            h.stats.d_nn1_max, 1000, 12, 16)
        nh = len(r[0])
        np.testing.assert_array_equal(r[0], g["gs_ids"][i, :nh])
        np.testing.assert_array_equal(r[1], g["gs_d"][i, :nh])
        assert tuple(r[2:]) == tuple(int(v) for v in g["gs_cnt"][i])


@pytest.mark.parametrize("tag", ["q_default", "q_tiny", "q_cap"])
def test_query_all_counters(golden_int, tag):
    g, h = golden_int
    k_out, max_it, prioq, vis = (int(v) for v in g[tag + "_cfg"])
    tau = float(g[tag + "_tau"])
    for i, q in enumerate(g["Q"]):
        r = O.query(oracle_layers(h), h.to_bottom, g["X"], q, k_out, tau, h.stats.d_nn1_max, max_it, prioq, vis)
        nh = len(r[0])
        np.testing.assert_array_equal(r[0], g[tag + "_ids"][i, :nh])
        np.testing.assert_array_equal(r[1], g[tag + "_dists"][i, :nh])
        assert tuple(r[2:]) == tuple(int(v) for v in g[tag + "_cnt"][i]), (tag, i)


def test_sym_check_pair(golden_int):
    g, h = golden_int
    L = h.layers[0]
    X = g["X"]
    for (x, z), v, fb in zip(g["sym_pairs"], g["sym_verdict"], g["sym_fb"]):
        got_v, got_fb = O.sym_check_pair(X, h.rows_for(0), L.adjacency, L.k_nn, L.sym_count, int(x), int(z),
                                         O.squared_l2(X[x], X[z]), 0.5, L.live_d_nn1_max(), 16, 4, 64, 128, 8)
        assert got_v == v
        if v == 2:
            np.testing.assert_array_equal(got_fb, fb)


def test_float_queries_bitwise(golden_float):
    """Float data: the checker follows the reference's sequential FP64 sums,
    so it is bitwise equal there too."""
    g, h = golden_float
    for i, q in enumerate(g["Q"]):
        r = O.query(oracle_layers(h), h.to_bottom, g["X"], q, 5, 0.6, h.stats.d_nn1_max)
        nh = len(r[0])
        np.testing.assert_array_equal(r[0], g["q_ids"][i, :nh])
        np.testing.assert_array_equal(r[1], g["q_dists"][i, :nh])
        assert tuple(r[2:]) == tuple(int(v) for v in g["q_cnt"][i])


def test_sift10k_queries_bitwise(golden_sift):
    g, h, Q = golden_sift
    for tag, tau in (("q3", 0.3), ("q6", 0.6), ("q8", 0.8)):
        for i in range(0, len(Q), 5):
            r = O.query(oracle_layers(h), h.to_bottom, h.vectors(), Q[i], 10, tau, h.stats.d_nn1_max)
            np.testing.assert_array_equal(r[0], g[tag + "_ids"][i, : len(r[0])])
            np.testing.assert_array_equal(r[1], g[tag + "_dists"][i, : len(r[1])])
            assert tuple(r[2:]) == tuple(int(v) for v in g[tag + "_cnt"][i])


def test_term_codes_match_reference():
    assert TERM_CODE == {"stopping-rule": O.TERM_STOPPING, "queue-empty": O.TERM_QUEUE_EMPTY,
                         "iteration-cap": O.TERM_ITERATION_CAP}
