"""ctypes front of the CPU checker oracle/ggnn_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker.  The product package
(paper_1912_01059_b200) never imports it.

Signatures mirror the reference kernel module `graphann._core`
(/root/reference/pkg/src/graphann/_core.pyx): same argument order, same
return tuples, so parity tests read like the reference's test_backends.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libggnn_oracle.so"

TERM_STOPPING = 0
TERM_QUEUE_EMPTY = 1
TERM_ITERATION_CAP = 2

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < (HERE / "ggnn_oracle.c").stat().st_mtime:
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.ggo_sqdist.argtypes = [P, P, i64]
        L.ggo_sqdist.restype = f64
        L.ggo_exhaustive_topk.argtypes = [P, i64, i64, P, i32, P, P]
        L.ggo_exhaustive_topk.restype = i32
        L.ggo_batch_bruteforce.argtypes = [P, i64, P, i32, i32, P, P]
        L.ggo_batch_bruteforce.restype = None
        L.ggo_greedy_search.argtypes = [P, i64, P, P, i64, i32, i32, P, P, P, P, i32, i32, f64,
                                        f64, ctypes.c_long, i32, i32, P, P, P]
        L.ggo_greedy_search.restype = i32
        L.ggo_sym_check_pair.argtypes = [P, i64, P, P, i64, i32, i32, P, i32, i32, f64, f64, f64,
                                         ctypes.c_long, i32, i32, i32, i32, P]
        L.ggo_sym_check_pair.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def squared_l2(a, b) -> float:
    a, b = _f32(a), _f32(b)
    if a.shape[0] != b.shape[0]:
        raise ValueError("vector lengths differ")
    return float(lib().ggo_sqdist(_p(a), _p(b), a.shape[0]))


def squared_l2_many(q, X, rows):
    q, X, rows = _f32(q), _f32(X), _i32(rows)
    return np.array([lib().ggo_sqdist(_p(q), _p(X[r]), X.shape[1]) for r in rows], dtype=np.float64)


def exhaustive_topk(X, q, k):
    X, q = _f32(X), _f32(q)
    k = min(int(k), X.shape[0])
    ids = np.empty(k, dtype=np.int32)
    dists = np.empty(k, dtype=np.float64)
    got = lib().ggo_exhaustive_topk(_p(X), X.shape[0], X.shape[1], _p(q), k, _p(ids), _p(dists))
    return ids[:got], dists[:got]


def batch_bruteforce(X, member_rows, k_nn):
    X, member_rows = _f32(X), _i32(member_rows)
    m = member_rows.shape[0]
    pos = np.empty((m, k_nn), dtype=np.int32)
    dist = np.empty((m, k_nn), dtype=np.float64)
    lib().ggo_batch_bruteforce(_p(X), X.shape[1], _p(member_rows), m, k_nn, _p(pos), _p(dist))
    return pos, dist


def greedy_search(X, to_row, adj, k_nn, sym_count, q, seed_ids, seed_dists, k_out, tau,
                  d_nn1_max, max_iterations, prioq_size, visited_size):
    X, to_row, adj, sym_count, q = _f32(X), _i32(to_row), _i32(adj), _i32(sym_count), _f32(q)
    seed_ids = _i32(seed_ids)
    seed_dists = np.ascontiguousarray(seed_dists, dtype=np.float64)
    ids = np.empty(k_out, dtype=np.int32)
    dists = np.empty(k_out, dtype=np.float64)
    cnt = np.zeros(5, dtype=np.int64)
    nh = lib().ggo_greedy_search(
        _p(X), X.shape[1], _p(to_row), _p(adj), adj.shape[0], adj.shape[1], k_nn, _p(sym_count),
        _p(q), _p(seed_ids), _p(seed_dists), seed_ids.shape[0], k_out, float(tau),
        float(d_nn1_max), int(max_iterations), prioq_size, visited_size, _p(ids), _p(dists),
        _p(cnt))
    if nh < 0:
        raise MemoryError("oracle allocation failed")
    return (ids[:nh].copy(), dists[:nh].copy(), int(cnt[0]), int(cnt[1]), int(cnt[2]),
            int(cnt[3]), int(cnt[4]))


def sym_check_pair(X, to_row, adj, k_nn, sym_count, x, z, d_xz, tau, d_nn1_max, budget, k_out,
                   prioq_size, visited_size, n_fallback, scratch=None):
    X, to_row, adj, sym_count = _f32(X), _i32(to_row), _i32(adj), _i32(sym_count)
    fb = np.full(n_fallback, -1, dtype=np.int32)
    v = lib().ggo_sym_check_pair(
        _p(X), X.shape[1], _p(to_row), _p(adj), adj.shape[0], adj.shape[1], k_nn, _p(sym_count),
        int(x), int(z), float(d_xz), float(tau), float(d_nn1_max), int(budget), int(k_out),
        int(prioq_size), int(visited_size), int(n_fallback), _p(fb))
    if v < 0:
        raise MemoryError("oracle allocation failed")
    return v, fb


def reference_module():
    """The compiled reference (oracle/_ref/graphann_ref, built by build_ref.sh), or None."""
    import sys

    ref_dir = HERE / "_ref"
    if not (ref_dir / "graphann_ref").exists():
        return None
    if str(ref_dir) not in sys.path:
        sys.path.insert(0, str(ref_dir))
    import graphann_ref  # noqa: E402

    return graphann_ref


if os.environ.get("GGNN_ORACLE_BUILD_ON_IMPORT"):
    lib()


def query(layers, to_bottom, X, q, k_out, tau, d_nn1_max, max_iterations=1000, prioq_size=256, visited_size=512):
    """search.query (search.py:115-137) composed from the checker kernels:
    exact top-layer scan, greedy search on layer 0, then the query()
    counter adjustments.  `layers` is a list of (adjacency, k_nn, sym_count)."""
    X = _f32(X)
    top_rows = np.arange(X.shape[0], dtype=np.int32) if len(layers) == 1 else _i32(to_bottom[-1])
    k = min(k_out, len(top_rows))
    local, sd = exhaustive_topk(X[top_rows], q, k)
    seeds = top_rows[local].astype(np.int32)
    adj, k_nn, symc = layers[0]
    ids, dists, v, t, term, distinct, forgotten = greedy_search(
        X, np.arange(X.shape[0], dtype=np.int32), adj, k_nn, symc, q, seeds, sd, k_out, tau, d_nn1_max,
        max_iterations, prioq_size, visited_size)
    return ids, dists, v + len(top_rows), t, term, distinct + len(top_rows) - len(seeds), forgotten


def merge_shard_results(parts, permutation, k_out):
    """_merge_shard_results (shard.py:91-110): `parts` is a list of
    (offset, ids, dists, visited, steps, term_code) per shard with shard-local
    ids; returns (global ids, dists, visited sum, steps sum, term of the best
    hit's shard or 1 (queue-empty) when nothing was found)."""
    pairs = []
    visited = steps = 0
    for offset, ids, dists, v, t, term in parts:
        for local, dist in zip(ids, dists):
            pairs.append((float(dist), int(permutation[offset + int(local)]), int(term)))
        visited += int(v)
        steps += int(t)
    pairs.sort(key=lambda p: (p[0], p[1]))
    top = pairs[:k_out]
    term = top[0][2] if top else TERM_QUEUE_EMPTY
    return (np.array([p[1] for p in top], dtype=np.int32), np.array([p[0] for p in top], dtype=np.float64),
            visited, steps, term)
