"""The kernel seam on the GPU: the functions of the reference's `graphann._core`
(/root/reference/pkg/src/graphann/_core.pyx) with the same names, arguments
and return values, each executed by libggnn_b200.so.  Host arrays are copied
to the device per call (read-only dataset tables are cached), so these
per-call entry points exist for drop-in compatibility; the library's own
build / query code calls the batched C ABI directly.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .device import DeviceVectors, sanitize

TERM_STOPPING = 0
TERM_QUEUE_EMPTY = 1
TERM_ITERATION_CAP = 2


def _identity_or_none(to_row: np.ndarray, n: int):
    to_row = np.ascontiguousarray(to_row, dtype=np.int32)
    if to_row.shape[0] <= n and np.array_equal(to_row, np.arange(to_row.shape[0], dtype=np.int32)):
        return None
    return N.to_dev(to_row)


def _query_dev(dv: DeviceVectors, q: np.ndarray):
    q = np.ascontiguousarray(q, dtype=np.float32).reshape(1, -1)
    return dv.queries(q)


def squared_l2(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.shape[0] != b.shape[0]:
        raise ValueError("vector lengths differ")
    return float(squared_l2_many(a, b[None, :], np.zeros(1, dtype=np.int32))[0])


def squared_l2_many(q, X, rows) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float32)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    dv = DeviceVectors.of_array(X)
    keep, qs = _query_dev(dv, q)
    out = N.empty((rows.shape[0],), N.torch().float64)
    rd = N.to_dev(rows)
    N.call("ggnn_squared_l2_many", ctypes.byref(dv.struct), ctypes.byref(qs), N.ptr(rd), rows.shape[0], N.ptr(out),
           N.stream_ptr())
    return out.cpu().numpy()


def _topk(dv, rows_dev, nrows, q, k):
    keep, qs = _query_dev(dv, q)
    k = int(min(k, nrows))
    t = N.torch()
    ids = N.empty((1, k), t.int32)
    dists = N.empty((1, k), t.float64)
    N.call("ggnn_exhaustive_topk", ctypes.byref(dv.struct), N.ptr(rows_dev), nrows, ctypes.byref(qs), k, N.ptr(ids),
           N.ptr(dists), N.stream_ptr())
    ids, dists = ids.cpu().numpy()[0], dists.cpu().numpy()[0]
    N.check_tc_timeouts("bf")
    return ids, dists


def exhaustive_topk(X, q, k):
    """Exact top-k of q against every row of X; ties by ascending row."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    dv = DeviceVectors.of_array(X)
    return _topk(dv, None, X.shape[0], q, k)


def exhaustive_topk_rows(dataset, rows, q, k):
    """exhaustive_topk over X[rows] without gathering on the host; returned ids
    are positions into `rows`."""
    dv = DeviceVectors.of(dataset)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    return _topk(dv, N.to_dev(rows), rows.shape[0], q, k)


def batch_bruteforce(X, member_rows, k_nn):
    """Within-batch exact kNN: (positions into member_rows, dists), -1 / inf
    padded (_core.pyx:107-130)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    member_rows = np.ascontiguousarray(member_rows, dtype=np.int32)
    m = member_rows.shape[0]
    if m == 0:
        return np.full((0, k_nn), -1, dtype=np.int32), np.full((0, k_nn), np.inf)
    dv = DeviceVectors.of_array(X)
    t = N.torch()
    nodes = N.to_dev(member_rows)
    offs = N.to_dev(np.array([0, m], dtype=np.int64))
    pos = N.empty((m, k_nn), t.int32)
    dist = N.empty((m, k_nn), t.float64)
    N.call("ggnn_leaf_knn", ctypes.byref(dv.struct), N.ptr(nodes), None, N.ptr(offs), 1, m, k_nn, N.ptr(pos),
           N.ptr(dist), None, 0, None, None, None, N.stream_ptr())
    pos, dist = pos.cpu().numpy(), dist.cpu().numpy()
    N.check_tc_timeouts("leaf")
    return pos, dist


def _layer_struct(adj, k_nn, sym_count, to_row_dev):
    adj = np.ascontiguousarray(adj, dtype=np.int32)
    nc, k = adj.shape
    san = sanitize(N.to_dev(adj), N.to_dev(np.ascontiguousarray(sym_count, dtype=np.int32)), nc, k, k_nn)
    return san, N.Layer(N.ptr(san), N.ptr(to_row_dev), None, nc, k, k_nn, 0.0)


def greedy_search(X, to_row, adj, k_nn, sym_count, q, seed_ids, seed_dists, k_out, tau, d_nn1_max, max_iterations,
                  prioq_size, visited_size):
    """Returns (ids, dists, visited_count, steps, term, distinct, forgotten)
    exactly like _core.greedy_search (_core.pyx:314-353)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    dv = DeviceVectors.of_array(X)
    tr = _identity_or_none(to_row, X.shape[0])
    san, layer = _layer_struct(adj, k_nn, sym_count, tr)
    keep, qs = _query_dev(dv, q)
    seed_ids = np.ascontiguousarray(seed_ids, dtype=np.int32).reshape(1, -1)
    seed_dists = np.ascontiguousarray(seed_dists, dtype=np.float64).reshape(1, -1)
    # exact re-score whenever keys are FP64 (float table, or float queries on a
    # uint8 table); the kernel ignores the flag for exact uint8 / uint8 keys
    flags = N.FLAG_DISTINCT | N.FLAG_EXACT_DISTS
    params = N.search_params(k_out, prioq_size, visited_size, tau, max_iterations, flags)
    t = N.torch()
    ids = N.empty((1, k_out), t.int32)
    dists = N.empty((1, k_out), t.float64)
    cnt = N.empty((1, 5), t.int32)
    sid, sd = N.to_dev(seed_ids), N.to_dev(seed_dists)
    for exact in (False, True):  # compact distinct-set first; exact on overflow (-1)
        nb = N.load().ggnn_search_workspace_bytes(1, ctypes.byref(params), -1 if exact else seed_ids.shape[1])
        ws = N.empty((max(nb, 1),), t.uint8)
        N.call("ggnn_greedy_batch", ctypes.byref(dv.struct), ctypes.byref(layer), ctypes.byref(qs), N.ptr(sid),
               N.ptr(sd), seed_ids.shape[1], ctypes.byref(params), float(d_nn1_max), N.ptr(ids), N.ptr(dists),
               N.ptr(cnt), N.ptr(ws), nb, N.stream_ptr())
        if int(cnt[0, 3].item()) >= 0:
            break
    ids, dists, c = ids.cpu().numpy()[0], dists.cpu().numpy()[0], cnt.cpu().numpy()[0]
    nh = int((ids >= 0).sum())
    return ids[:nh].copy(), dists[:nh].copy(), int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[4])


class SymScratch:
    """Interface twin of the reference's per-worker scratch (_core.pyx:356-372);
    device state is per launch, so only the fallback buffer lives here."""

    def __init__(self, node_count, k_total, cap, visited_size, budget, n_fallback):
        self.fb = np.full(n_fallback, -1, dtype=np.int32)


def sym_check_pair(X, to_row, adj, k_nn, sym_count, x, z, d_xz, tau, d_nn1_max, budget, k_out, prioq_size,
                   visited_size, n_fallback, scratch):
    """(verdict, fallbacks) of one reachability check (_core.pyx:375-435)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    dv = DeviceVectors.of_array(X)
    tr = _identity_or_none(to_row, X.shape[0])
    san, layer = _layer_struct(adj, k_nn, sym_count, tr)
    t = N.torch()
    px = N.to_dev(np.array([x], dtype=np.int32))
    pz = N.to_dev(np.array([z], dtype=np.int32))
    pd = N.to_dev(np.array([d_xz], dtype=np.float64))
    verdict = N.empty((1,), t.int32)
    fb = N.empty((1, max(n_fallback, 1)), t.int32)
    N.call("ggnn_sym_check_batch", ctypes.byref(dv.struct), ctypes.byref(layer), N.ptr(px), N.ptr(pz), N.ptr(pd), 1,
           float(tau), float(d_nn1_max), int(budget), int(k_out), int(prioq_size), int(visited_size),
           int(n_fallback), N.ptr(verdict), N.ptr(fb), N.stream_ptr())
    scratch.fb[:] = fb.cpu().numpy()[0, :n_fallback]
    return int(verdict.item()), scratch.fb
