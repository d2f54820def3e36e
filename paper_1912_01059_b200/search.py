"""Greedy best-first graph search on the GPU (drop-in for graphann.search).

API and result types follow /root/reference/pkg/src/graphann/search.py; each
call is one batched kernel launch (ggnn_query_batch / ggnn_greedy_batch /
ggnn_descent_batch) instead of the reference's per-query C call.  All
distances are squared L2; tau is applied in squared space (search.py:45-54).
"""

from __future__ import annotations

import gc
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .config import QueryConfig
from .device import DeviceVectors, device_hierarchy

TERMINATED_BY = {0: "stopping-rule", 1: "queue-empty", 2: "iteration-cap"}

# queries per rerun launch when a compact distinct-set overflowed (their exact
# per-query sets live in device workspace, up to 256 KB each)
_DISTINCT_CHUNK = 512


@dataclass(slots=True)
class QueryResult:
    """Ascending (id, distance) results plus search-effort diagnostics."""

    ids: np.ndarray
    dists: np.ndarray
    visited_count: int
    steps: int
    terminated_by: str
    distinct_touched: int = 0
    forgotten: int = 0

    @property
    def hits(self) -> list[tuple[int, float]]:
        return [(int(i), float(d)) for i, d in zip(self.ids, self.dists)]


def stopping_check(d_next: float, d_best_k: float, d_best_1: float, d_nn1_max: float, tau: float) -> bool:
    """True when the closest unvisited candidate lies beyond the slack
    d_best_k + tau * min(d_nn1_max, d_best_1); strict (search.py:45-54).
    The device kernel evaluates the same expression in FP64."""
    return bool(d_next > d_best_k + tau * min(d_nn1_max, d_best_1))


@dataclass
class BatchResult:
    """Array form of a query batch: ids / dists (m, k_out), -1 / inf padded;
    counters (m, 5) = visited, steps, term code, distinct, forgotten.
    distinct_touched is -1 when the batch did not compute it (query_arrays
    without distinct=True); batch_query / query always compute it."""

    ids: np.ndarray
    dists: np.ndarray
    counters: np.ndarray

    def results(self) -> list[QueryResult]:
        """Per-query QueryResult objects; their id / distance arrays are views
        of this batch's (private) host arrays, one row each."""
        k = self.ids.shape[1] if self.ids.ndim == 2 else 0
        nh = (self.ids >= 0).sum(axis=1)
        ir, dr = list(self.ids), list(self.dists)  # full-row views (C-level), trimmed below where short
        for i in np.nonzero(nh < k)[0].tolist():
            ir[i] = ir[i][:nh[i]]
            dr[i] = dr[i][:nh[i]]
        cnt = self.counters.tolist()
        term = TERMINATED_BY
        # thousands of small objects: the cyclic collector would run several
        # times during the list build and find nothing to collect
        gc_on = gc.isenabled()
        gc.disable()
        try:
            return [QueryResult(ir[i], dr[i], c[0], c[1], term[c[2]], c[3], c[4]) for i, c in enumerate(cnt)]
        finally:
            if gc_on:
                gc.enable()


def _params(cfg: QueryConfig, flags: int):
    return N.search_params(cfg.k_out, cfg.prioq_size, cfg.visited_size, cfg.tau, cfg.max_iterations, flags)


def _flags(dv: DeviceVectors, distinct: bool) -> int:
    """FLAG_EXACT_DISTS always: whenever a search's keys are FP64 (a float
    table, or float queries on a uint8 table) the returned hits are re-scored
    with the reference's sequential _sqdist and re-sorted; the kernel ignores
    the flag for uint8 queries on a uint8 table, whose keys are exact."""
    return N.FLAG_EXACT_DISTS | (N.FLAG_DISTINCT if distinct else 0)


def _qflags(dh, distinct: bool) -> int:
    """Flags of a query-kernel launch on dh's bottom layer: _flags plus
    GGNN_FLAG_UNIQUE_ROWS when no adjacency row repeats a neighbour (checked
    once per device hierarchy; the kernel then skips its duplicate filter)."""
    u = getattr(dh, "_unique0", None)
    if u is None:
        L = dh.layers[0]
        res = N.empty((1,), N.torch().int32)
        N.call("ggnn_rows_unique", N.ptr(L.adj), L.node_count, L.k, N.ptr(res), N.stream_ptr())
        u = dh._unique0 = bool(int(res.item()))
    return _flags(dh.vectors, distinct) | (N.FLAG_UNIQUE_ROWS if u else 0)


def _workspace(m, params, max_seeds):
    nbytes = N.load().ggnn_search_workspace_bytes(m, N.ctypes.byref(params), max_seeds)
    if not nbytes:
        return None, 0
    return N.empty((nbytes,), N.torch().uint8), nbytes


def _check_query(h, q: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.float32)
    if q.ndim != 1 or (h.dim and q.shape[0] != h.dim):
        raise ValueError(f"query shape {q.shape} does not match index dimension {h.dim}")
    return q


class _Staging:
    """Reusable device / pinned host buffers of the host-to-host query path
    (one per device): the query batch is uploaded once as float32, narrowed
    to uint8 on the device when every value is an integer in [0, 255]
    (ggnn_f32_to_u8), and the results come back through pinned buffers -- no
    per-call allocations, one synchronisation."""

    def __init__(self):
        self.m = self.d = self.k = 0

    def ensure(self, m: int, d: int, k: int):
        if m <= self.m and d == self.d and k == self.k:
            return self
        t = N.torch()
        m = max(m, self.m if (d == self.d and k == self.k) else 0)
        self.m, self.d, self.k = m, d, k
        self.ids_pin = t.empty((m, k), dtype=t.int32, pin_memory=True)
        self.dists_pin = t.empty((m, k), dtype=t.float64, pin_memory=True)
        self.cnt_pin = t.empty((m, 5), dtype=t.int32, pin_memory=True)
        self.flag_pin = t.empty((1,), dtype=t.int32, pin_memory=True)
        self.q_f32 = N.empty((m, d), t.float32)
        self.q_u8 = N.empty((m, d), t.uint8)
        self.ids = N.empty((m, k), t.int32)
        self.dists = N.empty((m, k), t.float64)
        self.cnt = N.empty((m, 5), t.int32)
        self.flag = N.empty((1,), t.int32)
        # staged path: per-chunk arrival flags (epoch-stamped, never reset)
        self.chunk_flags = t.zeros((_STAGED_MAX_CHUNKS,), dtype=t.int32, device=N.device())
        self.epoch = 0
        self.epoch_pin = t.zeros((1,), dtype=t.int32, pin_memory=True)
        self.status = N.empty((1,), t.int32)
        self.status_pin = t.empty((1,), dtype=t.int32, pin_memory=True)
        # host-side views / device pointers of the fixed buffers, made once:
        # the staged call's prelude delays the first kernel of every batch
        self.epoch_np = self.epoch_pin.numpy()
        self.status_np = self.status_pin.numpy()
        self.ptrs = tuple(N.ptr(x) for x in (self.q_f32, self.chunk_flags, self.epoch_pin, self.ids, self.dists,
                                            self.cnt, self.status, self.status_pin))
        self.spare = None  # result arrays for the next call, allocated while a search runs
        return self

    def results(self, m: int, k: int):
        """Fresh page-locked result arrays (ids, dists, counters) for a call of
        m queries: the spare set made during the previous call when it fits."""
        t = N.torch()
        sp, self.spare = self.spare, None
        if sp is not None and sp[0].shape == (m, k):
            return sp
        return (t.empty((m, k), dtype=t.int32, pin_memory=True), t.empty((m, k), dtype=t.float64, pin_memory=True),
                t.empty((m, 5), dtype=t.int32, pin_memory=True))

    def prepare_spare(self, m: int, k: int):
        t = N.torch()
        self.spare = (t.empty((m, k), dtype=t.int32, pin_memory=True),
                      t.empty((m, k), dtype=t.float64, pin_memory=True),
                      t.empty((m, 5), dtype=t.int32, pin_memory=True))


_STAGING: dict = {}


# host-to-host batches are cut into this many chunks, alternating over two
# streams: chunk i+1's host copy and upload overlap chunk i's search, and
# chunk i's results come back while later chunks still search
_CHUNKS = int(__import__("os").environ.get("GGNN_E2E_CHUNKS", "2"))
# share of the batch in the first chunk (the only upload not hidden behind a search)
_FIRST = float(__import__("os").environ.get("GGNN_E2E_FIRST", "0.5"))
# staged path: ONE search launch over the whole batch while the copy stream
# uploads it chunk by chunk (a warp waits for its chunk's flag), so the batch
# has one drain instead of one per chunk launch
_STAGED = __import__("os").environ.get("GGNN_E2E_STAGED", "1") != "0"
_STAGED_CHUNKS = int(__import__("os").environ.get("GGNN_E2E_STAGED_CHUNKS", "8"))
_STAGED_MAX_CHUNKS = 64
_STREAMS: dict = {}


def _query_host_staged(dh, Q: np.ndarray, cfg: QueryConfig):
    """Host arrays in, host arrays out, the upload overlapped with ONE search
    launch (ggnn_query_batch_staged).  Returns None when the kernel reports a
    non-integral query on a uint8 table or a chunk that never arrived (the
    caller then takes the chunked path)."""
    t = N.torch()
    dv = dh.vectors
    m, d = Q.shape
    k = cfg.k_out
    dev = t.cuda.current_device()
    st = _STAGING.setdefault(dev, _Staging()).ensure(m, d, k)
    streams = _STREAMS.get(dev)
    if streams is None:
        streams = _STREAMS[dev] = (t.cuda.Stream(), t.cuda.Stream())
    main = t.cuda.current_stream()
    search_s, copy_s = streams
    nchunks = max(1, min(_STAGED_CHUNKS, _STAGED_MAX_CHUNKS, m // 256))
    st.epoch = (st.epoch % 0x7FFFFFFF) + 1
    st.epoch_np[0] = st.epoch  # no copy of the previous call is pending (it synchronised)
    params = _params(cfg, _qflags(dh, False))
    narrow = 1 if dv.exact_integers else 0
    # results land straight in fresh page-locked arrays that the caller keeps
    # (torch's caching host allocator makes these allocations cheap; the block
    # returns to its cache when the arrays die): no host-side copy out.  The
    # next call's set is allocated while this call's search runs.
    ids_h, dists_h, cnt_h = st.results(m, k)
    for s_ in streams:
        s_.wait_stream(main)
    q_f32, flags, epoch_pin, ids_d, dists_d, cnt_d, status_d, status_pin = st.ptrs
    N.call("ggnn_query_batch_host", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
           N.ptr(dh.top_rows), dh.ntop, N.P(Q.ctypes.data), m, N.ctypes.byref(params), dh.d_nn1_max,
           q_f32, flags, epoch_pin, nchunks, narrow, ids_d, dists_d, cnt_d, status_d, N.ptr(ids_h),
           N.ptr(dists_h), N.ptr(cnt_h), status_pin, N.P(search_s.cuda_stream), N.P(copy_s.cuda_stream))
    st.prepare_spare(m, k)
    for s_ in streams:
        main.wait_stream(s_)
    search_s.synchronize()
    copy_s.synchronize()
    if int(st.status_np[0]) != 0:
        return None
    return BatchResult(ids_h.numpy(), dists_h.numpy(), cnt_h.numpy())


# The staging buffers and stream pair of a device are shared by every call on
# that device: host threads calling query_arrays concurrently take turns
# (their searches would share the GPU anyway).
_HOST_LOCK = threading.Lock()


def _query_host_fast(dh, Q: np.ndarray, cfg: QueryConfig, distinct: bool = False) -> BatchResult:
    with _HOST_LOCK:
        return _query_host_fast_locked(dh, Q, cfg, distinct)


def _query_host_fast_locked(dh, Q: np.ndarray, cfg: QueryConfig, distinct: bool = False) -> BatchResult:
    t = N.torch()
    # staged: uint8 tables, and float tables whose query rows are page-locked
    # (read in place by the search, zero copy; uploading float rows in flagged
    # chunks measured slower than the chunked path on gist1m); no
    # distinct_touched logs
    if _STAGED and not distinct and Q.shape[0] >= 1024 and (
            dh.vectors.exact_integers or t.from_numpy(Q).is_pinned()):
        r = _query_host_staged(dh, Q, cfg)
        if r is not None:
            return r
    dv = dh.vectors
    m, d = Q.shape
    k = cfg.k_out
    dev = t.cuda.current_device()
    st = _STAGING.setdefault(dev, _Staging()).ensure(m, d, k)
    streams = _STREAMS.get(dev)
    if streams is None:
        streams = _STREAMS[dev] = (t.cuda.Stream(), t.cuda.Stream())
    main = t.cuda.current_stream()
    params = _params(cfg, _qflags(dh, distinct))
    nchunks = max(1, min(_CHUNKS, m // 1024))
    if nchunks > 1:
        first = max(1, min(m - 1, int(m * _FIRST)))
        bounds = [0] + [first + (m - first) * i // (nchunks - 1) for i in range(nchunks)]
    else:
        bounds = [0, m]
    narrow = dv.exact_integers
    if narrow:
        st.flag.fill_(1)
    for s in streams:
        s.wait_stream(main)
    for c in range(nchunks):
        lo, hi = bounds[c], bounds[c + 1]
        s = streams[c & 1]
        with t.cuda.stream(s):
            sp = N.P(s.cuda_stream)
            # straight from the caller's (pageable) array: the driver's staged
            # copy beats a host copy into pinned memory plus a DMA (0.31 vs
            # 0.41 ms for 10k x 128 float32, tools/hostreg_probe.py)
            st.q_f32[lo:hi].copy_(t.from_numpy(Q[lo:hi]), non_blocking=True)
            if narrow:  # uint8 queries when every value is an integer in [0, 255]
                N.call("ggnn_f32_to_u8", N.ptr(st.q_f32[lo:hi]), (hi - lo) * d, N.ptr(st.q_u8[lo:hi]),
                       N.ptr(st.flag), sp)
                qs = N.queries_struct(data=st.q_u8[lo:hi], dtype_code=N.GGNN_U8, m=hi - lo)
            else:
                qs = N.queries_struct(data=st.q_f32[lo:hi], dtype_code=N.GGNN_F32, m=hi - lo)
            ws, wsb = _workspace(hi - lo, params, cfg.k_out)  # distinct_touched logs (or none)
            N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
                   N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max,
                   N.ptr(st.ids[lo:hi]), N.ptr(st.dists[lo:hi]), N.ptr(st.cnt[lo:hi]), N.ptr(ws), wsb, sp)
            st.ids_pin[lo:hi].copy_(st.ids[lo:hi], non_blocking=True)
            st.dists_pin[lo:hi].copy_(st.dists[lo:hi], non_blocking=True)
            st.cnt_pin[lo:hi].copy_(st.cnt[lo:hi], non_blocking=True)
    if narrow:
        with t.cuda.stream(streams[(nchunks - 1) & 1]):
            streams[(nchunks - 1) & 1].wait_stream(streams[nchunks & 1])
            st.flag_pin.copy_(st.flag, non_blocking=True)
    for s in streams:
        main.wait_stream(s)
    main.synchronize()
    if narrow and int(st.flag_pin[0]) != 1:
        # some query is not integral: the uint8 searches above are void; search
        # the float batch (already on the device) against the uint8 table
        qs = N.queries_struct(data=st.q_f32, dtype_code=N.GGNN_F32, m=m)
        ws, wsb = _workspace(m, params, cfg.k_out)
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max,
               N.ptr(st.ids), N.ptr(st.dists), N.ptr(st.cnt), N.ptr(ws), wsb, N.stream_ptr())
        st.ids_pin[:m].copy_(st.ids[:m], non_blocking=True)
        st.dists_pin[:m].copy_(st.dists[:m], non_blocking=True)
        st.cnt_pin[:m].copy_(st.cnt[:m], non_blocking=True)
        main.synchronize()
    return BatchResult(st.ids_pin[:m].numpy().copy(), st.dists_pin[:m].numpy().copy(),
                       st.cnt_pin[:m].numpy().copy())


def query_arrays(h, queries: np.ndarray, cfg: QueryConfig | None = None, distinct: bool = False,
                 out: str = "numpy", _exact: bool = False):
    """Batched query(): top-layer scan + best-first search on layer 0 for every
    row of `queries` in one launch.  Returns a BatchResult (host arrays) or,
    with out="device", the device tensors (ids, dists, counters).
    distinct=True also computes distinct_touched (counter column 3; -1
    otherwise)."""
    cfg = cfg or QueryConfig()
    dh = device_hierarchy(h)
    dv = dh.vectors
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    if Q.ndim == 1:
        Q = Q[None, :]
    if Q.shape[1] != dv.d:
        raise ValueError(f"query dimension {Q.shape[1]} does not match index dimension {dv.d}")
    if out == "numpy" and Q.shape[0] > 0:
        res = _query_host_fast(dh, Q, cfg, distinct)
        redo = np.nonzero(res.counters[:, 3] < 0)[0] if distinct else ()
        for lo in range(0, len(redo), _DISTINCT_CHUNK):  # compact logs that overflowed: exact reruns
            sel = redo[lo:lo + _DISTINCT_CHUNK]
            sub = query_arrays(h, Q[sel], cfg, distinct=True, out="device", _exact=True)
            res.ids[sel], res.dists[sel], res.counters[sel] = (x.cpu().numpy() for x in sub)
        return res
    m = Q.shape[0]
    t = N.torch()
    ids = N.empty((m, cfg.k_out), t.int32)
    dists = N.empty((m, cfg.k_out), t.float64)
    cnt = N.empty((m, 5), t.int32)
    params = _params(cfg, _qflags(dh, distinct))
    dq, qs = dv.queries(Q)
    bottom = dh.layers[0]

    def launch(rows_lo, rows_hi, sub_q, out_ids, out_d, out_c, exact):
        ws, wsb = _workspace(rows_hi - rows_lo, params, -1 if exact else cfg.k_out)
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(bottom.struct), N.ptr(dh.top_rows),
               dh.ntop, N.ctypes.byref(sub_q), N.ctypes.byref(params), dh.d_nn1_max, out_ids, out_d, out_c,
               N.ptr(ws), wsb, N.stream_ptr())

    launch(0, m, qs, N.ptr(ids), N.ptr(dists), N.ptr(cnt), _exact)
    if distinct and m and not _exact:
        # queries whose compact distinct-set overflowed (distinct_touched = -1)
        # run again with exact per-query tables, a few at a time
        redo = np.nonzero(cnt[:, 3].cpu().numpy() < 0)[0]
        for lo in range(0, len(redo), _DISTINCT_CHUNK):
            sel = redo[lo:lo + _DISTINCT_CHUNK]
            sel_d = N.to_dev(sel.astype(np.int64))
            dq2 = dq[sel_d].contiguous()
            sub = N.Queries(N.ptr(dq2), None, len(sel), qs.dtype, 0)
            i2, d2, c2 = N.empty((len(sel), cfg.k_out), t.int32), N.empty((len(sel), cfg.k_out), t.float64), \
                N.empty((len(sel), 5), t.int32)
            launch(0, len(sel), sub, N.ptr(i2), N.ptr(d2), N.ptr(c2), True)
            ids[sel_d], dists[sel_d], cnt[sel_d] = i2, d2, c2
    if out == "device":
        return ids, dists, cnt
    return BatchResult(ids.cpu().numpy(), dists.cpu().numpy(), cnt.cpu().numpy())


def launch_query(h, queries: np.ndarray, cfg: QueryConfig, ids_p, dists_p, cnt_p, uploaded: dict | None = None) -> None:
    """One ggnn_query_batch launch of every row of `queries` on hierarchy h,
    writing into caller-owned device memory (ids int32 / dists f64 (m, k_out),
    counters int32 (m, 5)); distinct_touched is not computed.  `uploaded`
    (a dict the caller keeps) caches the device copy of `queries` per table
    dtype, so a batch searched on several shards is uploaded once."""
    dh = device_hierarchy(h)
    dv = dh.vectors
    key = (dv.dtype, dv.d)
    hit = uploaded.get(key) if uploaded is not None else None
    if hit is None:
        hit = dv.queries(np.ascontiguousarray(queries, dtype=np.float32))
        if uploaded is not None:
            uploaded[key] = hit
    dq, qs = hit
    params = _params(cfg, _qflags(dh, False))
    N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct), N.ptr(dh.top_rows),
           dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max, ids_p, dists_p, cnt_p, None, 0,
           N.stream_ptr())
    del dq


def query(h, q: np.ndarray, cfg: QueryConfig | None = None) -> QueryResult:
    """Top-to-bottom jump: brute-force the top layer, then search the bottom
    (search.py:115-137)."""
    q = _check_query(h, q)
    return query_arrays(h, q[None, :], cfg, distinct=True).results()[0]


def batch_query(h, queries: np.ndarray, cfg: QueryConfig | None = None, threads: int = 1) -> list[QueryResult]:
    """Independent queries, one GPU launch per batch (search.py:213-226).
    `threads` is accepted for signature compatibility and ignored."""
    queries = np.ascontiguousarray(queries, dtype=np.float32)
    if queries.ndim != 2 or (h.dim and queries.shape[1] != h.dim):
        raise ValueError(f"query shape {queries.shape} does not match index dimension {h.dim}")
    if queries.shape[0] == 0:
        return []
    return query_arrays(h, queries, cfg, distinct=True).results()


def top_layer_seeds(h, q: np.ndarray, k_out: int):
    """Exact top-min(k_out, |top|) of the top layer as dataset ids, plus the
    number of distances spent (search.py:100-112)."""
    from . import backend

    q = np.ascontiguousarray(q, dtype=np.float32)
    top = h.num_layers - 1
    rows = h.rows_for(top)
    local, dists = backend.impl.exhaustive_topk_rows(h.dataset, rows, q, min(k_out, len(rows)))
    return rows[local].astype(np.int32), dists, len(rows)


def greedy_search(X: np.ndarray, to_row: np.ndarray, layer, seed_ids, seed_dists, q: np.ndarray, cfg: QueryConfig,
                  d_nn1_max: float) -> QueryResult:
    """Best-first search on one layer from precomputed seeds
    (search.py:57-97)."""
    from . import backend

    seed_ids = np.asarray(seed_ids, dtype=np.int32)
    seed_dists = np.asarray(seed_dists, dtype=np.float64)
    if seed_ids.size == 0:
        raise ValueError("greedy search needs at least one seed")
    if seed_ids.min() < 0 or seed_ids.max() >= layer.node_count:
        raise ValueError("seed id out of range for this layer")
    q = np.ascontiguousarray(q, dtype=np.float32)
    ids, dists, visited, steps, term, distinct, forgotten = backend.impl.greedy_search(
        X, to_row, layer.adjacency, layer.k_nn, layer.sym_count, q, seed_ids, seed_dists, cfg.k_out, cfg.tau,
        d_nn1_max, cfg.max_iterations, cfg.prioq_size, cfg.visited_size)
    return QueryResult(ids, dists, visited, steps, TERMINATED_BY[term], distinct, forgotten)


def hierarchical_query(h, q: np.ndarray, cfg: QueryConfig | None = None, start_layer: int | None = None,
                       stop_layer: int = 0, segment: tuple[int, int] | None = None,
                       slack_bounds: list[float] | None = None, segment_cache: dict | None = None) -> QueryResult:
    """Layer-by-layer descent (search.py:140-210): brute-force the start
    layer (or one segment of it), then seed each finer layer's greedy search
    with the previous layer's k_out hits.  `segment_cache` is accepted for
    signature compatibility; the device keeps everything resident."""
    cfg = cfg or QueryConfig()
    q = _check_query(h, q)
    start = h.num_layers - 1 if start_layer is None else start_layer
    if not (0 <= stop_layer <= start < h.num_layers):
        raise ValueError(f"invalid layer range {start}..{stop_layer} for {h.num_layers} layers")
    lo, hi = segment if segment is not None else (0, h.layers[start].node_count)
    res = descent_arrays(h, q[None, :], cfg, start, stop_layer, np.array([lo], dtype=np.int32),
                         np.array([hi], dtype=np.int32), slack_bounds, distinct=True)
    return res.results()[0]


def descent_arrays(h, queries, cfg: QueryConfig, start: int, stop: int, seg_lo=None, seg_hi=None,
                   slack_bounds=None, distinct: bool = False, query_rows=None) -> BatchResult:
    """Batched hierarchical_query.  With `query_rows` (device int32) the
    queries are dataset rows (construction-time self queries)."""
    dh = device_hierarchy(h)
    dv = dh.vectors
    t = N.torch()
    layers = dh.layer_array()
    for j in range(dh.num_layers):
        if slack_bounds is not None:
            layers[j].slack = float(slack_bounds[j])
        elif j == 0:
            layers[j].slack = float(dh.d_nn1_max)
    if query_rows is not None:
        m = int(query_rows.shape[0])
        qs = N.queries_struct(rows=query_rows, dtype_code=dv.dtype)
        keep = query_rows
    else:
        keep, qs = dv.queries(np.ascontiguousarray(queries, dtype=np.float32))
        m = qs.m
    lo_d = N.to_dev(np.asarray(seg_lo, dtype=np.int32)) if seg_lo is not None else None
    hi_d = N.to_dev(np.asarray(seg_hi, dtype=np.int32)) if seg_hi is not None else None
    ids = N.empty((m, cfg.k_out), t.int32)
    dists = N.empty((m, cfg.k_out), t.float64)
    cnt = N.empty((m, 5), t.int32)
    params = _params(cfg, _flags(dv, distinct))
    for exact in (False, True):
        ws, wsb = _workspace(m, params, -1 if exact else cfg.k_out)
        N.call("ggnn_descent_batch", N.ctypes.byref(dv.struct), layers, dh.num_layers, start, stop,
               N.ctypes.byref(qs), N.ptr(lo_d), N.ptr(hi_d), N.ctypes.byref(params), N.ptr(ids), N.ptr(dists),
               N.ptr(cnt), N.ptr(ws), wsb, N.stream_ptr())
        if not distinct or not bool((cnt[:, 3] < 0).any()):
            break  # (a compact distinct-set overflowed: rerun with exact tables)
    del keep
    return BatchResult(ids.cpu().numpy(), dists.cpu().numpy(), cnt.cpu().numpy())


def exact_knn_rows(dataset, rows: np.ndarray, k: int):
    """Exact top-k of dataset rows `rows` against the whole dataset, ties by
    ascending id, in one ggnn_exhaustive_topk launch (k <= 32; up to 128 on
    the tensor-core path for uint8 tables)."""
    dv = DeviceVectors.of(dataset)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    t = N.torch()
    rd = N.to_dev(rows)
    qs = N.queries_struct(rows=rd, dtype_code=dv.dtype)
    ids = N.empty((len(rows), k), t.int32)
    dists = N.empty((len(rows), k), t.float64)
    N.call("ggnn_exhaustive_topk", N.ctypes.byref(dv.struct), None, dv.n, N.ctypes.byref(qs), int(k), N.ptr(ids),
           N.ptr(dists), N.stream_ptr())
    ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
    N.check_tc_timeouts("bf")
    return ids, dists


def exact_knn(dataset, queries: np.ndarray, k: int):
    """Exact top-k of external queries against the whole dataset, ties by
    ascending id (ground truth for recall), one launch (k limits as
    exact_knn_rows)."""
    dv = DeviceVectors.of(dataset)
    dq, qs = dv.queries(np.ascontiguousarray(queries, dtype=np.float32))
    t = N.torch()
    m = qs.m
    ids = N.empty((m, k), t.int32)
    dists = N.empty((m, k), t.float64)
    N.call("ggnn_exhaustive_topk", N.ctypes.byref(dv.struct), None, dv.n, N.ctypes.byref(qs), int(k), N.ptr(ids),
           N.ptr(dists), N.stream_ptr())
    ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
    N.check_tc_timeouts("bf")
    return ids, dists
