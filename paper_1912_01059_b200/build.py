"""Bottom-up hierarchical graph construction on the GPU (drop-in for graphann.build).

Control flow and RNG consumption follow /root/reference/pkg/src/graphann/build.py:
the seeded permutation and the per-child selection keys are drawn on the host
with numpy (so a GPU build partitions and samples exactly like the reference),
and every data-parallel phase runs as one batched kernel over all nodes:

  leaf kNN per bottom batch / coarse segment   ggnn_leaf_knn
  merge: descent from the top segment          ggnn_descent_batch (query rows = the nodes)
         + union into direct slots              ggnn_merge_rows
  symmetrize: reachability checks              ggnn_sym_check_batch
              + deterministic inverse-slot claims  ggnn_sym_claim_*
  statistics                                   ggnn_layer_stats

The reference mutates rows in place while later nodes of the same pass query
them (Gauss-Seidel); the GPU pass reads a snapshot and applies all updates
afterwards (Jacobi), and inverse-slot claims are resolved per destination in
(x, slot) priority order.  Graphs are therefore deterministic for a fixed seed
but statistically (not bitwise) equal to the reference's.
"""

from __future__ import annotations

import numpy as np

SYM_CHECK_BUDGET = 16  # expansions allowed per reachability check (build.py:31)
SYM_CHECK_PRIOQ = 64
SYM_CHECK_VISITED = 128
SYM_FALLBACK = 8
MAX_SLOTS = 32  # adjacency slots per node the kernels handle (ggnn_common.cuh MAX_K)
CLAIM_CHECK = int(__import__("os").environ.get("GGNN_CLAIM_CHECK", "4"))  # claim rounds per pending read-back
CLAIM_COMPACT = __import__("os").environ.get("GGNN_CLAIM_COMPACT", "1") != "0"  # rounds over the open requests only
# node windows per symmetrize pass: requests of x-window w are re-checked after the
# claims of windows < w, approximating the reference's sequential x order
# Node windows per symmetrize / merge pass: the reference walks the nodes of a
# pass in order and every node sees the links earlier nodes created; windows
# approximate that order (later windows see earlier windows' updates).  Small
# layers take fine windows (cheap, and where single links matter most:
# tests/golden/deep3k); large layers 16 (each window still fills the GPU).
SMALL_LAYER = int(__import__("os").environ.get("GGNN_SMALL_LAYER", "200000"))
_ENV = __import__("os").environ


def _sym_windows(nc: int) -> int:
    return int(_ENV.get("GGNN_SYM_WINDOWS", 128 if nc <= SMALL_LAYER else 16))


def _merge_windows(nc: int) -> int:
    return int(_ENV.get("GGNN_MERGE_WINDOWS", 64 if nc <= SMALL_LAYER else 16))
CONSENSUS_SAMPLE = 256
CONSENSUS_K = 10

# per-symmetrize-pass records when GGNN_TRACE is set (diagnostics)
TRACE = [] if __import__("os").environ.get("GGNN_TRACE") else None


def plan_geometry(n: int, s: int, g: int) -> tuple[int, int]:
    """Deepest tree with s * g**(l-1) <= n: returns (l, b = g**(l-1))
    (build.py:54-64)."""
    t = 0
    while s * g ** (t + 1) <= n:
        t += 1
    return t + 1, g**t


def partition_bottom(n: int, b: int, rng: np.random.Generator) -> tuple[np.ndarray, np.ndarray]:
    """Seeded shuffle cut into b contiguous batches of ceil/floor(n/b)
    (build.py:67-75): batch i = perm[offsets[i]:offsets[i+1]]."""
    perm = rng.permutation(n).astype(np.int32)
    base, rem = divmod(n, b)
    sizes = np.full(b, base, dtype=np.int64)
    sizes[:rem] += 1
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return perm, offsets


def select_points(weights: np.ndarray, count: int, rng: np.random.Generator) -> tuple[np.ndarray, bool]:
    """Weighted sampling without replacement with exponential keys log(u)/w,
    the `count` largest keys win; all-zero weights fall back to uniform
    (build.py:97-121)."""
    weights = np.asarray(weights, dtype=np.float64)
    m = len(weights)
    if count > m:
        raise ValueError(f"cannot select {count} from {m} nodes")
    u = rng.random(m)
    uniform = not (weights > 0).any()
    if uniform:
        keys = u
    else:
        with np.errstate(divide="ignore"):
            keys = np.log(u) / weights
    if count == m:
        return np.arange(m, dtype=np.int64), uniform
    chosen = np.argsort(-keys, kind="stable")[:count]
    return np.sort(chosen), uniform


def select_segments(weights: np.ndarray, seg_offsets: np.ndarray, quotas: np.ndarray,
                    rng: np.random.Generator) -> np.ndarray:
    """Vectorised select_points over consecutive segments: identical output
    to calling select_points(weights[lo:hi], quota, rng) segment by segment
    (one rng.random(total) draw equals the per-segment draws concatenated).
    Returns the chosen positions (into `weights`), ascending per segment.
    Segments are laid out as rows of a padded matrix and sorted row-wise
    (stable, descending key: ties keep position order, like the reference's
    stable argsort, _purepy.py:42 / build.py:120)."""
    weights = np.asarray(weights, dtype=np.float64)
    total = len(weights)
    u = rng.random(total)
    seg_offsets = np.asarray(seg_offsets, dtype=np.int64)
    nseg = len(seg_offsets) - 1
    if nseg <= 0 or total == 0:
        return np.zeros(0, dtype=np.int64)
    sizes = np.diff(seg_offsets)
    starts = seg_offsets[:-1]
    seg_id = np.repeat(np.arange(nseg), sizes)
    nz = sizes > 0
    any_pos = np.zeros(nseg, dtype=bool)
    any_pos[nz] = np.maximum.reduceat((weights > 0).astype(np.int8), starts[nz]) > 0
    with np.errstate(divide="ignore", invalid="ignore"):
        keys = np.where(any_pos[seg_id], np.log(u) / weights, u)
    width = int(sizes.max())
    pad = np.full((nseg, width), np.inf)  # padding sorts after every real key (stable)
    pad[seg_id, np.arange(total) - starts[seg_id]] = -keys
    order = np.argsort(pad, axis=1, kind="stable")
    take = np.arange(width)[None, :] < np.minimum(np.asarray(quotas, dtype=np.int64), sizes)[:, None]
    rows, cols = np.nonzero(take)
    chosen = starts[rows] + order[rows, cols]
    return chosen[np.lexsort((chosen, rows))]


def _segment_of(h, layer_index: int, node: int) -> int:
    if layer_index == 0:
        return int(h.bottom_segment_of[node])
    return node // h.s


def _worker_ranges(total: int, threads: int) -> list[tuple[int, int]]:
    threads = max(1, min(threads, total))
    step = (total + threads - 1) // threads
    return [(i, min(i + step, total)) for i in range(0, total, step)]


# =============================================================== GPU passes
import time  # noqa: E402
from dataclasses import dataclass, field  # noqa: E402

from . import _native as N  # noqa: E402
from . import _devgraph as G  # noqa: E402
from .config import BuildConfig, QueryConfig  # noqa: E402
from .data import ConfigError, Dataset  # noqa: E402
from .device import DeviceVectors  # noqa: E402
from .graph import SENTINEL, AdjacencyLayer, GraphStats, Hierarchy  # noqa: E402


@dataclass
class BuildStats:
    """Construction diagnostics (build.py:39-51)."""

    phase_seconds: dict[str, float] = field(default_factory=dict)
    mean_sym_used: float = 0.0
    sym_used_per_layer: list[float] = field(default_factory=list)
    d_nn1_trajectory: list[tuple[float, float]] = field(default_factory=list)
    consensus_trajectory: list[tuple[str, float]] = field(default_factory=list)
    reduced_knn_batches: int = 0
    dropped_sym_links: int = 0
    build_seconds: float = 0.0
    threads: int = 1
    # build accounting (build(..., accounting=True)): per phase, the searches'
    # visited / steps totals (ggnn_search_accounting) and the leaf kNN's
    # multiply-adds (sum over batches of m_b^2 * d)
    search_visited: dict[str, int] = field(default_factory=dict)
    search_steps: dict[str, int] = field(default_factory=dict)
    leaf_macs: int = 0

    def accounting_summary(self, d: int, e: int, k: int = 24) -> dict | None:
        """Algorithmic bytes per phase, V * d * e + T * (4k + 4) summed over
        the phase's searches (SURVEY.md 8d "Build accounting"), and the
        bytes / second each phase reached."""
        if not self.search_visited:
            return None
        per = {}
        for key, v in self.search_visited.items():
            b = v * d * e + self.search_steps.get(key, 0) * (4 * k + 4)
            sec = self.phase_seconds.get(key, 0.0)
            per[key] = {"bytes": b, "GB_per_s": b / sec / 1e9 if sec > 0 else None}
        total = sum(p["bytes"] for p in per.values())
        t_search = sum(self.phase_seconds.get(key, 0.0) for key in per)
        top = dict(sorted(per.items(), key=lambda kv: -kv[1]["bytes"])[:6])
        return {"search_bytes_total": total, "search_seconds": t_search,
                "search_GB_per_s": total / t_search / 1e9 if t_search else None,
                "visited_total": int(sum(self.search_visited.values())),
                "steps_total": int(sum(self.search_steps.values())),
                "leaf_knn_flops": 2 * self.leaf_macs, "top_phases": top}


def _merge_query_config(cfg: BuildConfig) -> QueryConfig:
    """Descent knobs of merge_layer (build.py:124-131)."""
    return QueryConfig(k_out=cfg.k, tau=cfg.tau_build, max_iterations=400, prioq_size=max(256, 2 * cfg.k),
                       visited_size=512)


def _sync():
    N.torch().cuda.synchronize()


def _leaf_layer(h, j: int, nodes: np.ndarray, offsets: np.ndarray) -> int:
    """Exact kNN inside every batch / segment of layer j (build_base over
    all batches in one launch).  Returns the number of reduced batches."""
    layer = h.layers[j]
    dev = layer._dev
    ws = G.workspace(h)
    dv = DeviceVectors.of(h.dataset)
    nodes_d = N.to_dev(np.asarray(nodes, dtype=np.int32))
    offs_d = N.to_dev(np.asarray(offsets, dtype=np.int64))
    nb = len(offsets) - 1
    max_batch = int(np.diff(offsets).max()) if nb else 0
    ws.reduced.zero_()
    N.call("ggnn_leaf_knn", N.ctypes.byref(dv.struct), N.ptr(nodes_d), N.ptr(dev.get("to_row")), N.ptr(offs_d), nb,
           max_batch, layer.k_nn, None, None, N.ptr(dev["adj"]), layer.k, N.ptr(dev["nnd"]), N.ptr(dev["dnn1"]),
           N.ptr(ws.reduced), N.stream_ptr())
    layer._version += 1
    reduced = int(ws.reduced.item())
    N.check_tc_timeouts("leaf")
    return reduced


def _seg_of0(h):
    cached = getattr(h, "_gpu_seg_of0", None)
    if cached is None or cached.numel() != h.n:
        cached = N.to_dev(np.asarray(h.bottom_segment_of, dtype=np.int32))
        h._gpu_seg_of0 = cached
    return cached


def _merge_pass(h, j: int):
    """merge_layer on the device: every node of layer j descends from its
    group's segment of the top layer (one launch), then merge_rows applies
    the hits.  Returns the rescued (displaced) neighbours as device arrays."""
    G.ensure_device(h)
    cfg = _merge_query_config(h.config)
    start = h.num_layers - 1
    shift = h.g ** (start - j)
    bounds = [G.live_max(h, L) for L in h.layers]
    structs = G.structs_array([G.layer_struct(L, bounds[i]) for i, L in enumerate(h.layers)])
    layer = h.layers[j]
    dev = layer._dev
    nc = layer.node_count
    dv = DeviceVectors.of(h.dataset)
    flags = N.FLAG_EXACT_DISTS  # (a no-op for exact uint8 keys)
    params = N.search_params(cfg.k_out, cfg.prioq_size, cfg.visited_size, cfg.tau, cfg.max_iterations, flags)
    t = N.torch()
    if j == 0:
        seg_of, seg_div = _seg_of0(h), shift
    else:
        seg_of, seg_div = t.arange(nc, dtype=t.int32, device=N.device()), h.s * shift
    ids = N.empty((nc, cfg.k_out), t.int32)
    dists = N.empty((nc, cfg.k_out), t.float64)
    resc_id = N.empty((nc, layer.k_nn), t.int32)
    resc_d = N.empty((nc, layer.k_nn), t.float64)
    # The reference merges node after node in place, so later descents walk
    # the links earlier nodes just gained (build.py:173-188).  A single
    # snapshot pass loses that: on strongly clustered data it measurably
    # weakens cross-cluster navigation (reference with a snapshot merge:
    # R@10 0.93 vs 0.98 on tests/golden/deep3k).  Descents therefore run in
    # consecutive node windows (_merge_windows), each applied before the next
    # descends.
    windows = max(1, min(_merge_windows(nc), nc))
    for w in range(windows):
        lo, hi = nc * w // windows, nc * (w + 1) // windows
        if hi <= lo:
            continue
        cnt = hi - lo
        N.call("ggnn_merge_descent", N.ctypes.byref(dv.struct), structs, h.num_layers, start, j,
               N.ptr(dev["rows_q"][lo:hi]), cnt, N.ptr(seg_of[lo:hi]), seg_div, h.s, N.ctypes.byref(params),
               N.ptr(ids[lo:hi]), N.ptr(dists[lo:hi]), None, N.stream_ptr())
        N.call("ggnn_merge_rows_range", lo, cnt, layer.k, layer.k_nn, N.ptr(dev["adj"]), N.ptr(dev["nnd"]),
               N.ptr(dev["symc"]), N.ptr(dev["dnn1"]), N.ptr(ids[lo:hi]), N.ptr(dists[lo:hi]), cfg.k_out,
               N.ptr(resc_id[lo:hi]), N.ptr(resc_d[lo:hi]), None, N.stream_ptr())
    layer._version += 1
    return resc_id, resc_d


def _symmetrize_dev(h, j: int, tau_build: float, resc=None) -> int:
    """symmetrize on the device (build.py:200-266).

    1. one launch checks every (x, z) pair of the layer on the current graph
       and records the verdict-2 pairs as requests (pair-index priority);
    2. claim rounds: every open request proposes to its current target and
       each target accepts the lowest pair index; between rounds the open
       requests are re-checked on the updated graph, so -- as in the
       reference's sequential pass -- a link claimed earlier can make a later
       request unnecessary.  Returns the number of dropped links."""
    G.ensure_device(h)
    layer = h.layers[j]
    dev = layer._dev
    ws = G.workspace(h)
    dv = DeviceVectors.of(h.dataset)
    d_max = G.live_max(h, layer)
    k_out = max(1, layer.k_nn)
    prioq = max(SYM_CHECK_PRIOQ, 2 * k_out)
    resc_id, resc_d = resc if resc is not None else (None, None)
    per_node = layer.k_nn + (int(resc_id.shape[1]) if resc_id is not None else 0)
    ws.ensure_requests(max(4096, layer.node_count * per_node // 16), SYM_FALLBACK)
    lstruct = G.layer_struct(layer, d_max)
    if TRACE is not None:
        _sync()
        t_check = time.perf_counter()
    while True:
        ws.req_count.zero_()
        N.call("ggnn_sym_check_layer", N.ctypes.byref(dv.struct), N.ctypes.byref(lstruct), N.ptr(dev["nnd"]),
               N.ptr(resc_id), N.ptr(resc_d), per_node, float(tau_build), d_max, SYM_CHECK_BUDGET, k_out, prioq,
               SYM_CHECK_VISITED, SYM_FALLBACK, N.ptr(ws.req), N.ptr(ws.req_count), ws.req_cap, N.stream_ptr())
        cnt = int(ws.req_count.item())
        if cnt <= ws.req_cap:
            break
        ws.ensure_requests(2 * cnt, SYM_FALLBACK)  # checks do not mutate the layer: rerun
    dropped = rounds = 0
    if TRACE is not None:
        _sync()
        t_claim = time.perf_counter()
    if cnt:
        ws.stage[:cnt].zero_()
        ws.tgt[:cnt].fill_(-1)
        ws.dropped.zero_()
        nc = layer.node_count
        windows = max(1, min(_sym_windows(nc), cnt))
        # the rounds' item list: all requests at first, then (at every
        # read-back) only those still open -- most settle in the first rounds,
        # and late rounds would otherwise scan every settled request again
        idx, n_items, flip = None, cnt, 0
        while True:
            x_end = nc if rounds >= windows else (nc * (rounds + 1) + windows - 1) // windows
            if rounds:
                N.call("ggnn_sym_recheck", N.ctypes.byref(dv.struct), N.ctypes.byref(lstruct), N.ptr(ws.req),
                       n_items, N.ptr(ws.stage), x_end, float(tau_build), d_max, SYM_CHECK_BUDGET, k_out, prioq,
                       SYM_CHECK_VISITED, SYM_FALLBACK, N.ptr(idx), N.stream_ptr())
            N.call("ggnn_sym_claim_round", N.ptr(ws.req), n_items, SYM_FALLBACK, N.ptr(dev["adj"]),
                   N.ptr(dev["symc"]), layer.k, layer.k_nn, N.ptr(ws.best), N.ptr(ws.stage), N.ptr(ws.tgt),
                   N.ptr(ws.dropped), N.ptr(ws.pending), x_end, N.ptr(ws.first), N.ptr(idx), N.stream_ptr())
            rounds += 1
            # the open-request count is read back (a host sync) only every
            # CLAIM_CHECK rounds: rounds after the last request settled are
            # no-ops (every kernel skips settled requests), so the extra ones
            # cost launches, not results
            if not CLAIM_COMPACT:
                if x_end == nc and (rounds - windows) % CLAIM_CHECK == 0 and int(ws.pending.item()) == 0:
                    break
                continue
            if (rounds - windows) % CLAIM_CHECK == 0 or (rounds < windows and rounds % (2 * CLAIM_CHECK) == 0):
                out = ws.open_idx[flip]
                N.call("ggnn_sym_compact", N.ptr(ws.stage), N.ptr(idx), n_items, N.ptr(out), N.ptr(ws.n_open),
                       N.stream_ptr())
                idx, n_items, flip = out, int(ws.n_open.item()), flip ^ 1
                if x_end == nc and n_items == 0:
                    break
        layer._version += 1
        dropped = int(ws.dropped.item())
    if TRACE is not None:
        _sync()
        t_end = time.perf_counter()
        stage = ws.stage[:cnt].cpu().numpy() if cnt else np.zeros(0)
        TRACE.append({"layer": j, "nodes": layer.node_count, "pairs": layer.node_count * per_node, "requests": cnt,
                      "check_s": t_claim - t_check, "claim_s": t_end - t_claim,
                      "claimed": int((stage == -1).sum()), "resolved": int((stage == -3).sum()), "dropped": dropped,
                      "rounds": rounds, "mean_sym": float(dev["symc"].double().mean().item())})
    return dropped


def _rescued_dict(resc) -> dict[int, list[tuple[int, float]]]:
    ids = resc[0].cpu().numpy()
    ds = resc[1].cpu().numpy()
    out = {}
    for x in np.nonzero(ids[:, 0] >= 0)[0]:
        row = [(int(i), float(d)) for i, d in zip(ids[x], ds[x]) if i >= 0]
        out[int(x)] = row
    return out


def _rescued_arrays(rescued: dict, nc: int):
    width = max((len(v) for v in rescued.values()), default=0)
    if width == 0:
        return None
    ids = np.full((nc, width), -1, dtype=np.int32)
    ds = np.zeros((nc, width), dtype=np.float64)
    for x, lst in rescued.items():
        for t, (z, d) in enumerate(lst):
            ids[x, t] = z
            ds[x, t] = d
    return N.to_dev(ids), N.to_dev(ds)


# ============================================================ reference API
def build_base(layer: AdjacencyLayer, X: np.ndarray, to_row: np.ndarray, members: np.ndarray) -> bool:
    """Exact within-batch kNN lists written into `layer` (build.py:78-94);
    True when the batch was too small to fill all k_nn slots."""
    from . import backend

    members = np.asarray(members, dtype=np.int32)
    k_nn = layer.k_nn
    pos, dists = backend.impl.batch_bruteforce(X, np.asarray(to_row)[members], k_nn)
    k_eff = min(k_nn, len(members) - 1)
    layer.touch()
    if k_eff > 0:
        ids = np.where(pos[:, :k_eff] >= 0, members[pos[:, :k_eff]], SENTINEL)
        layer.adjacency[members, :k_eff] = ids
        layer.nn_dists[members, :k_eff] = dists[:, :k_eff]
        layer.d_nn1[members] = dists[:, 0]
    else:
        layer.d_nn1[members] = np.inf
    return k_eff < k_nn


def merge_layer(h: Hierarchy, layer_index: int, tau_build: float, threads: int = 1):
    """Fuse the partitions of one layer (build.py:146-197): every node
    descends from its group's top segment and merges the hits into its direct
    slots.  Returns {node: [(displaced id, dist), ...]}.  `threads` is ignored."""
    if layer_index == 0 and h.bottom_segment_of is None:
        raise RuntimeError("merge/refine need construction bookkeeping; they apply to freshly built hierarchies, "
                           "not loaded ones")
    return _rescued_dict(_merge_pass(h, layer_index))


def symmetrize(h: Hierarchy, layer_index: int, tau_build: float, rescued=None, threads: int = 1) -> int:
    """Add inverse links where a neighbour cannot reach back (build.py:200-266);
    returns the number of dropped links."""
    G.ensure_device(h)
    resc = _rescued_arrays(rescued, h.layers[layer_index].node_count) if rescued else None
    return _symmetrize_dev(h, layer_index, tau_build, resc)


def refine_layer(h: Hierarchy, layer_index: int, tau_build: float, threads: int = 1) -> int:
    """One more fuse-and-symmetrize round (build.py:269-272)."""
    if layer_index == 0 and h.bottom_segment_of is None:
        raise RuntimeError("merge/refine need construction bookkeeping; they apply to freshly built hierarchies, "
                           "not loaded ones")
    resc = _merge_pass(h, layer_index)
    return _symmetrize_dev(h, layer_index, tau_build, resc)


def compute_stats(h: Hierarchy) -> GraphStats:
    """Mean and max first-neighbour distance over the bottom layer
    (build.py:275-280)."""
    layer = h.layers[0]
    if layer.device_authoritative:
        mx, s, cnt, bad = G.workspace(h).stats(layer._dev["dnn1"])
        if bad:
            raise ValueError("bottom layer has nodes without a first neighbor")
        return GraphStats(s / cnt, mx)
    d = layer.d_nn1
    if not np.isfinite(d).all():
        raise ValueError("bottom layer has nodes without a first neighbor")
    return GraphStats(float(d.mean()), float(d.max()))


def _bottom_d_nn1(h) -> tuple[float, float]:
    mx, s, cnt, _ = G.workspace(h).stats(h.layers[0]._dev["dnn1"])
    if cnt == 0:
        return (float("inf"), float("inf"))
    return (s / cnt, mx)


def _sample_consensus(h, sample: np.ndarray) -> float:
    """Exact-neighbour overlap of the bottom direct slots on sampled nodes."""
    from .search import exact_knn_rows

    layer = h.layers[0]
    k = min(CONSENSUS_K, layer.k_nn, layer.node_count - 1)
    ids, _ = exact_knn_rows(h.dataset, np.asarray(sample, dtype=np.int32), k + 1)
    adj = layer._dev["adj"][N.to_dev(np.asarray(sample, dtype=np.int64))][:, :k].cpu().numpy()
    total = 0.0
    for i, node in enumerate(sample):
        truth = [int(v) for v in ids[i] if int(v) != node][:k]
        mine = set(int(v) for v in adj[i] if v != SENTINEL)
        total += len(set(truth) & mine) / k
    return total / len(sample)


def _select_level(h: Hierarchy, level: int, rng: np.random.Generator) -> np.ndarray:
    """s points per new segment, split over the g child segments, weighted by
    first-neighbour distance (build.py:417-450), vectorised."""
    cfg = h.config
    child = h.layers[level - 1]
    dnn1 = child._dev["dnn1"].cpu().numpy() if child.device_authoritative else child.d_nn1
    if level == 1:
        child_offsets = np.asarray(h.layer_offsets[0], dtype=np.int64)
        child_count = len(child_offsets) - 1
        weights = dnn1[h.bottom_perm]
    else:
        child_count = child.node_count // cfg.s
        child_offsets = np.arange(0, child_count * cfg.s + 1, cfg.s, dtype=np.int64)
        weights = dnn1
    group_count = child_count // cfg.g
    used = group_count * cfg.g
    quota_base, quota_rem = divmod(cfg.s, cfg.g)
    ci = np.arange(used) % cfg.g
    quotas = quota_base + (ci < quota_rem).astype(np.int64)
    offs = child_offsets[: used + 1]
    chosen = select_segments(weights[: offs[-1]], offs, quotas, rng)
    if level == 1:
        return np.asarray(h.bottom_perm, dtype=np.int32)[chosen]
    return chosen.astype(np.int32)


def build(dataset: Dataset, cfg: BuildConfig | None = None, threads: int = 1,
          track_consensus: bool = False, accounting: bool = False) -> tuple[Hierarchy, BuildStats]:
    """Construct the full hierarchy on the GPU (build.py:297-406).
    Deterministic for a fixed (dataset, cfg.seed); `threads` is ignored.
    accounting=True fills BuildStats' per-phase search totals."""
    cfg = cfg or BuildConfig()
    n = dataset.n
    if n < cfg.s:
        raise ConfigError(f"dataset has {n} points but batches need at least s={cfg.s}")
    if cfg.k > MAX_SLOTS:
        # one warp lane per adjacency slot in every search and merge kernel
        raise ConfigError(f"k must be <= {MAX_SLOTS} on the GPU path (got k={cfg.k})")
    rng = np.random.default_rng(cfg.seed)
    consensus_rng = np.random.default_rng((cfg.seed, 0xC0115E15))
    stats = BuildStats(threads=threads)
    _sync()
    t_begin = time.perf_counter()

    l, b = plan_geometry(n, cfg.s, cfg.g)
    perm, offsets = partition_bottom(n, b, rng)
    bottom = AdjacencyLayer.from_device(n, cfg.k, cfg.k_nn, G.new_layer_dev(n, cfg.k, cfg.k_nn))
    h = Hierarchy([bottom], [None], cfg.s, cfg.g, cfg, dim=dataset.d)
    h.attach(dataset)
    batch_of = np.empty(n, dtype=np.int32)
    batch_of[perm] = np.repeat(np.arange(b, dtype=np.int32), np.diff(offsets))
    h.bottom_segment_of = batch_of
    h.bottom_perm = perm
    h.layer_offsets = [offsets]
    G.ensure_device(h)
    sample = None
    if track_consensus:
        sample = consensus_rng.choice(n, size=min(CONSENSUS_SAMPLE, n), replace=False)

    acc = None
    if accounting:
        acc = N.torch().zeros(2, dtype=N.torch().int64, device=N.device())
        N.call("ggnn_search_accounting", N.ptr(acc))

    def timed(key, fn, *args):
        t0 = time.perf_counter()
        out = fn(*args)
        _sync()
        stats.phase_seconds[key] = stats.phase_seconds.get(key, 0.0) + time.perf_counter() - t0
        if acc is not None:
            v, t = (int(x) for x in acc.tolist())
            if v or t:
                stats.search_visited[key] = stats.search_visited.get(key, 0) + v
                stats.search_steps[key] = stats.search_steps.get(key, 0) + t
                acc.zero_()
        return out

    try:
        _build_levels(h, cfg, stats, timed, perm, offsets, l, rng, sample)
    finally:
        if acc is not None:
            N.call("ggnn_search_accounting", None)
    if accounting:
        sizes = np.diff(np.asarray(offsets, dtype=np.int64))
        stats.leaf_macs = int((sizes * sizes).sum()) * dataset.d
        for L in h.layers[1:]:
            stats.leaf_macs += (L.node_count // cfg.s) * cfg.s * cfg.s * dataset.d
    h.stats = compute_stats(h)
    per_layer = [float(L._dev["symc"].double().mean().item()) for L in h.layers]
    stats.sym_used_per_layer = per_layer
    stats.mean_sym_used = per_layer[0]
    _sync()
    stats.build_seconds = time.perf_counter() - t_begin
    from .device import _token

    h._device_cache = (_token(h), G.device_hierarchy_from_build(h))
    return h, stats


def _build_levels(h, cfg, stats, timed, perm, offsets, l, rng, sample):
    """The level loop of build(): leaf kNN + symmetrize of layer 0, then per
    level selection, coarse brute force, merges and refinements."""

    def refine(j):
        return _symmetrize_dev(h, j, cfg.tau_build, _merge_pass(h, j))

    stats.reduced_knn_batches = timed("level0/base", _leaf_layer, h, 0, perm, offsets)
    stats.dropped_sym_links += timed("level0/sym", _symmetrize_dev, h, 0, cfg.tau_build, None)
    stats.d_nn1_trajectory.append(_bottom_d_nn1(h))
    for level in range(1, l):
        selected = timed(f"level{level}/select", _select_level, h, level, rng)
        nc = len(selected)
        layer = AdjacencyLayer.from_device(nc, cfg.k, cfg.k_nn, G.new_layer_dev(nc, cfg.k, cfg.k_nn))
        h.layers.append(layer)
        h.to_bottom.append(h.rows_for(level - 1)[selected].astype(np.int32))
        h.invalidate_caches()
        layer._dev["to_row"] = N.to_dev(h.to_bottom[level])
        layer._dev["down"] = N.to_dev(selected)
        layer._dev["rows_q"] = layer._dev["to_row"]
        seg_offsets = np.arange(0, (nc // cfg.s) * cfg.s + 1, cfg.s, dtype=np.int64)
        stats.reduced_knn_batches += timed(f"level{level}/base", _leaf_layer, h, level,
                                           np.arange(nc, dtype=np.int32), seg_offsets)
        stats.dropped_sym_links += timed(f"level{level}/sym", _symmetrize_dev, h, level, cfg.tau_build, None)
        for j in range(level - 1, -1, -1):
            resc = timed(f"level{level}/merge{j}", _merge_pass, h, j)
            stats.dropped_sym_links += timed(f"level{level}/merge{j}/sym", _symmetrize_dev, h, j, cfg.tau_build,
                                             resc)
            if j == 0 and sample is not None:
                stats.consensus_trajectory.append((f"level{level}/merge", _sample_consensus(h, sample)))
            for r in range(cfg.refinements):
                stats.dropped_sym_links += timed(f"level{level}/refine{j}.{r}", refine, j)
                if j == 0 and sample is not None:
                    stats.consensus_trajectory.append((f"level{level}/refine{r}", _sample_consensus(h, sample)))
        stats.d_nn1_trajectory.append(_bottom_d_nn1(h))
