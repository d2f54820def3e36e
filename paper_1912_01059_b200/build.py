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
CONSENSUS_SAMPLE = 256
CONSENSUS_K = 10


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
    Returns the chosen positions (into `weights`), ascending per segment."""
    weights = np.asarray(weights, dtype=np.float64)
    total = len(weights)
    u = rng.random(total)
    nseg = len(seg_offsets) - 1
    sizes = np.diff(seg_offsets)
    seg_id = np.repeat(np.arange(nseg), sizes)
    pos_pos = weights > 0
    any_pos = np.zeros(nseg, dtype=bool)
    np.logical_or.at(any_pos, seg_id, pos_pos)
    with np.errstate(divide="ignore", invalid="ignore"):
        keys = np.where(any_pos[seg_id], np.log(u) / weights, u)
    idx = np.arange(total)
    # stable descending key order within each segment: sort by (segment, -key, index)
    order = np.lexsort((idx, -keys, seg_id))
    ordered_seg = seg_id[order]
    first = np.searchsorted(ordered_seg, np.arange(nseg), side="left")
    within = idx - first[ordered_seg]
    chosen = order[within < np.asarray(quotas)[ordered_seg]]
    return chosen[np.lexsort((chosen, seg_id[chosen]))]


def _segment_of(h, layer_index: int, node: int) -> int:
    if layer_index == 0:
        return int(h.bottom_segment_of[node])
    return node // h.s


def _worker_ranges(total: int, threads: int) -> list[tuple[int, int]]:
    threads = max(1, min(threads, total))
    step = (total + threads - 1) // threads
    return [(i, min(i + step, total)) for i in range(0, total, step)]
