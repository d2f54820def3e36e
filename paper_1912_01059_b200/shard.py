"""Sharded indices (drop-in for graphann.shard, /root/reference/pkg/src/graphann/shard.py).

The dataset is shuffled once with default_rng(cfg.seed) and cut into
contiguous shards of `shard_size` (shard.py:54-65); each shard gets its own
hierarchy and shards never link to each other, so they build independently.
A query batch runs on every shard; the query kernel writes each shard's
(m, k_out) lists straight into that shard's "block" of one device buffer
(include/ggnn_shard.h), ggnn_shard_globalize maps local ids to dataset ids,
and ggnn_shard_merge takes the exact top-k_out by (distance, dataset id) --
_merge_shard_results (shard.py:91-110) for the whole batch in one launch.

On one GPU the shards are searched back to back (the reference's
oversubscribed mode); with one process per GPU the same
blocks are the NCCL all-gather buffers (distributed.py).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from .build import BuildStats, build
from .config import BuildConfig, QueryConfig
from .data import Dataset, FormatError
from .graph import Hierarchy
from .index_file import load_index, save_index
from .search import BatchResult, QueryResult, launch_query

MANIFEST = "manifest.json"
PERMFILE = "permutation.i32"


@dataclass
class ShardedIndex:
    shards: list[tuple[int, Hierarchy]]  # (offset into the shuffled order, sub-index)
    shard_size: int
    permutation: np.ndarray  # shuffled position -> dataset id
    config: BuildConfig

    def __post_init__(self):
        expect = 0
        for off, h in self.shards:
            if off != expect:
                raise ValueError(f"shard offsets must tile 0..n-1, got {[o for o, _ in self.shards]}")
            expect = off + h.n
        if expect != len(self.permutation):
            raise ValueError("shards do not cover the permutation range")
        self._gid_dev: dict = {}

    def gid_of_local(self, i: int):
        """Device int32 slice permutation[offset : offset + n_i] of shard i."""
        key = (i, N.torch().cuda.current_device())
        t = self._gid_dev.get(key)
        if t is None:
            off, h = self.shards[i]
            t = N.to_dev(np.ascontiguousarray(self.permutation[off:off + h.n], dtype=np.int32))
            self._gid_dev[key] = t
        return t


def shard_datasets(dataset: Dataset, shard_size: int, seed: int) -> tuple[np.ndarray, list[tuple[int, Dataset]]]:
    """Seeded shuffle, contiguous slices, per-shard copies (shard.py:54-65)."""
    n = dataset.n
    perm = np.random.default_rng(seed).permutation(n).astype(np.int32)
    out = []
    for i in range(math.ceil(n / shard_size)):
        lo, hi = i * shard_size, min((i + 1) * shard_size, n)
        out.append((lo, Dataset(dataset.vectors[perm[lo:hi]].copy())))
    return perm, out


def build_sharded(dataset: Dataset, shard_size: int, cfg: BuildConfig | None = None,
                  threads: int = 1) -> tuple[ShardedIndex, list[BuildStats]]:
    """ceil(n / shard_size) independent GPU builds (shard.py:68-88)."""
    cfg = cfg or BuildConfig()
    if shard_size < cfg.s:
        raise ValueError(f"shard_size must be >= s (got {shard_size} < {cfg.s})")
    perm, subsets = shard_datasets(dataset, shard_size, cfg.seed)
    shards, stats = [], []
    for idx, (offset, sub) in enumerate(subsets):
        try:
            h, st = build(sub, cfg, threads=threads)
        except Exception as exc:
            raise RuntimeError(f"shard {idx} (offset {offset}) failed to build") from exc
        shards.append((offset, h))
        stats.append(st)
    return ShardedIndex(shards, shard_size, perm, cfg), stats


# ------------------------------------------------------------- block buffers
def block_layout(m: int, k: int) -> tuple[int, int, int]:
    """(block bytes, dists offset, counters offset) of one shard block."""
    lib = N.load()
    return (int(lib.ggnn_shard_block_bytes(m, k)), int(lib.ggnn_shard_block_dists_offset(m, k)),
            int(lib.ggnn_shard_block_counters_offset(m, k)))


def block_pointers(buf, g: int, m: int, k: int):
    """Device pointers (ids, dists, counters) of block g inside `buf`."""
    bb, doff, coff = block_layout(m, k)
    base = buf.data_ptr() + g * bb
    return N.P(base), N.P(base + doff), N.P(base + coff)


def search_into_block(h: Hierarchy, Q: np.ndarray, cfg: QueryConfig, buf, g: int, gid_of_local,
                      uploaded: dict | None = None) -> None:
    """query() of every row of Q on hierarchy h, written into block g of
    `buf` with ids mapped to dataset ids through gid_of_local (device int32).
    `uploaded`: the caller's per-batch cache of the device queries."""
    m = Q.shape[0]
    ids_p, dists_p, cnt_p = block_pointers(buf, g, m, cfg.k_out)
    launch_query(h, Q, cfg, ids_p, dists_p, cnt_p, uploaded)
    N.call("ggnn_shard_globalize", ids_p, m * cfg.k_out, N.ptr(gid_of_local), int(gid_of_local.numel()),
           N.stream_ptr())


def merge_blocks(buf, G: int, m: int, k: int, k_out: int):
    """ggnn_shard_merge over G blocks -> device (ids, dists, counters)."""
    t = N.torch()
    ids = N.empty((m, k_out), t.int32)
    dists = N.empty((m, k_out), t.float64)
    cnt = N.empty((m, 5), t.int32)
    N.call("ggnn_shard_merge", N.ptr(buf), G, m, k, k_out, N.ptr(ids), N.ptr(dists), N.ptr(cnt), N.stream_ptr())
    return ids, dists, cnt


def query_sharded_arrays(si: ShardedIndex, queries: np.ndarray, cfg: QueryConfig | None = None,
                         out: str = "numpy"):
    """Batched query_sharded: every shard answers the batch on this GPU, then
    one merge launch.  Returns a BatchResult (or device tensors)."""
    cfg = cfg or QueryConfig()
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    if Q.ndim == 1:
        Q = Q[None, :]
    m, G = Q.shape[0], len(si.shards)
    bb = block_layout(m, cfg.k_out)[0]
    buf = N.empty((G * bb,), N.torch().uint8)
    up = {}  # the batch is uploaded once for all shards
    for g, (_, h) in enumerate(si.shards):
        search_into_block(h, Q, cfg, buf, g, si.gid_of_local(g), up)
    ids, dists, cnt = merge_blocks(buf, G, m, cfg.k_out, cfg.k_out)
    if out == "device":
        return ids, dists, cnt
    return BatchResult(ids.cpu().numpy(), dists.cpu().numpy(), cnt.cpu().numpy())


def query_sharded(si: ShardedIndex, q: np.ndarray, cfg: QueryConfig | None = None, threads: int = 1) -> QueryResult:
    """Query every shard and merge to the global top k_out (shard.py:113-128);
    `threads` is ignored."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    if q.ndim != 1:
        raise ValueError(f"expected one query vector, got shape {q.shape}")
    return query_sharded_arrays(si, q[None, :], cfg).results()[0]


def batch_query_sharded(si: ShardedIndex, queries: np.ndarray, cfg: QueryConfig | None = None) -> list[QueryResult]:
    return query_sharded_arrays(si, queries, cfg).results()


# ---------------------------------------------------------------- persistence
def save_sharded(si: ShardedIndex, dir_path) -> None:
    """manifest.json + permutation.i32 + shard_XXXX.idx (shard.py:131-147)."""
    root = Path(dir_path)
    root.mkdir(parents=True, exist_ok=True)
    files = [f"shard_{i:04d}.idx" for i in range(len(si.shards))]
    manifest = {"version": 1, "shard_count": len(si.shards), "shard_size": si.shard_size,
                "n": int(len(si.permutation)), "offsets": [off for off, _ in si.shards],
                "config": si.config.to_dict(), "permutation_file": PERMFILE, "shard_files": files}
    (root / MANIFEST).write_text(json.dumps(manifest, indent=2, sort_keys=True))
    (root / PERMFILE).write_bytes(np.ascontiguousarray(si.permutation, dtype="<i4").tobytes())
    for f, (_, h) in zip(files, si.shards):
        save_index(h, root / f)


def _manifest(root: Path) -> tuple[dict, np.ndarray]:
    mf = root / MANIFEST
    if not mf.exists():
        raise FormatError(f"{root}: missing {MANIFEST}")
    manifest = json.loads(mf.read_text())
    if manifest.get("version") != 1:
        raise FormatError(f"{root}: unsupported sharded-index version {manifest.get('version')}")
    perm = np.frombuffer((root / manifest["permutation_file"]).read_bytes(), dtype="<i4").astype(np.int32)
    return manifest, perm


def load_sharded(dir_path, dataset: Dataset) -> ShardedIndex:
    """Load every shard and attach its slice of the dataset (shard.py:159-172)."""
    root = Path(dir_path)
    manifest, perm = _manifest(root)
    shards = []
    for off, fname in zip(manifest["offsets"], manifest["shard_files"]):
        h = load_index(root / fname)
        h.attach(Dataset(dataset.vectors[perm[off:off + h.n]].copy()))
        shards.append((off, h))
    return ShardedIndex(shards, manifest["shard_size"], perm, BuildConfig.from_dict(manifest["config"]))


def iter_shard_results(dir_path, dataset: Dataset, q: np.ndarray, cfg: QueryConfig | None = None):
    """Yield (offset, QueryResult) one shard at a time, holding one sub-index
    (host and device) at a time (shard.py:175-187)."""
    from .search import query

    cfg = cfg or QueryConfig()
    root = Path(dir_path)
    manifest, perm = _manifest(root)
    for off, fname in zip(manifest["offsets"], manifest["shard_files"]):
        h = load_index(root / fname)
        h.attach(Dataset(dataset.vectors[perm[off:off + h.n]].copy()))
        yield off, query(h, q, cfg)
        del h


def query_sharded_sequential_arrays(dir_path, dataset: Dataset, queries: np.ndarray,
                                    cfg: QueryConfig | None = None) -> BatchResult:
    """Bounded-memory batched sharded query: shards are loaded, searched into
    their block and released one at a time, then merged once."""
    cfg = cfg or QueryConfig()
    root = Path(dir_path)
    manifest, perm = _manifest(root)
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    if Q.ndim == 1:
        Q = Q[None, :]
    m, G = Q.shape[0], len(manifest["offsets"])
    bb = block_layout(m, cfg.k_out)[0]
    buf = N.empty((G * bb,), N.torch().uint8)
    for g, (off, fname) in enumerate(zip(manifest["offsets"], manifest["shard_files"])):
        h = load_index(root / fname)
        h.attach(Dataset(dataset.vectors[perm[off:off + h.n]].copy()))
        gid = N.to_dev(np.ascontiguousarray(perm[off:off + h.n], dtype=np.int32))
        search_into_block(h, Q, cfg, buf, g, gid)
        N.torch().cuda.synchronize()
        del h, gid
    ids, dists, cnt = merge_blocks(buf, G, m, cfg.k_out, cfg.k_out)
    return BatchResult(ids.cpu().numpy(), dists.cpu().numpy(), cnt.cpu().numpy())


def query_sharded_sequential(dir_path, dataset: Dataset, q: np.ndarray, cfg: QueryConfig | None = None) -> QueryResult:
    """Bounded-memory variant of query_sharded over a persisted directory
    (shard.py:190-199)."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    return query_sharded_sequential_arrays(dir_path, dataset, q[None, :], cfg).results()[0]
