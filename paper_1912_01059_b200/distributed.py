"""One shard per GPU: multi-process sharded build and search.

The paper's multi-GPU mode (reference shard.py:1-12,
91-128): shard r of the seeded permutation lives on rank r (one process per
GPU, torch.distributed over NCCL).  Builds need no communication.  A query
batch is replicated on every rank; each rank's query kernel writes its
(m, k_out) results into its own shard block, ids are globalized in place
(ggnn_shard_globalize), one all_gather_into_tensor moves the G blocks to
every rank (0.8 MB per rank at m = 10k, k_out = 10), and ggnn_shard_merge
produces the exact global top-k_out.  The send buffer IS the query kernel's
output, so the only data movement besides the search is the all-gather.

    grp = ShardGroup.from_dataset(dataset, cfg)      # every rank, same args
    res = grp.query_arrays(Q, QueryConfig(...))      # every rank gets the merged result
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as N
from .config import BuildConfig, QueryConfig
from .data import Dataset
from .search import BatchResult


class ShardGroup:
    """This rank's shard plus the process group that holds the others."""

    def __init__(self, h, gid_of_local: np.ndarray, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.h = h
        self.gid_host = np.ascontiguousarray(gid_of_local, dtype=np.int32)
        self._gid_dev = None

    # ---------------------------------------------------------- construction
    @classmethod
    def from_dataset(cls, dataset: Dataset, cfg: BuildConfig | None = None, group=None, build_fn=None):
        """Every rank passes the same dataset; rank r builds shard r of
        shard_datasets(dataset, ceil(n / world), cfg.seed) -- the same shards
        build_sharded makes for shard_size = ceil(n / world)."""
        import torch.distributed as dist

        from .build import build

        cfg = cfg or BuildConfig()
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        n = dataset.n
        size = math.ceil(n / world)
        if size < cfg.s:
            raise ValueError(f"shard size {size} < s={cfg.s}: too many ranks for {n} points")
        perm = np.random.default_rng(cfg.seed).permutation(n).astype(np.int32)
        lo, hi = rank * size, min((rank + 1) * size, n)
        gid = perm[lo:hi]
        sub = Dataset(dataset.vectors[gid].copy())
        h, stats = (build_fn or build)(sub, cfg)
        grp = cls(h, gid, group)
        grp.build_stats = stats
        return grp

    # -------------------------------------------------------------- search
    def gid_dev(self):
        if self._gid_dev is None:
            self._gid_dev = N.to_dev(self.gid_host)
        return self._gid_dev

    def block_bytes(self, m: int, k: int) -> int:
        from .shard import block_layout

        return block_layout(m, k)[0]

    def new_buffer(self, nbytes: int):
        return N.empty((nbytes,), N.torch().uint8)

    def search_block(self, Q: np.ndarray, cfg: QueryConfig, buf) -> None:
        """Search the local shard into block 0 of `buf`, ids globalized."""
        from .shard import search_into_block

        search_into_block(self.h, Q, cfg, buf, 0, self.gid_dev())

    def merge(self, recv, m: int, cfg: QueryConfig):
        from .shard import merge_blocks

        return merge_blocks(recv, self.world, m, cfg.k_out, cfg.k_out)

    def exchange(self, send, recv) -> None:
        """All-gather of the shard blocks (NCCL on device buffers; a gloo
        group -- CPU tests, several ranks sharing one GPU -- stages through
        host memory)."""
        if recv.is_cuda and self.dist.get_backend(self.group) == "gloo":
            r = recv.cpu()
            self.dist.all_gather_into_tensor(r, send.cpu(), group=self.group)
            recv.copy_(r)
            return
        self.dist.all_gather_into_tensor(recv, send, group=self.group)

    def exact_arrays(self, queries: np.ndarray, k: int, out: str = "numpy"):
        """Exact global top-k (k <= 32) of a replicated batch: every rank
        scans its shard (ggnn_exhaustive_topk) into its block, then the same
        all-gather + merge as a search (ground truth for sharded recall)."""
        from .device import DeviceVectors
        from .shard import block_pointers

        Q = np.ascontiguousarray(queries, dtype=np.float32)
        m = Q.shape[0]
        bb = self.block_bytes(m, k)
        send = self.new_buffer(bb)
        send.zero_()
        recv = self.new_buffer(self.world * bb)
        dv = DeviceVectors.of(self.h.dataset)
        dq, qs = dv.queries(Q)
        ids_p, dists_p, _ = block_pointers(send, 0, m, k)
        N.call("ggnn_exhaustive_topk", N.ctypes.byref(dv.struct), None, dv.n, N.ctypes.byref(qs), int(k), ids_p,
               dists_p, N.stream_ptr())
        N.call("ggnn_shard_globalize", ids_p, m * k, N.ptr(self.gid_dev()), int(self.gid_host.shape[0]),
               N.stream_ptr())
        self.exchange(send, recv)
        from .shard import merge_blocks

        ids, dists, cnt = merge_blocks(recv, self.world, m, k, k)
        del dq
        if out == "device":
            return ids, dists
        return np.asarray(ids.cpu()), np.asarray(dists.cpu())

    def query_arrays(self, queries: np.ndarray, cfg: QueryConfig | None = None, out: str = "numpy"):
        """Sharded query of a replicated batch; every rank returns the merged
        global result (shard.py:113-128 for the whole batch)."""
        cfg = cfg or QueryConfig()
        Q = np.ascontiguousarray(queries, dtype=np.float32)
        if Q.ndim == 1:
            Q = Q[None, :]
        m = Q.shape[0]
        bb = self.block_bytes(m, cfg.k_out)
        send = self.new_buffer(bb)
        recv = self.new_buffer(self.world * bb)
        self.search_block(Q, cfg, send)
        self.exchange(send, recv)
        ids, dists, cnt = self.merge(recv, m, cfg)
        if out == "device":
            return ids, dists, cnt
        return BatchResult(np.asarray(ids.cpu()), np.asarray(dists.cpu()), np.asarray(cnt.cpu()))
