"""Shards over GPUs: multi-process sharded build and search.

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
    """This rank's shards plus the process group that holds the others.

    Global shard i lives on rank i // S (S = shards per rank, the same on
    every rank), so an all-gather of every rank's S consecutive blocks lays
    the blocks out in global shard order.  `ShardGroup(h, gid)` is the
    one-shard-per-rank case; without an initialised process group the group
    is this process alone (world 1: one GPU searching all its shards in turn,
    the north star's QPS_1)."""

    def __init__(self, h=None, gid_of_local: np.ndarray | None = None, group=None, shards=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        if shards is None:
            shards = [(h, gid_of_local)]
        self.shards = [(hh, np.ascontiguousarray(g, dtype=np.int32)) for hh, g in shards]
        self.h, self.gid_host = self.shards[0]
        self._gid_devs = {}

    @property
    def per_rank(self) -> int:
        return len(self.shards)

    @property
    def n_blocks(self) -> int:
        """Shards in the whole group (= merged blocks per query)."""
        return self.world * self.per_rank

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

    @classmethod
    def from_local_shards(cls, loader, n_shards: int, cfg: BuildConfig | None = None, group=None, build_fn=None):
        """Rank-local construction: this rank builds only its own shards
        i = rank * S ... rank * S + S - 1 (S = n_shards / world) from
        `loader(i) -> (Dataset, gid)` (gid: the shard's dataset ids, int32);
        no rank ever holds the whole dataset (C5: 8 x 12.5M uint8 shards)."""
        import torch.distributed as dist

        from .build import build

        cfg = cfg or BuildConfig()
        on = dist.is_available() and dist.is_initialized()
        world, rank = (dist.get_world_size(group), dist.get_rank(group)) if on else (1, 0)
        if n_shards % world:
            raise ValueError(f"{n_shards} shards do not divide over {world} ranks")
        per = n_shards // world
        shards, stats = [], []
        for i in range(rank * per, (rank + 1) * per):
            ds, gid = loader(i)
            h, st = (build_fn or build)(ds, cfg)
            shards.append((h, gid))
            stats.append(st)
        grp = cls(group=group, shards=shards)
        grp.build_stats = stats
        return grp

    # -------------------------------------------------------------- search
    def gid_dev(self, s: int = 0):
        if s not in self._gid_devs:
            self._gid_devs[s] = N.to_dev(self.shards[s][1])
        return self._gid_devs[s]

    def block_bytes(self, m: int, k: int) -> int:
        from .shard import block_layout

        return block_layout(m, k)[0]

    def new_buffer(self, nbytes: int):
        return N.empty((nbytes,), N.torch().uint8)

    def search_block(self, Q: np.ndarray, cfg: QueryConfig, buf) -> None:
        """Search every local shard s into block s of `buf`, ids globalized
        (the shards one after the other on this rank's stream)."""
        up = {}  # the batch is uploaded once for all local shards
        for s, (h, gid) in enumerate(self.shards):
            self.search_shard(s, h, gid, Q, cfg, buf, up)

    def search_shard(self, s: int, h, gid, Q: np.ndarray, cfg: QueryConfig, buf, uploaded=None) -> None:
        from .shard import search_into_block

        search_into_block(h, Q, cfg, buf, s, self.gid_dev(s), uploaded)

    def merge(self, recv, m: int, cfg: QueryConfig):
        from .shard import merge_blocks

        return merge_blocks(recv, self.n_blocks, m, cfg.k_out, cfg.k_out)

    def exchange(self, send, recv) -> None:
        """All-gather of the shard blocks (NCCL on device buffers; a gloo
        group -- CPU tests, several ranks sharing one GPU -- stages through
        host memory; world 1: the blocks are already all here)."""
        if not self.on:
            if recv.data_ptr() != send.data_ptr():
                recv.copy_(send)
            return
        if recv.is_cuda and self.dist.get_backend(self.group) == "gloo":
            r = recv.cpu()
            self.dist.all_gather_into_tensor(r, send.cpu(), group=self.group)
            recv.copy_(r)
            return
        self.dist.all_gather_into_tensor(recv, send, group=self.group)

    def exact_arrays(self, queries: np.ndarray, k: int, out: str = "numpy"):
        """Exact global top-k of a replicated batch: every rank scans its
        shards (ggnn_exhaustive_topk) into its blocks, then the same
        all-gather + merge as a search (ground truth for sharded recall)."""
        from .device import DeviceVectors
        from .shard import block_pointers

        Q = np.ascontiguousarray(queries, dtype=np.float32)
        m = Q.shape[0]
        bb = self.block_bytes(m, k)
        send = self.new_buffer(self.per_rank * bb)
        send.zero_()
        recv = self.new_buffer(self.n_blocks * bb) if self.on else send
        for s, (h, gid) in enumerate(self.shards):
            dv = DeviceVectors.of(h.dataset)
            dq, qs = dv.queries(Q)
            ids_p, dists_p, _ = block_pointers(send, s, m, k)
            N.call("ggnn_exhaustive_topk", N.ctypes.byref(dv.struct), None, dv.n, N.ctypes.byref(qs), int(k), ids_p,
                   dists_p, N.stream_ptr())
            N.check_tc_timeouts("bf")
            N.call("ggnn_shard_globalize", ids_p, m * k, N.ptr(self.gid_dev(s)), int(gid.shape[0]), N.stream_ptr())
            del dq
        self.exchange(send, recv)
        from .shard import merge_blocks

        ids, dists, cnt = merge_blocks(recv, self.n_blocks, m, k, k)
        if out == "device":
            return ids, dists
        return np.asarray(ids.cpu()), np.asarray(dists.cpu())

    def query_arrays(self, queries: np.ndarray, cfg: QueryConfig | None = None, out: str = "numpy",
                     exchange: str = "nccl"):
        """Sharded query of a replicated batch; every rank returns the merged
        global result (shard.py:113-128 for the whole batch).  exchange="p2p"
        fuses the exchange into the search (P2PExchange); same results."""
        cfg = cfg or QueryConfig()
        Q = np.ascontiguousarray(queries, dtype=np.float32)
        if Q.ndim == 1:
            Q = Q[None, :]
        m = Q.shape[0]
        if exchange == "p2p":
            if self.per_rank != 1 or not self.on:
                raise ValueError("the fused exchange needs exactly one shard per rank in a process group")
            ids, dists, cnt = self.p2p(m, cfg.k_out).query(Q, cfg)
        elif exchange == "nccl":
            bb = self.block_bytes(m, cfg.k_out)
            send = self.new_buffer(self.per_rank * bb)
            recv = self.new_buffer(self.n_blocks * bb) if self.on else send
            self.search_block(Q, cfg, send)
            self.exchange(send, recv)
            ids, dists, cnt = self.merge(recv, m, cfg)
        else:
            raise ValueError(f"exchange must be 'nccl' or 'p2p', got {exchange!r}")
        if out == "device":
            return ids, dists, cnt
        return BatchResult(np.asarray(ids.cpu()), np.asarray(dists.cpu()), np.asarray(cnt.cpu()))

    def p2p(self, m: int, k: int) -> "P2PExchange":
        """The (collectively created) fused-exchange state for batches of m
        queries and k results; cached per (m, k).  Every rank must call it
        with the same arguments in the same order."""
        cache = self.__dict__.setdefault("_p2p", {})
        if (m, k) not in cache:
            cache[(m, k)] = P2PExchange(self, m, k)
        return cache[(m, k)]

    def close(self) -> None:
        """Release the fused-exchange mappings (collective)."""
        for x in self.__dict__.pop("_p2p", {}).values():
            x.close()


class P2PExchange:
    """Search and exchange fused over peer memory (include/ggnn_p2p.h).

    Every rank owns one receive allocation of two parity halves, each G shard
    blocks + G flags, and maps every peer's allocation through CUDA IPC (over
    NVLink / NVSwitch on a multi-GPU node; two ranks on one GPU work too).
    One step on the rank's stream:
      ggnn_query_batch_push   -- each warp stores its finished query's
                                 globalized row into block `rank` of all G
                                 allocations (transfer overlaps the search)
      ggnn_p2p_signal         -- system fence, epoch -> flag `rank` everywhere
      ggnn_shard_merge_wait   -- spin (bounded) on the G local flags, merge
    Epoch e uses parity e & 1: a rank can only reach epoch e after every
    peer signalled e - 1, which on that peer's stream follows its merge of
    e - 2, so a half is never overwritten while it is being merged."""

    def __init__(self, grp: ShardGroup, m: int, k: int):
        t = N.torch()
        self.grp, self.m, self.k, self.G, self.rank = grp, m, k, grp.world, grp.rank
        if self.G > 8:
            raise ValueError("the fused exchange supports at most 8 ranks")
        nbytes = N.load().ggnn_p2p_bytes(self.G, m, k)
        self.own = N.P()
        handle = (N.ctypes.c_uint8 * 64)()
        N.call("ggnn_p2p_alloc", N.ctypes.c_size_t(nbytes), N.ctypes.byref(self.own), handle)
        handles = [None] * self.G
        grp.dist.all_gather_object(handles, bytes(handle), group=grp.group)
        self.peers = []
        for g, hb in enumerate(handles):
            if g == self.rank:
                self.peers.append(self.own)
                continue
            p = N.P()
            buf = (N.ctypes.c_uint8 * 64).from_buffer_copy(hb)
            N.call("ggnn_p2p_open", buf, N.ctypes.byref(p))
            self.peers.append(p)
        grp.dist.barrier(group=grp.group)
        self.epoch = 0
        self.push = N.Push()
        for g, p in enumerate(self.peers):
            self.push.d_peers[g] = p
        self.push.nranks, self.push.rank = self.G, self.rank
        gid = grp.gid_dev()
        self.push.d_gid_of_local, self.push.gid_size = N.ptr(gid), int(grp.gid_host.shape[0])
        self.error = t.zeros((1,), dtype=t.int32, device=N.device())
        # the shard-local results (unused by the merge) land here
        self.local_ids = N.empty((m, k), t.int32)
        self.local_dists = N.empty((m, k), t.float64)
        self.local_cnt = N.empty((m, 5), t.int32)

    def search_push(self, h, Q: np.ndarray, cfg: QueryConfig) -> None:
        """Launch the push search + signal of the next epoch (no merge)."""
        from .device import device_hierarchy
        from .search import _params, _qflags

        if Q.shape[0] != self.m or cfg.k_out != self.k:
            raise ValueError("batch shape does not match this exchange")
        self.epoch += 1
        self.push.parity = self.epoch & 1
        dh = device_hierarchy(h)
        dv = dh.vectors
        dq, qs = dv.queries(Q)
        params = _params(cfg, _qflags(dh, False))
        N.call("ggnn_query_batch_push", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max,
               N.ptr(self.local_ids), N.ptr(self.local_dists), N.ptr(self.local_cnt), N.ctypes.byref(self.push),
               N.stream_ptr())
        N.call("ggnn_p2p_signal", N.ctypes.byref(self.push), self.m, self.k, N.ctypes.c_uint32(self.epoch),
               N.stream_ptr())
        self._dq = dq  # keep the device queries alive until the stream passes them

    def merge_into(self, ids, dists, cnt) -> None:
        N.call("ggnn_shard_merge_wait", self.own, self.epoch & 1, N.ctypes.c_uint32(self.epoch), self.G, self.m,
               self.k, self.k, N.ptr(ids), N.ptr(dists), N.ptr(cnt), N.ptr(self.error), N.stream_ptr())

    def query(self, Q: np.ndarray, cfg: QueryConfig):
        t = N.torch()
        self.search_push(self.grp.h, Q, cfg)
        ids = N.empty((self.m, self.k), t.int32)
        dists = N.empty((self.m, self.k), t.float64)
        cnt = N.empty((self.m, 5), t.int32)
        self.merge_into(ids, dists, cnt)
        self.check()
        return ids, dists, cnt

    def check(self) -> None:
        if int(self.error.item()):
            raise N.NativeError("fused exchange: a peer's rows did not arrive within the wait bound")

    def close(self) -> None:
        N.torch().cuda.synchronize()
        self.grp.dist.barrier(group=self.grp.group)  # nobody writes into our allocation any more
        for g, p in enumerate(self.peers):
            if g != self.rank:
                N.call("ggnn_p2p_close", p)
        self.grp.dist.barrier(group=self.grp.group)
        N.call("ggnn_p2p_free", self.own)
        self.peers = []
