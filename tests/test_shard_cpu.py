"""Multi-process sharding plumbing on CPU (gloo, world_size 2 and 3).

The per-rank search and the merge are the GPU kernels in production; here a
test subclass replaces exactly those two methods with the CPU checker (exact
per-shard scans written into the real shard-block layout, and the oracle's
restatement of _merge_shard_results, shard.py:91-110), so everything else --
shard assignment from the seeded permutation, id globalization, the
all-gather block order and the block layout of include/ggnn_shard.h -- runs
as shipped.  Expected result: every rank holds the exact global top-k_out
(reference test_shard.py:78-97: oracle-substituted shards merge to the
global brute force).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O  # tests/conftest.py puts oracle/ on sys.path (the CPU checker)
import paper_1912_01059_b200 as ga
from paper_1912_01059_b200.distributed import ShardGroup
from paper_1912_01059_b200.shard import block_layout

K_OUT = 5


class CpuShardGroup(ShardGroup):
    def new_buffer(self, nbytes):
        return torch.zeros(nbytes, dtype=torch.uint8)

    def search_shard(self, s, h, gid, Q, cfg, buf, uploaded=None):
        m, k = Q.shape[0], cfg.k_out
        bb, doff, coff = block_layout(m, k)
        raw = buf.numpy()[s * bb:(s + 1) * bb]
        ids = raw[: m * k * 4].view(np.int32).reshape(m, k)
        dists = raw[doff: doff + m * k * 8].view(np.float64).reshape(m, k)
        cnt = raw[coff: coff + m * 20].view(np.int32).reshape(m, 5)
        X = h.vectors
        g = self.rank * self.per_rank + s  # global shard index
        for i in range(m):
            lid, ld = O.exhaustive_topk(X, Q[i], k)
            ids[i] = -1
            dists[i] = np.inf
            ids[i, : len(lid)] = gid[lid]
            dists[i, : len(lid)] = ld
            cnt[i] = [X.shape[0], 1 + g, g % 3, 7, 9]

    def merge(self, recv, m, cfg):
        k = cfg.k_out
        bb, doff, coff = block_layout(m, k)
        raw = recv.numpy()
        n_total = int(max(raw[g * bb: g * bb + m * k * 4].view(np.int32).max() for g in range(self.n_blocks))) + 1
        ident = np.arange(n_total, dtype=np.int32)
        out_ids = np.full((m, k), -1, dtype=np.int32)
        out_d = np.full((m, k), np.inf)
        out_c = np.zeros((m, 5), dtype=np.int32)
        for i in range(m):
            parts = []
            for g in range(self.n_blocks):
                blk = raw[g * bb:(g + 1) * bb]
                ids = blk[: m * k * 4].view(np.int32).reshape(m, k)[i]
                ds = blk[doff: doff + m * k * 8].view(np.float64).reshape(m, k)[i]
                c = blk[coff: coff + m * 20].view(np.int32).reshape(m, 5)[i]
                keep = ids >= 0
                parts.append((0, ids[keep], ds[keep], c[0], c[1], c[2]))
            gi, gd, v, t, term = O.merge_shard_results(parts, ident, k)
            out_ids[i, : len(gi)] = gi
            out_d[i, : len(gd)] = gd
            out_c[i] = [v, t, term, 0, 0]
        return torch.from_numpy(out_ids), torch.from_numpy(out_d), torch.from_numpy(out_c)


def _data(n=503, d=8, m=24, seed=5):
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 16, size=(n, d)).astype(np.float32)  # many distance ties
    Q = rng.integers(0, 16, size=(m, d)).astype(np.float32)
    return X, Q


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Q = _data()
        cfg = ga.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, seed=11)
        grp = CpuShardGroup.from_dataset(ga.Dataset(X), cfg, build_fn=lambda sub, c: (sub, None))
        res = grp.query_arrays(Q, ga.QueryConfig(k_out=K_OUT, prioq_size=16))
        q.put((rank, res.ids, res.dists, res.counters, grp.gid_host))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_query_plumbing_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    X, Q = _data()
    # the ranks' shards tile the seeded permutation (shard.py:54-65)
    perm = np.random.default_rng(11).permutation(X.shape[0]).astype(np.int32)
    np.testing.assert_array_equal(np.concatenate([o[4] for o in out]), perm)
    owner = np.empty(X.shape[0], dtype=np.int32)
    for r, *_rest, gid in out:
        owner[gid] = r
    for i in range(Q.shape[0]):
        ids, ds = O.exhaustive_topk(X, Q[i], K_OUT)  # global brute force, ties by id
        for r, rid, rd, rc, _ in out:
            np.testing.assert_array_equal(rid[i], ids)
            np.testing.assert_array_equal(rd[i], ds)
            sizes = [len(o[4]) for o in out]
            assert rc[i, 0] == sum(sizes)
            assert rc[i, 1] == sum(1 + g for g in range(world))
            assert rc[i, 2] == owner[ids[0]] % 3
            assert rc[i, 3] == 0 and rc[i, 4] == 0


N_SHARDS = 8


def _shard_loader(i):
    """Rank-local loader of shard i of the 8-shard layout (the seeded
    permutation cut into 8 contiguous slices, shard.py:54-65)."""
    X, _ = _data()
    perm = np.random.default_rng(11).permutation(X.shape[0]).astype(np.int32)
    size = -(-X.shape[0] // N_SHARDS)
    gid = perm[i * size:(i + 1) * size]
    return ga.Dataset(X[gid].copy()), gid


def _local_worker(rank, world, port, q):
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Q = _data()
        grp = CpuShardGroup.from_local_shards(_shard_loader, N_SHARDS, build_fn=lambda sub, c: (sub, None))
        res = grp.query_arrays(Q, ga.QueryConfig(k_out=K_OUT, prioq_size=16))
        q.put((rank, res.ids, res.dists, res.counters, [g for _, g in grp.shards]))
    finally:
        if world > 1:
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_eight_shards_over_ranks_equal_one_rank(world):
    """A fixed 8-shard index over 2 and 4 ranks (each rank loads and holds
    only its 8 / world shards) answers exactly like one process holding all
    8 shards and searching them in turn (the north star's QPS_1 layout);
    both equal the global brute force."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    runs = {}
    for w in (1, world):
        procs = [ctx.Process(target=_local_worker, args=(r, w, port + (w > 1), q)) for r in range(w)]
        for p in procs:
            p.start()
        runs[w] = sorted([q.get(timeout=120) for _ in range(w)], key=lambda t: t[0])
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    X, Q = _data()
    one = runs[1][0]
    assert len(one[4]) == N_SHARDS
    held = [g for r in runs[world] for g in r[4]]  # ranks hold consecutive shards in global order
    assert len(held) == N_SHARDS and all(len(r[4]) == N_SHARDS // world for r in runs[world])
    for a, b in zip(held, one[4]):
        np.testing.assert_array_equal(a, b)
    for r, ids, ds, cnt, _ in runs[world]:
        np.testing.assert_array_equal(ids, one[1])
        np.testing.assert_array_equal(ds, one[2])
        np.testing.assert_array_equal(cnt, one[3])
    for i in range(Q.shape[0]):
        ids, ds = O.exhaustive_topk(X, Q[i], K_OUT)
        np.testing.assert_array_equal(one[1][i], ids)
        np.testing.assert_array_equal(one[2][i], ds)
        assert one[3][i, 1] == sum(1 + g for g in range(N_SHARDS))
