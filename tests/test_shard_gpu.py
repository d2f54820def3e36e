"""Sharded search on the GPU vs the reference (same graphs) and vs the CPU
checker (merge kernel), plus index persistence round trips of GPU graphs."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import paper_1912_01059_b200 as ga
from paper_1912_01059_b200 import _native as N
from paper_1912_01059_b200.shard import block_layout, merge_blocks
from test_persist import _golden_shards

pytestmark = pytest.mark.gpu


def test_same_graph_sharded_query_bitwise():
    """Reference-built shards queried on the GPU: ids, dists, visited, steps
    and terminated_by equal the reference's query_sharded (shard.py:113-128)."""
    g, X, si = _golden_shards()
    from conftest import load_golden

    Q = load_golden("kernels_int.npz")["Q"]
    res = ga.query_sharded_arrays(si, Q, ga.QueryConfig(k_out=6, tau=0.6))
    np.testing.assert_array_equal(res.ids, g["q_ids"])
    np.testing.assert_array_equal(res.dists, g["q_dists"])
    np.testing.assert_array_equal(res.counters[:, :3], g["q_cnt"])
    one = ga.query_sharded(si, Q[3], ga.QueryConfig(k_out=6, tau=0.6))
    np.testing.assert_array_equal(one.ids, g["q_ids"][3][g["q_ids"][3] >= 0])


@pytest.mark.parametrize("G,k_in,k_out", [(1, 10, 10), (3, 6, 6), (8, 10, 10), (5, 24, 24), (9, 12, 7), (40, 4, 32),
                                          (3, 50, 40), (4, 40, 100), (8, 100, 100)])
def test_merge_kernel_vs_oracle(G, k_in, k_out):
    rng = np.random.default_rng(G * 100 + k_in)
    m = 257
    bb, doff, coff = block_layout(m, k_in)
    raw = np.zeros(G * bb, dtype=np.uint8)
    n_total = G * 1000
    ident = np.arange(n_total, dtype=np.int32)
    gids = rng.permutation(n_total).astype(np.int32).reshape(G, 1000)
    parts_all = [[] for _ in range(m)]
    for gi in range(G):
        blk = raw[gi * bb:(gi + 1) * bb]
        ids = blk[: m * k_in * 4].view(np.int32).reshape(m, k_in)
        ds = blk[doff: doff + m * k_in * 8].view(np.float64).reshape(m, k_in)
        cnt = blk[coff: coff + m * 20].view(np.int32).reshape(m, 5)
        for i in range(m):
            nh = int(rng.integers(0, k_in + 1)) if i % 7 == 0 else k_in
            d = np.sort(rng.integers(0, 40, size=nh).astype(np.float64))  # heavy cross-shard ties
            sel = rng.choice(1000, size=nh, replace=False)
            idl = gids[gi, sel]
            order = np.lexsort((idl, d))
            ids[i] = -1
            ds[i] = np.inf
            ids[i, :nh] = idl[order]
            ds[i, :nh] = d[order]
            cnt[i] = [int(rng.integers(0, 999)), int(rng.integers(0, 99)), int(rng.integers(0, 3)), 5, 5]
            parts_all[i].append((0, ids[i, :nh].copy(), ds[i, :nh].copy(), cnt[i, 0], cnt[i, 1], cnt[i, 2]))
    buf = N.to_dev(raw)
    ids, dists, cnt = merge_blocks(buf, G, m, k_in, k_out)
    ids, dists, cnt = ids.cpu().numpy(), dists.cpu().numpy(), cnt.cpu().numpy()
    for i in range(m):
        gi_, gd, v, t, term = O.merge_shard_results(parts_all[i], ident, k_out)
        nh = len(gi_)
        np.testing.assert_array_equal(ids[i, :nh], gi_)
        np.testing.assert_array_equal(dists[i, :nh], gd)
        assert (ids[i, nh:] == -1).all() and np.isinf(dists[i, nh:]).all()
        assert tuple(cnt[i]) == (v, t, term, 0, 0)


@pytest.mark.parametrize("G,k_in,k_out", [(2, 10, 10), (3, 6, 4), (8, 10, 10), (33, 3, 5)])
def test_merge_kernel_local_order_ties(G, k_in, k_out):
    """Blocks as the sharded search really writes them: each shard's list is
    ordered by (dist, LOCAL id) and then globalized through a permutation that
    reverses local order, so inside a shard two hits tied on distance come out
    in descending global id.  The merged ids, dists, sums and terminated_by
    (taken from the shard holding the best hit, which need not be its list's
    first entry) equal the reference's _merge_shard_results (shard.py:91-110)."""
    rng = np.random.default_rng(G * 31 + k_in)
    m, per = 300, 400
    n_total = G * per
    perm = np.arange(n_total, dtype=np.int32)[::-1].copy()  # reverses every tie
    bb, doff, coff = block_layout(m, k_in)
    raw = np.zeros(G * bb, dtype=np.uint8)
    parts_all = [[] for _ in range(m)]
    for gi in range(G):
        off = gi * per
        blk = raw[gi * bb:(gi + 1) * bb]
        ids = blk[: m * k_in * 4].view(np.int32).reshape(m, k_in)
        ds = blk[doff: doff + m * k_in * 8].view(np.float64).reshape(m, k_in)
        cnt = blk[coff: coff + m * 20].view(np.int32).reshape(m, 5)
        for i in range(m):
            nh = int(rng.integers(0, k_in + 1)) if i % 11 == 0 else k_in
            d = rng.integers(0, 3, size=nh).astype(np.float64)  # almost every hit ties
            loc = rng.choice(per, size=nh, replace=False).astype(np.int32)
            order = np.lexsort((loc, d))  # the shard's own (dist, local id) order
            loc, d = loc[order], d[order]
            ids[i] = -1
            ds[i] = np.inf
            ids[i, :nh] = perm[off + loc]  # ggnn_shard_globalize
            ds[i, :nh] = d
            cnt[i] = [int(rng.integers(0, 999)), int(rng.integers(0, 99)), gi % 3, 5, 5]
            parts_all[i].append((off, loc, d, cnt[i, 0], cnt[i, 1], cnt[i, 2]))
    ids, dists, cnt = merge_blocks(N.to_dev(raw), G, m, k_in, k_out)
    ids, dists, cnt = ids.cpu().numpy(), dists.cpu().numpy(), cnt.cpu().numpy()
    wrong_first = 0
    for i in range(m):
        gi_, gd, v, t, term = O.merge_shard_results(parts_all[i], perm, k_out)
        nh = len(gi_)
        np.testing.assert_array_equal(ids[i, :nh], gi_)
        np.testing.assert_array_equal(dists[i, :nh], gd)
        assert (ids[i, nh:] == -1).all()
        assert tuple(cnt[i]) == (v, t, term, 0, 0), i
        if nh:
            heads = {int(perm[p[0] + p[1][0]]) for p in parts_all[i] if len(p[1])}
            wrong_first += int(gi_[0]) not in heads
    assert wrong_first > 0  # the case position-0 matching missed is exercised


def test_gpu_built_shards_merge_exact_and_persist(tmp_path):
    from paper_1912_01059_b200.synthetic import make_latent16

    base, Q = make_latent16(n=3000, d=32, m=200, seed=3)
    ds = ga.Dataset(base)
    cfg = ga.BuildConfig(seed=7)
    si, stats = ga.build_sharded(ds, 1100, cfg)
    assert [o for o, _ in si.shards] == [0, 1100, 2200] and len(stats) == 3
    qc = ga.QueryConfig(k_out=10, tau=0.6)
    res = ga.query_sharded_arrays(si, Q, qc)
    # oracle-substituted merge of the per-shard GPU answers (test_shard.py:78-97)
    per = [ga.query_arrays(h, Q, qc) for _, h in si.shards]
    for i in range(len(Q)):
        parts = []
        for (off, h), r in zip(si.shards, per):
            keep = r.ids[i] >= 0
            parts.append((off, r.ids[i][keep], r.dists[i][keep], r.counters[i, 0], r.counters[i, 1],
                          r.counters[i, 2]))
        gi, gd, v, t, term = O.merge_shard_results(parts, si.permutation, 10)
        np.testing.assert_array_equal(res.ids[i, :len(gi)], gi)
        np.testing.assert_array_equal(res.dists[i, :len(gd)], gd)
        assert tuple(res.counters[i, :3]) == (v, t, term)
    gt = ga.brute_force_oracle(ds, Q, 10)
    assert ga.recall_at(res.ids, gt.ids[:, 0], 10) >= 0.95
    # persistence: the sequential (one shard resident at a time) path answers identically
    ga.save_sharded(si, tmp_path / "sh")
    seq = ga.shard.query_sharded_sequential_arrays(tmp_path / "sh", ds, Q, qc)
    np.testing.assert_array_equal(seq.ids, res.ids)
    np.testing.assert_array_equal(seq.dists, res.dists)
    back = ga.load_sharded(tmp_path / "sh", ds)
    np.testing.assert_array_equal(ga.query_sharded_arrays(back, Q, qc).ids, res.ids)


def test_gpu_built_index_save_load_query(tmp_path):
    from paper_1912_01059_b200.synthetic import make_latent16

    base, Q = make_latent16(n=2500, d=64, m=100, seed=9)
    ds = ga.Dataset(base)
    h, _ = ga.build(ds, ga.BuildConfig(seed=7))
    qc = ga.QueryConfig(k_out=10, tau=0.5)
    a = ga.query_arrays(h, Q, qc)
    ga.save_index(h, tmp_path / "g.idx")
    h2 = ga.load_index(tmp_path / "g.idx").attach(ds)
    b = ga.query_arrays(h2, Q, qc)
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dists, b.dists)
    np.testing.assert_array_equal(a.counters, b.counters)
    # and the CPU checker, querying the loaded file's graph, agrees bit for bit
    layers = [(L.adjacency, L.k_nn, L.sym_count) for L in h2.layers]
    for i in range(0, 100, 7):
        ids, dd, v, t, term, _, _ = O.query(layers, h2.to_bottom, base, Q[i], 10, 0.5, h2.stats.d_nn1_max)
        np.testing.assert_array_equal(a.ids[i, :len(ids)], ids)
        assert (a.counters[i, 0], a.counters[i, 1], a.counters[i, 2]) == (v, t, term)


def test_brute_force_oracle_and_knn_graph():
    rng = np.random.default_rng(1)
    X = rng.integers(0, 8, size=(700, 6)).astype(np.float32)
    ds = ga.Dataset(X)
    Q = rng.integers(0, 8, size=(50, 6)).astype(np.float32)
    gt = ga.brute_force_oracle(ds, Q, 7)
    for i in range(50):
        ids, d = O.exhaustive_topk(X, Q[i], 7)
        np.testing.assert_array_equal(gt.ids[i], ids)
        np.testing.assert_array_equal(gt.dists[i], d)
    with pytest.raises(ValueError):
        ga.brute_force_oracle(ds, Q, 10_000)
    kg = ga.oracle_knn_graph(ds, 3)
    for i in range(0, 700, 37):
        ids, _ = O.exhaustive_topk(X, X[i], 4)
        np.testing.assert_array_equal(kg[i], [v for v in ids if v != i][:3])


def test_fused_exchange_kernels_one_process():
    """The push search + signal + merge-wait kernels with G = 3 "ranks" in
    one process (own allocations, no IPC): every rank's merged result equals
    the unfused block search + ggnn_shard_merge, over 4 epochs (both
    parities, each reused)."""
    import ctypes

    import torch

    from paper_1912_01059_b200.search import _flags, _params
    from paper_1912_01059_b200.device import device_hierarchy
    from paper_1912_01059_b200.synthetic import make_latent16

    base, Q = make_latent16(n=3000, d=32, m=130, seed=5)
    ds = ga.Dataset(base)
    si, _ = ga.build_sharded(ds, 1000, ga.BuildConfig(seed=7))
    G, m = len(si.shards), Q.shape[0]
    allocs = []
    for _ in range(G):
        p, hd = ctypes.c_void_p(), (ctypes.c_uint8 * 64)()
        N.call("ggnn_p2p_alloc", ctypes.c_size_t(N.load().ggnn_p2p_bytes(G, m, 10)), ctypes.byref(p), hd)
        allocs.append(p)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    gids = [si.gid_of_local(g) for g in range(G)]
    try:
        for epoch, tau in zip(range(1, 5), (0.6, 0.3, 0.6, 0.5)):
            cfg = ga.QueryConfig(k_out=10, tau=tau)
            ref = ga.query_sharded_arrays(si, Q, cfg)
            keep = []
            for g, (_, h) in enumerate(si.shards):
                push = N.Push()
                for j in range(G):
                    push.d_peers[j] = allocs[j]
                push.nranks, push.rank, push.parity = G, g, epoch & 1
                push.d_gid_of_local, push.gid_size = N.ptr(gids[g]), int(gids[g].numel())
                dh = device_hierarchy(h)
                dq, qs = dh.vectors.queries(Q)
                loc = [N.empty((m, 10), torch.int32), N.empty((m, 10), torch.float64), N.empty((m, 5), torch.int32)]
                N.call("ggnn_query_batch_push", ctypes.byref(dh.vectors.struct), ctypes.byref(dh.layers[0].struct),
                       N.ptr(dh.top_rows), dh.ntop, ctypes.byref(qs),
                       ctypes.byref(_params(cfg, _flags(dh.vectors, False))), dh.d_nn1_max, *map(N.ptr, loc),
                       ctypes.byref(push), N.stream_ptr())
                N.call("ggnn_p2p_signal", ctypes.byref(push), m, 10, ctypes.c_uint32(epoch), N.stream_ptr())
                keep += [dq, loc]
            for g in range(G):
                out = [N.empty((m, 10), torch.int32), N.empty((m, 10), torch.float64), N.empty((m, 5), torch.int32)]
                N.call("ggnn_shard_merge_wait", allocs[g], epoch & 1, ctypes.c_uint32(epoch), G, m, 10, 10,
                       *map(N.ptr, out), N.ptr(err), N.stream_ptr())
                assert int(err.item()) == 0
                np.testing.assert_array_equal(out[0].cpu().numpy(), ref.ids)
                np.testing.assert_array_equal(out[1].cpu().numpy(), ref.dists)
                np.testing.assert_array_equal(out[2].cpu().numpy(), ref.counters)
    finally:
        torch.cuda.synchronize()
        for p in allocs:
            N.call("ggnn_p2p_free", p)


def _group_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_1912_01059_b200.distributed import ShardGroup
    from paper_1912_01059_b200.synthetic import make_latent16

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # ranks share the one GPU
    try:
        base, Q = make_latent16(n=3000, d=32, m=150, seed=3)
        grp = ShardGroup.from_dataset(ga.Dataset(base), ga.BuildConfig(seed=7))
        res = grp.query_arrays(Q, ga.QueryConfig(k_out=10, tau=0.6))
        gt_ids, gt_d = grp.exact_arrays(Q, 10)
        # the fused exchange (CUDA IPC between the two processes): three
        # epochs so both parity halves are written and one is reused
        p2p = [grp.query_arrays(Q, ga.QueryConfig(k_out=10, tau=0.6), exchange="p2p") for _ in range(3)]
        grp.close()
        q.put((rank, res.ids, res.dists, res.counters, gt_ids, gt_d,
               [(r.ids, r.dists, r.counters) for r in p2p]))
    finally:
        dist.destroy_process_group()


def test_shard_group_real_kernels_two_ranks():
    """ShardGroup with the real kernels (2 ranks on one GPU, gloo exchange):
    equals query_sharded_arrays over the same shards built in one process,
    and its exact path equals the single-index brute force."""
    import socket

    import torch.multiprocessing as mp

    from paper_1912_01059_b200.synthetic import make_latent16

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_group_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    base, Q = make_latent16(n=3000, d=32, m=150, seed=3)
    ds = ga.Dataset(base)
    si, _ = ga.build_sharded(ds, 1500, ga.BuildConfig(seed=7))
    ref = ga.query_sharded_arrays(si, Q, ga.QueryConfig(k_out=10, tau=0.6))
    gt = ga.brute_force_oracle(ds, Q, 10)
    for _, ids, dists, cnt, gi, gd, p2p in out:
        for pi, pd, pc in p2p:
            np.testing.assert_array_equal(pi, ref.ids)
            np.testing.assert_array_equal(pd, ref.dists)
            np.testing.assert_array_equal(pc, ref.counters)
        np.testing.assert_array_equal(ids, ref.ids)
        np.testing.assert_array_equal(dists, ref.dists)
        np.testing.assert_array_equal(cnt, ref.counters)
        np.testing.assert_array_equal(gi, gt.ids)
        np.testing.assert_array_equal(gd, gt.dists)


@pytest.mark.parametrize("d,hi,k", [(32, 4, 10), (128, 256, 1), (128, 256, 32), (96, 256, 7), (224, 16, 12)])
def test_bruteforce_tensor_cores_vs_checker(d, hi, k):
    """tcgen05 kind::i8 exhaustive top-k (ggnn_exhaustive_topk_tc): ids and
    distances equal the reference's exhaustive_topk (CPU checker, ties by row)
    on uint8 data with many distance ties; n and m not multiples of the tiles."""
    from paper_1912_01059_b200.device import DeviceVectors

    rng = np.random.default_rng(d * 7 + k)
    n, m = 5003, 301
    X = rng.integers(0, hi, size=(n, d)).astype(np.float32)
    X.setflags(write=False)
    Q = rng.integers(0, hi, size=(m, d)).astype(np.float32)
    dv = DeviceVectors.of_array(X)
    dq, qs = dv.queries(Q)
    t = N.torch()
    ids = N.empty((m, k), t.int32)
    dists = N.empty((m, k), t.float64)
    N.call("ggnn_exhaustive_topk_tc", N.ctypes.byref(dv.struct), N.ctypes.byref(qs), k, N.ptr(ids), N.ptr(dists),
           N.stream_ptr())
    ids, dists = ids.cpu().numpy(), dists.cpu().numpy()
    assert N.load().ggnn_bf_timeouts() == 0
    for i in range(m):
        ri, rd = O.exhaustive_topk(X, Q[i], k)
        np.testing.assert_array_equal(ids[i], ri)
        np.testing.assert_array_equal(dists[i], rd)


@pytest.mark.parametrize("k", [33, 100, 128])
def test_bruteforce_tensor_cores_large_k(k):
    """k > 32 (the reference CLI's gt default is 100): one list per query in the
    tensor-core kernel, then a k-way merge of the split lists."""
    rng = np.random.default_rng(k)
    n, m, d = 9001, 130, 64
    X = rng.integers(0, 8, size=(n, d)).astype(np.float32)
    Q = rng.integers(0, 8, size=(m, d)).astype(np.float32)
    gt = ga.brute_force_oracle(ga.Dataset(X), Q, k)
    for i in range(0, m, 7):
        ri, rd = O.exhaustive_topk(X, Q[i], k)
        np.testing.assert_array_equal(gt.ids[i], ri)
        np.testing.assert_array_equal(gt.dists[i], rd)
    # below the tensor-core size the warp scan selects ceil(k / 32) passes of 32
    small = ga.brute_force_oracle(ga.Dataset(X[:1000]), Q, k)
    for i in range(0, m, 9):
        ri, rd = O.exhaustive_topk(X[:1000], Q[i], k)
        np.testing.assert_array_equal(small.ids[i], ri)
        np.testing.assert_array_equal(small.dists[i], rd)


@pytest.mark.parametrize("kind,k", [("normal", 10), ("dups", 32), ("gist", 10), ("offset", 1)])
def test_bruteforce_tf32_tensor_cores_vs_checker(kind, k):
    """Float tables on tcgen05 kind::tf32 (3xTF32 Gram of centred rows, a
    rigorous error bound selects candidates, sequential FP64 re-score): the
    exhaustive top-k equals the reference's exhaustive_topk (CPU checker, ties
    by row) bit for bit -- including duplicated rows (exact ties), the C3
    generator at d = 960, and rows far from the origin."""
    rng = np.random.default_rng(len(kind) * 10 + k)
    if kind == "normal":
        X = rng.standard_normal((9001, 64)).astype(np.float32)
        Q = rng.standard_normal((300, 64)).astype(np.float32)
    elif kind == "dups":
        base = rng.standard_normal((3000, 32)).astype(np.float32)
        X = np.concatenate([base, base, base[:2000]])
        Q = base[rng.integers(0, 3000, size=200)] + np.float32(0.01) * rng.standard_normal((200, 32)).astype(np.float32)
    elif kind == "gist":
        from paper_1912_01059_b200.synthetic import make_latent16

        X, Q = make_latent16(n=6000, d=960, m=64, seed=7, as_float=True)
    else:
        X = (500.0 + rng.standard_normal((5000, 24)) * 0.05).astype(np.float32)
        Q = (500.0 + rng.standard_normal((100, 24)) * 0.05).astype(np.float32)
    X = np.ascontiguousarray(X, dtype=np.float32)
    Q = np.ascontiguousarray(Q, dtype=np.float32)
    gt = ga.brute_force_oracle(ga.Dataset(X), Q, k)
    for i in range(len(Q)):
        ri, rd = O.exhaustive_topk(X, Q[i], k)
        np.testing.assert_array_equal(gt.ids[i], ri)
        np.testing.assert_array_equal(gt.dists[i], rd)
    # dataset rows as queries (exact_knn_rows: the build's consensus probe)
    from paper_1912_01059_b200.search import exact_knn_rows

    rows = rng.choice(X.shape[0], size=40, replace=False).astype(np.int32)
    ids, dd = exact_knn_rows(ga.Dataset(X), rows, k)
    for j, r in enumerate(rows):
        ri, rd = O.exhaustive_topk(X, X[r], k)
        np.testing.assert_array_equal(ids[j], ri)
        np.testing.assert_array_equal(dd[j], rd)
