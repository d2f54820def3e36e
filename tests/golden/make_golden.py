"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (the reference is not present on the GPU box):

    ./oracle/build_ref.sh              # compiles /root/reference/pkg -> oracle/_ref/graphann_ref
    python tests/golden/make_golden.py

Every expected value below is produced by the compiled reference
(`graphann_ref`, backend "compiled"); inputs are seeded and stored (or, for
the 10k x 128 instance, regenerated from the reference's own generator
`make_sift_shaped`, tests/conftest.py:79-87, with a content hash recorded).

Fixtures:
  kernels_int.npz   integer 600x20 data (test_backends.py:21-25), reference
                    build with its CFG; exhaustive_topk, batch_bruteforce,
                    greedy_search (incl. tiny caches), sym_check_pair and
                    query() results with all counters.
  float_small.npz   float clustered 400x12 (test_backends.py:97-111) build and
                    query() results: float parity is tolerance-based.
  sift10k.npz       make_sift_shaped 10k x 128 built with BuildConfig(seed=7)
                    (tests/conftest.py:125-129); layers, stats, and query()
                    results for 100 queries at tau 0.3/0.6/0.8, k_out=10.
  ref_int.idx       the kernels_int.npz hierarchy written by the reference's
                    save_index (GGNN v1 bytes, index_file.py:55-91).
  latent20k.npz     reference build of latent16 (SURVEY 8d G_B) 20k x 128 with
                    BuildConfig(seed=7); query() ids for 2000 fresh queries at
                    tau 0.3 / 0.45 / 0.6 (GPU-built vs reference-built recall,
                    the north star's 0.5-point bar).
  gist3k.npz        float latent16 (d = 960, the C3 "GIST-like" generator)
                    3000 x 960: reference graph + query() results (float parity).
  deep3k.npz        gen_synthetic clustered d = 96, rows L2-normalised (the C4
                    "Deep-like" generator) 3000 x 96: reference graph + results.
  deep100k.npz      the C4 generator (gen_synthetic clustered, 1024 clusters,
                    rows L2-normalised) at 100k x 96 + 1000 held-out queries:
                    query() ids of the reference-built graph at tau 0.3 / 0.6
                    / 1.0 / 2.0 (medium-scale build parity on clustered data).
  latent200k.npz    the C2 generator (latent16) at 200k x 128 + 5000 fresh
                    queries: query() ids of the reference-built graph at tau
                    0.3 / 0.45 / 0.6 (build parity closer to C2's scale).
  sharded_int.npz   reference build_sharded of the kernels_int data
                    (shard_size 250 -> 3 shards), every shard's graph, the
                    permutation, and query_sharded results (ids, dists,
                    visited, steps, term) for the kernels_int queries.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as O  # noqa: E402
from paper_1912_01059_b200.synthetic import make_sift_shaped  # noqa: E402

OUT = Path(__file__).resolve().parent


def graph_arrays(h, prefix=""):
    out = {}
    out[prefix + "num_layers"] = np.int64(h.num_layers)
    out[prefix + "s"] = np.int64(h.s)
    out[prefix + "g"] = np.int64(h.g)
    out[prefix + "stats"] = np.array([h.stats.d_nn1_mean, h.stats.d_nn1_max], dtype=np.float64)
    c = h.config
    out[prefix + "config"] = np.array([c.k, c.k_nn, c.k_sym, c.s, c.g, c.refinements, c.seed], dtype=np.int64)
    out[prefix + "tau_build"] = np.float64(c.tau_build)
    for j, L in enumerate(h.layers):
        out[f"{prefix}adj{j}"] = L.adjacency
        out[f"{prefix}nnd{j}"] = L.nn_dists
        out[f"{prefix}sym{j}"] = L.sym_count
        out[f"{prefix}dnn1_{j}"] = L.d_nn1
        if j:
            out[f"{prefix}tob{j}"] = h.to_bottom[j]
    return out


def query_table(R, h, Q, cfg):
    res = R.batch_query(h, Q, cfg)
    k = cfg.k_out
    ids = np.full((len(res), k), -1, dtype=np.int32)
    dists = np.full((len(res), k), np.inf)
    cnt = np.zeros((len(res), 5), dtype=np.int64)
    term_code = {"stopping-rule": 0, "queue-empty": 1, "iteration-cap": 2}
    for i, r in enumerate(res):
        ids[i, : len(r.ids)] = r.ids
        dists[i, : len(r.dists)] = r.dists
        cnt[i] = [r.visited_count, r.steps, term_code[r.terminated_by], r.distinct_touched, r.forgotten]
    return ids, dists, cnt


def make_kernels_int(R):
    core = R.backend.impl
    rng = np.random.default_rng(77)
    X = rng.integers(0, 256, size=(600, 20)).astype(np.float32)
    cfg = R.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, refinements=1, seed=13)
    h, stats = R.build(R.Dataset(X.copy()), cfg)
    out = {"X": X, "dropped": np.int64(stats.dropped_sym_links)}
    out.update(graph_arrays(h))
    qrng = np.random.default_rng(4242)
    Q = qrng.integers(0, 256, size=(100, 20)).astype(np.float32)
    out["Q"] = Q
    # exhaustive top-k over the whole dataset (k=9), ties by row
    tk_ids, tk_d = zip(*[core.exhaustive_topk(X, q, 9) for q in Q])
    out["topk_ids"], out["topk_d"] = np.stack(tk_ids), np.stack(tk_d)
    # within-batch brute force on a few member sets
    for b, m in enumerate((40, 17, 5, 2)):
        mem = qrng.choice(600, m, replace=False).astype(np.int32)
        pos, dist = core.batch_bruteforce(X, mem, 6)
        out[f"bb_mem{b}"], out[f"bb_pos{b}"], out[f"bb_dist{b}"] = mem, pos, dist
    # query() with all counters at three cache geometries
    for tag, qc in (
        ("q_default", R.QueryConfig(k_out=6, tau=0.6)),
        ("q_tiny", R.QueryConfig(k_out=4, tau=0.6, max_iterations=50, prioq_size=8, visited_size=8)),
        ("q_cap", R.QueryConfig(k_out=3, tau=2.0, max_iterations=7, prioq_size=6, visited_size=3)),
    ):
        ids, dists, cnt = query_table(R, h, Q, qc)
        out[tag + "_ids"], out[tag + "_dists"], out[tag + "_cnt"] = ids, dists, cnt
        out[tag + "_cfg"] = np.array([qc.k_out, qc.max_iterations, qc.prioq_size, qc.visited_size], dtype=np.int64)
        out[tag + "_tau"] = np.float64(qc.tau)
    # greedy_search from random seeds on layer 0 (hand-made seeds)
    L = h.layers[0]
    seeds = qrng.integers(0, 600, size=(100, 5)).astype(np.int32)
    gs_ids = np.full((100, 6), -1, dtype=np.int32)
    gs_d = np.full((100, 6), np.inf)
    gs_cnt = np.zeros((100, 5), dtype=np.int64)
    for i in range(100):
        sd = np.array([core.squared_l2(Q[i], X[s]) for s in seeds[i]])
        r = core.greedy_search(X, h.rows_for(0), L.adjacency, L.k_nn, L.sym_count, Q[i], seeds[i], sd,
                               6, 0.4, h.stats.d_nn1_max, 1000, 12, 16)
        gs_ids[i, : len(r[0])], gs_d[i, : len(r[1])] = r[0], r[1]
        gs_cnt[i] = r[2:]
    out["gs_seeds"], out["gs_ids"], out["gs_d"], out["gs_cnt"] = seeds, gs_ids, gs_d, gs_cnt
    # sym_check_pair on random (x, z) pairs of layer 0
    pairs = qrng.integers(0, 600, size=(400, 2)).astype(np.int32)
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    sc = core.SymScratch(L.node_count, L.k, 4 + 64, 128, 16, 8)
    verdicts, fbs = [], []
    for x, z in pairs:
        v, fb = core.sym_check_pair(X, h.rows_for(0), L.adjacency, L.k_nn, L.sym_count, int(x), int(z),
                                    core.squared_l2(X[x], X[z]), 0.5, h.stats.d_nn1_max, 16, 4, 64, 128, 8, sc)
        verdicts.append(v)
        fbs.append(fb.copy() if v == 2 else np.full(8, -1, dtype=np.int32))
    out["sym_pairs"], out["sym_verdict"], out["sym_fb"] = pairs, np.array(verdicts), np.stack(fbs)
    np.savez_compressed(OUT / "kernels_int.npz", **out)
    print("kernels_int.npz", {k: v.shape for k, v in out.items() if hasattr(v, "shape")}.__len__(), "arrays")


def make_float_small(R):
    ds = R.gen_synthetic(400, 12, seed=3, law="clustered", clusters=8)
    cfg = R.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, refinements=1, seed=13)
    h, _ = R.build(ds, cfg)
    rng = np.random.default_rng(99)
    Q = (rng.standard_normal((50, 12)) * 2).astype(np.float32)
    out = {"X": ds.vectors.copy(), "Q": Q}
    out.update(graph_arrays(h))
    ids, dists, cnt = query_table(R, h, Q, R.QueryConfig(k_out=5, tau=0.6))
    out["q_ids"], out["q_dists"], out["q_cnt"] = ids, dists, cnt
    np.savez_compressed(OUT / "float_small.npz", **out)
    print("float_small.npz")


def make_sift10k(R):
    base, queries = make_sift_shaped()
    sha = hashlib.sha256(base.tobytes() + queries.tobytes()).hexdigest()
    h, stats = R.build(R.Dataset(base.copy()), R.BuildConfig(seed=7))
    out = {"data_sha256": np.array(sha), "build_seconds_ref": np.float64(stats.build_seconds)}
    g = graph_arrays(h)
    # nn_dists are recomputable; keep the fixture small
    out.update({k: v for k, v in g.items() if not k.startswith("nnd")})
    for tau in (0.3, 0.6, 0.8):
        ids, dists, cnt = query_table(R, h, queries, R.QueryConfig(k_out=10, tau=tau))
        t = f"{int(round(tau * 10))}"
        out[f"q{t}_ids"], out[f"q{t}_dists"], out[f"q{t}_cnt"] = ids, dists, cnt
    np.savez_compressed(OUT / "sift10k.npz", **out)
    print("sift10k.npz build", stats.build_seconds, "s")


def make_index_and_sharded(R):
    g = np.load(OUT / "kernels_int.npz")
    X, Q = g["X"], g["Q"]
    cfg = R.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, refinements=1, seed=13)
    h, _ = R.build(R.Dataset(X.copy()), cfg)
    assert np.array_equal(h.layers[0].adjacency, g["adj0"]), "reference build is not reproducible"
    R.save_index(h, OUT / "ref_int.idx")
    si, _ = R.build_sharded(R.Dataset(X.copy()), 250, cfg)
    out = {"perm": si.permutation, "offsets": np.array([o for o, _ in si.shards], dtype=np.int64),
           "shard_size": np.int64(si.shard_size)}
    for i, (_, hs) in enumerate(si.shards):
        out.update(graph_arrays(hs, prefix=f"s{i}_"))
    qc = R.QueryConfig(k_out=6, tau=0.6)
    term_code = {"stopping-rule": 0, "queue-empty": 1, "iteration-cap": 2}
    ids = np.full((len(Q), 6), -1, dtype=np.int32)
    dists = np.full((len(Q), 6), np.inf)
    cnt = np.zeros((len(Q), 3), dtype=np.int64)
    for i, q in enumerate(Q):
        r = R.query_sharded(si, q, qc)
        ids[i, : len(r.ids)], dists[i, : len(r.dists)] = r.ids, r.dists
        cnt[i] = [r.visited_count, r.steps, term_code[r.terminated_by]]
    out["q_ids"], out["q_dists"], out["q_cnt"] = ids, dists, cnt
    np.savez_compressed(OUT / "sharded_int.npz", **out)
    print("ref_int.idx", (OUT / "ref_int.idx").stat().st_size, "bytes; sharded_int.npz", len(si.shards), "shards")


def deep_like(n, m, d=96, seed=1234):
    """C4 generator: gen_synthetic clustered, rows L2-normalised;
    the last m rows are the held-out queries."""
    from paper_1912_01059_b200.data import gen_synthetic

    X = gen_synthetic(n + m, d, seed=seed, law="clustered", clusters=64).vectors.astype(np.float64)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X = X.astype(np.float32)
    return X[:n].copy(), X[n:].copy()


def make_float_shapes(R):
    from paper_1912_01059_b200.synthetic import make_latent16

    for name, (base, queries) in (("gist3k", make_latent16(n=3000, d=960, m=200, seed=1234, as_float=True)),
                                  ("deep3k", deep_like(3000, 200))):
        sha = hashlib.sha256(base.tobytes() + queries.tobytes()).hexdigest()
        h, stats = R.build(R.Dataset(base.copy()), R.BuildConfig(seed=7))
        out = {"data_sha256": np.array(sha), "build_seconds_ref": np.float64(stats.build_seconds)}
        out.update({k: v for k, v in graph_arrays(h).items() if not k.startswith("nnd")})
        ids, dists, cnt = query_table(R, h, queries, R.QueryConfig(k_out=10, tau=0.6))
        out["q_ids"], out["q_dists"], out["q_cnt"] = ids, dists, cnt
        np.savez_compressed(OUT / f"{name}.npz", **out)
        print(name, "build", stats.build_seconds, "s")


def make_latent20k(R):
    from paper_1912_01059_b200.synthetic import make_latent16

    base, queries = make_latent16(n=20000, d=128, m=2000, seed=1234)
    sha = hashlib.sha256(base.tobytes() + queries.tobytes()).hexdigest()
    h, stats = R.build(R.Dataset(base.copy()), R.BuildConfig(seed=7))
    out = {"data_sha256": np.array(sha), "build_seconds_ref": np.float64(stats.build_seconds)}
    for tau in (0.3, 0.45, 0.6):
        ids, dists, cnt = query_table(R, h, queries, R.QueryConfig(k_out=10, tau=tau))
        t = f"{int(round(tau * 100)):03d}"
        out[f"q{t}_ids"], out[f"q{t}_cnt"] = ids, cnt[:, :3]
    np.savez_compressed(OUT / "latent20k.npz", **out)
    print("latent20k build", stats.build_seconds, "s")


def make_latent200k(R):
    """C2's generator at 200k x 128 (latent16, integer-valued) with 5000 fresh
    queries: the reference-built graph's query() ids at tau 0.3 / 0.45 / 0.6
    (build parity one order of magnitude closer to C2 than latent20k)."""
    from paper_1912_01059_b200.synthetic import make_latent16

    base, queries = make_latent16(n=200_000, d=128, m=5000, seed=1234)
    sha = hashlib.sha256(base.tobytes() + queries.tobytes()).hexdigest()
    h, stats = R.build(R.Dataset(base.copy()), R.BuildConfig(seed=7))
    out = {"data_sha256": np.array(sha), "build_seconds_ref": np.float64(stats.build_seconds)}
    for tau in (0.3, 0.45, 0.6):
        ids, dists, cnt = query_table(R, h, queries, R.QueryConfig(k_out=10, tau=tau))
        t = f"{int(round(tau * 100)):03d}"
        out[f"q{t}_ids"], out[f"q{t}_cnt"] = ids, cnt[:, :3]
    np.savez_compressed(OUT / "latent200k.npz", **out)
    print("latent200k build", stats.build_seconds, "s")


def deep_c4(n, m, d=96, seed=1234):
    """C4 generator at size n (1024 clusters as in bench.py --workload deep10m)."""
    from paper_1912_01059_b200.data import gen_synthetic

    X = gen_synthetic(n + m, d, seed=seed, law="clustered", clusters=1024).vectors.astype(np.float64)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X = X.astype(np.float32)
    return X[:n].copy(), X[n:].copy()


def make_deep100k(R):
    base, queries = deep_c4(100_000, 1000)
    sha = hashlib.sha256(base.tobytes() + queries.tobytes()).hexdigest()
    h, stats = R.build(R.Dataset(base.copy()), R.BuildConfig(seed=7))
    out = {"data_sha256": np.array(sha), "build_seconds_ref": np.float64(stats.build_seconds)}
    for tau in (0.3, 0.6, 1.0, 2.0):
        ids, dists, cnt = query_table(R, h, queries, R.QueryConfig(k_out=10, tau=tau))
        t = f"{int(round(tau * 100)):03d}"
        out[f"q{t}_ids"], out[f"q{t}_cnt"] = ids, cnt[:, :3]
    np.savez_compressed(OUT / "deep100k.npz", **out)
    print("deep100k build", stats.build_seconds, "s")


def main():
    R = O.reference_module()
    if R is None:
        raise SystemExit("run oracle/build_ref.sh first (needs /root/reference)")
    assert R.backend.BACKEND == "compiled"
    which = sys.argv[1:] or ["int", "float", "sift", "index", "shapes", "latent20k"]
    if "int" in which:
        make_kernels_int(R)
    if "float" in which:
        make_float_small(R)
    if "sift" in which:
        make_sift10k(R)
    if "index" in which:
        make_index_and_sharded(R)
    if "shapes" in which:
        make_float_shapes(R)
    if "latent20k" in which:
        make_latent20k(R)
    if "deep100k" in which:
        make_deep100k(R)
    if "latent200k" in which:
        make_latent200k(R)


if __name__ == "__main__":
    main()
