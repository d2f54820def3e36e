"""GGNN v1 index files and sharded manifests (host logic, no GPU), plus the
oracle's restatement of the shard merge pinned to the reference's own
query_sharded outputs (tests/golden/sharded_int.npz)."""

from __future__ import annotations

import json

import numpy as np
import pytest

import oracle as O
import paper_1912_01059_b200 as ga
from conftest import GOLDEN, golden_hierarchy, load_golden
from paper_1912_01059_b200.index_file import IndexFormatError, load_index, save_index
from paper_1912_01059_b200.shard import ShardedIndex, load_sharded, save_sharded


def test_load_reference_index_file():
    g = load_golden("kernels_int.npz")
    h = load_index(GOLDEN / "ref_int.idx")
    assert h.num_layers == int(g["num_layers"]) and (h.s, h.g) == (int(g["s"]), int(g["g"]))
    for j, L in enumerate(h.layers):
        np.testing.assert_array_equal(L.adjacency, g[f"adj{j}"])
        np.testing.assert_array_equal(L.nn_dists, g[f"nnd{j}"])
        np.testing.assert_array_equal(L.sym_count, g[f"sym{j}"])
        np.testing.assert_array_equal(L.d_nn1, g[f"dnn1_{j}"])
        if j:
            np.testing.assert_array_equal(h.to_bottom[j], g[f"tob{j}"])
    assert (h.stats.d_nn1_mean, h.stats.d_nn1_max) == tuple(g["stats"])


def test_save_is_byte_identical_to_reference(tmp_path):
    h = load_index(GOLDEN / "ref_int.idx")
    save_index(h, tmp_path / "x.idx")
    assert (tmp_path / "x.idx").read_bytes() == (GOLDEN / "ref_int.idx").read_bytes()


@pytest.mark.parametrize("how", ["flip", "truncate", "short"])
def test_corruption_detected(tmp_path, how):
    blob = bytearray((GOLDEN / "ref_int.idx").read_bytes())
    if how == "flip":
        blob[100] ^= 0x40
    elif how == "truncate":
        blob = blob[:-50]
    else:
        blob = blob[:10]
    p = tmp_path / "bad.idx"
    p.write_bytes(bytes(blob))
    with pytest.raises(IndexFormatError):
        load_index(p)


def _golden_shards():
    g = load_golden("sharded_int.npz")
    X = load_golden("kernels_int.npz")["X"]
    perm = g["perm"]
    shards = []
    for i, off in enumerate(g["offsets"]):
        sub = {k[len(f"s{i}_"):]: v for k, v in g.items() if k.startswith(f"s{i}_")}
        n_i = sub["adj0"].shape[0]
        shards.append((int(off), golden_hierarchy(sub, X[perm[off:off + n_i]])))
    return g, X, ShardedIndex(shards, int(g["shard_size"]), perm, shards[0][1].config)


def test_sharded_manifest_round_trip(tmp_path):
    g, X, si = _golden_shards()
    save_sharded(si, tmp_path / "sh")
    man = json.loads((tmp_path / "sh" / "manifest.json").read_text())
    assert man["shard_count"] == 3 and man["offsets"] == [int(o) for o in g["offsets"]]
    back = load_sharded(tmp_path / "sh", ga.Dataset(X.copy()))
    np.testing.assert_array_equal(back.permutation, si.permutation)
    for (o1, h1), (o2, h2) in zip(si.shards, back.shards):
        assert o1 == o2
        np.testing.assert_array_equal(h1.layers[0].adjacency, h2.layers[0].adjacency)
        np.testing.assert_array_equal(h1.dataset.vectors, h2.dataset.vectors)


def test_oracle_shard_merge_matches_reference():
    """Per-shard CPU-checker queries + the oracle merge reproduce the
    reference's query_sharded bit for bit (pins oracle.merge_shard_results)."""
    g, X, si = _golden_shards()
    Q = load_golden("kernels_int.npz")["Q"]
    for i, q in enumerate(Q):
        parts = []
        for off, h in si.shards:
            layers = [(L.adjacency, L.k_nn, L.sym_count) for L in h.layers]
            ids, ds, v, t, term, _, _ = O.query(layers, h.to_bottom, h.dataset.vectors, q, 6, 0.6,
                                                h.stats.d_nn1_max)
            parts.append((off, ids, ds, v, t, term))
        gi, gd, v, t, term = O.merge_shard_results(parts, si.permutation, 6)
        nh = len(gi)
        np.testing.assert_array_equal(gi, g["q_ids"][i, :nh])
        np.testing.assert_array_equal(gd, g["q_dists"][i, :nh])
        assert (v, t, term) == tuple(int(c) for c in g["q_cnt"][i])


def test_texmex_io_round_trip_and_reference_bytes(tmp_path):
    """fvecs / bvecs / ivecs files: byte-identical to the reference's writers
    and readable by its readers (when the compiled reference is present)."""
    rng = np.random.default_rng(3)
    X = rng.integers(0, 256, size=(7, 5)).astype(np.float32)
    ids = rng.integers(0, 100, size=(4, 3)).astype(np.int32)
    ga.write_vectors(tmp_path / "a.fvecs", X)
    ga.write_vectors(tmp_path / "a.bvecs", X, fmt="bvecs")
    ga.write_ids(tmp_path / "a.ivecs", ids)
    np.testing.assert_array_equal(ga.load_vectors(tmp_path / "a.fvecs").vectors, X)
    np.testing.assert_array_equal(ga.load_vectors(tmp_path / "a.bvecs", fmt="bvecs").vectors, X)
    np.testing.assert_array_equal(ga.load_ids(tmp_path / "a.ivecs"), ids)
    (tmp_path / "bad.fvecs").write_bytes((tmp_path / "a.fvecs").read_bytes()[:-3])
    with pytest.raises(ga.FormatError):
        ga.load_vectors(tmp_path / "bad.fvecs")
    R = O.reference_module()
    if R is not None:
        R.write_vectors(tmp_path / "r.fvecs", X)
        R.write_vectors(tmp_path / "r.bvecs", X, fmt="bvecs")
        R.write_ids(tmp_path / "r.ivecs", ids)
        for ext in ("fvecs", "bvecs", "ivecs"):
            assert (tmp_path / f"r.{ext}").read_bytes() == (tmp_path / f"a.{ext}").read_bytes()
