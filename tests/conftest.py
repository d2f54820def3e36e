"""Shared fixtures.

* `gpu` marker: tests that need a CUDA device (the driver runs them on a B200).
* Golden fixtures (tests/golden/*.npz) are produced by the UNMODIFIED
  reference via tests/golden/make_golden.py; `golden_hierarchy` rebuilds the
  reference's graph as a drop-in Hierarchy so the same graph can be queried by
  the GPU path ("same graph" parity).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

import paper_1912_01059_b200 as ga  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
TERM_CODE = {"stopping-rule": 0, "queue-empty": 1, "iteration-cap": 2}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on a B200 via gpurun)")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_hierarchy(g: dict, X: np.ndarray) -> "ga.Hierarchy":
    """The reference-built graph stored in a golden fixture as a Hierarchy."""
    k, k_nn, k_sym, s, gg, refinements, seed = (int(v) for v in g["config"])
    cfg = ga.BuildConfig(k=k, k_nn=k_nn, k_sym=k_sym, s=s, g=gg, refinements=refinements,
                         tau_build=float(g["tau_build"]), seed=seed)
    layers, to_bottom = [], [None]
    for j in range(int(g["num_layers"])):
        adj = g[f"adj{j}"]
        layer = ga.AdjacencyLayer(adj.shape[0], k, k_nn)
        layer.adjacency[:] = adj
        if f"nnd{j}" in g:
            layer.nn_dists[:] = g[f"nnd{j}"]
        layer.sym_count[:] = g[f"sym{j}"]
        layer.d_nn1[:] = g[f"dnn1_{j}"]
        layers.append(layer)
        if j:
            to_bottom.append(g[f"tob{j}"].astype(np.int32))
    stats = ga.GraphStats(float(g["stats"][0]), float(g["stats"][1]))
    h = ga.Hierarchy(layers, to_bottom, s, gg, cfg, stats, dim=X.shape[1])
    h.attach(ga.Dataset(np.ascontiguousarray(X, dtype=np.float32).copy()))
    return h


def oracle_layers(h):
    return [(L.adjacency, L.k_nn, L.sym_count) for L in h.layers]


@pytest.fixture(scope="session")
def golden_int():
    g = load_golden("kernels_int.npz")
    return g, golden_hierarchy(g, g["X"])


@pytest.fixture(scope="session")
def golden_float():
    g = load_golden("float_small.npz")
    return g, golden_hierarchy(g, g["X"])


@pytest.fixture(scope="session")
def golden_sift():
    from paper_1912_01059_b200.synthetic import make_sift_shaped
    import hashlib

    g = load_golden("sift10k.npz")
    base, queries = make_sift_shaped()
    sha = hashlib.sha256(base.tobytes() + queries.tobytes()).hexdigest()
    assert sha == str(g["data_sha256"]), "make_sift_shaped no longer reproduces the golden data"
    return g, golden_hierarchy(g, base), queries
