"""The reference's OWN Python code running on this package's kernels.

`graphann.backend.impl` is the reference's plugin point (backend.py:17-29,
looked up late by every caller).  Swapping it for paper_1912_01059_b200's
`_gpu_backend` (the `_core` function set on libggnn_b200.so) and running the
unmodified reference functions -- query / batch_query (search.py), build with
its build_base / symmetrize / merge_layer (build.py) -- must give results bit
for bit equal to the same functions on the reference's compiled `_core`, on
integer data (exact distances; test_backends.py:64-95 is the reference's own
version of this check between its two backends).

Needs the compiled reference (oracle/_ref, built by oracle/build_ref.sh; it
travels to the GPU box with the repository snapshot); skipped without it.
"""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    R = O.reference_module()
    if R is None:
        pytest.skip("compiled reference (oracle/_ref) not present")
    assert R.backend.BACKEND == "compiled"
    return R


class _swap:
    """Temporarily point the reference's backend at the GPU kernels."""

    def __init__(self, R):
        from paper_1912_01059_b200 import _gpu_backend

        self.R, self.gpu = R, _gpu_backend

    def __enter__(self):
        self.old = self.R.backend.impl
        self.R.backend.impl = self.gpu
        return self

    def __exit__(self, *exc):
        self.R.backend.impl = self.old


def _fields(r):
    return (r.ids.tolist(), r.dists.tolist(), r.visited_count, r.steps, r.terminated_by, r.distinct_touched,
            r.forgotten)


def test_reference_query_on_gpu_backend(ref):
    R = ref
    g = load_golden("kernels_int.npz")
    X = g["X"]
    from conftest import GOLDEN

    h = R.load_index(GOLDEN / "ref_int.idx").attach(R.Dataset(X.copy()))
    Q = g["Q"]
    for cfg in (R.QueryConfig(k_out=6, tau=0.6), R.QueryConfig(k_out=4, tau=1.5, prioq_size=8, visited_size=5),
                R.QueryConfig(k_out=40, tau=0.8, prioq_size=90)):
        want = [_fields(R.query(h, q, cfg)) for q in Q[:40]]
        with _swap(R):
            got = [_fields(R.query(h, q, cfg)) for q in Q[:40]]
            got_batch = [_fields(r) for r in R.batch_query(h, Q[:40], cfg)]
        assert got == want
        assert got_batch == want


def test_reference_build_on_gpu_backend(ref):
    """The reference's whole build (build_base -> batch_bruteforce, symmetrize
    -> sym_check_pair / SymScratch, merge_layer -> hierarchical_query ->
    exhaustive_topk + greedy_search) with the GPU kernels: every layer's
    adjacency, nn_dists, sym_count and d_nn1 equal the compiled build's."""
    R = ref
    rng = np.random.default_rng(5)
    X = rng.integers(0, 64, size=(160, 12)).astype(np.float32)  # small: every kernel call is one launch
    cfg = R.BuildConfig(k=8, k_nn=4, k_sym=4, s=16, g=2, refinements=1, seed=3)
    h_ref, st_ref = R.build(R.Dataset(X.copy()), cfg)
    with _swap(R):
        h_gpu, st_gpu = R.build(R.Dataset(X.copy()), cfg)
    assert h_gpu.num_layers == h_ref.num_layers
    for a, b in zip(h_gpu.layers, h_ref.layers):
        np.testing.assert_array_equal(a.adjacency, b.adjacency)
        np.testing.assert_array_equal(a.nn_dists, b.nn_dists)
        np.testing.assert_array_equal(a.sym_count, b.sym_count)
        np.testing.assert_array_equal(a.d_nn1, b.d_nn1)
    assert st_gpu.dropped_sym_links == st_ref.dropped_sym_links
    assert h_gpu.stats == h_ref.stats
