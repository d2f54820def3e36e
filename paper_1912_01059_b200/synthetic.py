"""Seeded synthetic datasets of the benchmark shapes (BASELINE.json configs).

Two generators, both integer-valued in [0, 255] so that float32 squared
distances (and the device's lossless uint8 copy) are exact:

* ``make_sift_shaped`` -- the reference test-suite's SIFT stand-in ("G_A"),
  restated from /root/reference/pkg/tests/conftest.py:79-87.
* ``make_latent16``    -- the low-intrinsic-dimension SIFT analogue ("G_B")
  defined in SURVEY.md section 8(d); for n >= 1M rows it is generated in
  chunks of 1M rows with seed (seed, chunk) so that memory stays bounded.
"""

from __future__ import annotations

import numpy as np


def make_sift_shaped(n=10000, d=128, m=100, seed=1234):
    """Integer-valued clustered vectors mimicking SIFT descriptor scale."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(30, 225, size=(64, d))
    assign = rng.integers(0, 64, size=n)
    base = np.clip(np.rint(centers[assign] + rng.normal(0, 12, (n, d))), 0, 255)
    picks = rng.choice(n, size=m, replace=False)
    queries = np.clip(np.rint(base[picks] + rng.normal(0, 12, (m, d))), 0, 255)
    return base.astype(np.float32), queries.astype(np.float32)


def _latent_draw(rng, A, C, k, d, as_float):
    z = C[rng.integers(0, 64, size=k)] + 0.6 * rng.standard_normal((k, 16))
    x = 128.0 + 28.0 * (z @ A) + rng.normal(0, 2, (k, d))
    if as_float:
        return (np.clip(x, 0, 255) / 255.0).astype(np.float32)
    return np.clip(np.rint(x), 0, 255).astype(np.float32)


CHUNK = 1_000_000


def make_latent16(n=10000, d=128, m=1000, seed=1234, as_float=False):
    """G_B ("latent16"): base (n, d) then queries (m, d), float32.

    as_float=True gives the GIST-like float variant (no rint, divided by 255)
    used for the d=960 configuration.
    """
    if n <= CHUNK:
        rng = np.random.default_rng(seed)
        A = rng.standard_normal((16, d)) / 4.0
        C = rng.standard_normal((64, 16)) * 2.0
        base = _latent_draw(rng, A, C, n, d, as_float)
        queries = _latent_draw(rng, A, C, m, d, as_float)
        return base, queries
    # chunked canonical stream: shared (A, C) from `seed`, rows from (seed, chunk)
    rng0 = np.random.default_rng(seed)
    A = rng0.standard_normal((16, d)) / 4.0
    C = rng0.standard_normal((64, 16)) * 2.0
    base = np.empty((n, d), dtype=np.float32)
    for c, lo in enumerate(range(0, n, CHUNK)):
        hi = min(n, lo + CHUNK)
        rng = np.random.default_rng((seed, c))
        base[lo:hi] = _latent_draw(rng, A, C, hi - lo, d, as_float)
    rngq = np.random.default_rng((seed, 0x51E7))
    queries = _latent_draw(rngq, A, C, m, d, as_float)
    return base, queries


def make_latent16_shard(n=1_000_000, d=128, shard=0, seed=1234, as_float=False):
    """Base rows of shard `shard` of a multi-million-point latent16 index
    (bench.py --gpus N): shard 0 is exactly make_latent16(n, d)'s base (the
    C2 data), shard s > 0 draws n further rows of the same distribution (the
    shared (A, C) of `seed`) from the stream (seed, 0x5AD, s)."""
    if shard == 0:
        return make_latent16(n=n, d=d, m=1, seed=seed, as_float=as_float)[0]
    rng0 = np.random.default_rng(seed)
    A = rng0.standard_normal((16, d)) / 4.0
    C = rng0.standard_normal((64, 16)) * 2.0
    out = np.empty((n, d), dtype=np.float32)
    for c, lo in enumerate(range(0, n, CHUNK)):
        hi = min(n, lo + CHUNK)
        out[lo:hi] = _latent_draw(np.random.default_rng((seed, 0x5AD, shard, c)), A, C, hi - lo, d, as_float)
    return out


def make_latent16_queries(m=10000, d=128, batch=1, seed=1234, as_float=False):
    """Query batch `batch` >= 1 of the latent16 workload: m further rows of the
    same distribution (the shared (A, C) of `seed`) from the stream
    (seed, 0x9E57, batch).  Batch 0 is the query set make_latent16 returns
    (bench.py: a fresh batch every step)."""
    rng0 = np.random.default_rng(seed)
    A = rng0.standard_normal((16, d)) / 4.0
    C = rng0.standard_normal((64, 16)) * 2.0
    return _latent_draw(np.random.default_rng((seed, 0x9E57, batch)), A, C, m, d, as_float)


def make_deep_like(n, m, d=96, seed=1234, clusters=1024):
    """C4 (Deep10M-shaped): the reference's clustered generator (data.py:163-192,
    `clusters` Gaussian centres) with rows L2-normalised; base = the first n
    rows, queries = the m rows held out after them."""
    from .data import gen_synthetic

    X = gen_synthetic(n + m, d, seed=seed, law="clustered", clusters=clusters).vectors.astype(np.float64)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X = X.astype(np.float32)
    return X[:n].copy(), X[n:].copy()


def make_deep_like_queries(m, d=96, batch=1, seed=1234, clusters=1024):
    """Query batch `batch` >= 1 of the C4 workload: rows around the same
    cluster centres (the generator's first draw from `seed`), drawn from the
    stream (seed, 0xDEE9, batch), L2-normalised."""
    centers = np.random.default_rng(seed).standard_normal((clusters, d)) * 5.0
    rng = np.random.default_rng((seed, 0xDEE9, batch))
    X = centers[rng.integers(0, clusters, size=m)] + rng.standard_normal((m, d)) * 0.25
    X = X.astype(np.float32).astype(np.float64)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    return X.astype(np.float32)
