"""Vector containers, the L2 distance helper and synthetic datasets.

`Dataset` follows graphann.data.Dataset (data.py:29-63): float32, C-contiguous,
finite, read-only.  Its device copy is created lazily (see device.py) and is a
lossless uint8 table when every value is an integer in [0, 255].
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np


class FormatError(ValueError):
    """Malformed vector / id / index files."""


class ConfigError(ValueError):
    """Invalid configuration values."""


@dataclass(frozen=True)
class Dataset:
    vectors: np.ndarray
    _device: dict = field(default_factory=dict, compare=False, repr=False)

    def __post_init__(self):
        v = self.vectors
        if v.ndim != 2 or v.shape[0] < 1 or v.shape[1] < 1:
            raise ValueError(f"expected a non-empty 2-D array, got shape {v.shape}")
        if v.dtype != np.float32:
            raise ValueError(f"expected float32 vectors, got {v.dtype}")
        if not v.flags["C_CONTIGUOUS"]:
            raise ValueError("vectors must be C-contiguous")
        finite = np.isfinite(v).all(axis=1)
        if not finite.all():
            raise ValueError(f"non-finite value in vector {int(np.argmin(finite))}")
        v.setflags(write=False)

    @property
    def n(self) -> int:
        return self.vectors.shape[0]

    @property
    def d(self) -> int:
        return self.vectors.shape[1]

    def content_hash(self) -> str:
        return hashlib.sha256(self.vectors.tobytes()).hexdigest()[:16]


def squared_distance(a: np.ndarray, b: np.ndarray) -> float:
    """Squared L2 distance, float32 inputs with sequential float64
    accumulation (the reference's _sqdist, _core.pyx:30-37), evaluated on the
    GPU by ggnn_squared_l2_many."""
    from . import backend

    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    return float(backend.impl.squared_l2(a, b))


def gen_synthetic(n: int, d: int, seed: int, law: str = "uniform", clusters: int = 8) -> Dataset:
    """Seeded synthetic data with the reference's generator laws
    (data.py:163-192): uniform U[0,1), gaussian N(0,1), or `clusters`
    Gaussian centres (scale 5) with N(0, 0.25^2) spread."""
    if n < 1 or d < 1:
        raise ValueError(f"n and d must be >= 1, got n={n} d={d}")
    rng = np.random.default_rng(seed)
    if law == "uniform":
        arr = rng.random((n, d), dtype=np.float32)
    elif law == "gaussian":
        arr = rng.standard_normal((n, d)).astype(np.float32)
    elif law == "clustered":
        if clusters < 1:
            raise ValueError("clustered law needs clusters >= 1")
        centers = rng.standard_normal((clusters, d)) * 5.0
        assign = rng.integers(0, clusters, size=n)
        arr = (centers[assign] + rng.standard_normal((n, d)) * 0.25).astype(np.float32)
    else:
        raise ValueError(f"unknown law {law!r}")
    return Dataset(arr)


# ------------------------------------------------------------- TexMex files
# fvecs / bvecs / ivecs: every record is a little-endian int32 dimension
# followed by that many float32 / uint8 / int32 values (data.py:80-160 in the
# reference).  Host utilities: parsed with one reshape of the raw bytes.
_ELEM = {"fvecs": np.dtype("<f4"), "bvecs": np.dtype("u1"), "ivecs": np.dtype("<i4")}


def _records(path, kind: str) -> np.ndarray:
    raw = np.fromfile(path, dtype=np.uint8)
    if raw.size < 4:
        raise FormatError(f"{path}: no records (file has {raw.size} bytes)")
    d = int(raw[:4].view("<i4")[0])
    if d <= 0:
        raise FormatError(f"{path}: invalid dimension {d} at byte offset 0")
    esz = _ELEM[kind].itemsize
    rec = 4 + d * esz
    n, tail = divmod(raw.size, rec)
    if tail:
        raise FormatError(f"{path}: truncated {kind} file, {tail} trailing bytes after {n} records of {rec} bytes "
                          f"(byte offset {n * rec})")
    table = raw.reshape(n, rec)
    dims = np.ascontiguousarray(table[:, :4]).view("<i4").ravel()
    if (dims != d).any():
        bad = int(np.argmax(dims != d))
        raise FormatError(f"{path}: inconsistent dimension, record {bad} claims {int(dims[bad])} (expected {d}, "
                          f"byte offset {bad * rec})")
    return np.ascontiguousarray(table[:, 4:]).view(_ELEM[kind]).reshape(n, d)


def load_vectors(path, fmt: str = "fvecs") -> Dataset:
    """fvecs or bvecs file -> Dataset (bvecs bytes promoted to float32)."""
    if fmt not in ("fvecs", "bvecs"):
        raise ValueError(f"unknown vector format {fmt!r} (expected 'fvecs' or 'bvecs')")
    arr = _records(path, fmt).astype(np.float32)
    if fmt == "fvecs":
        finite = np.isfinite(arr).all(axis=1)
        if not finite.all():
            raise FormatError(f"{path}: non-finite value in record {int(np.argmin(finite))}")
    return Dataset(arr)


def load_ids(path) -> np.ndarray:
    """ivecs id table -> (m, k) int32."""
    arr = _records(path, "ivecs").astype(np.int32)
    if (arr < 0).any():
        r, c = np.argwhere(arr < 0)[0]
        raise FormatError(f"{path}: negative index {int(arr[r, c])} in record {int(r)}")
    return arr


def _write(path, body: np.ndarray, kind: str) -> None:
    n, d = body.shape
    out = np.empty((n, 4 + d * _ELEM[kind].itemsize), dtype=np.uint8)
    out[:, :4] = np.full((n, 1), d, dtype="<i4").view(np.uint8)
    out[:, 4:] = np.ascontiguousarray(body.astype(_ELEM[kind])).view(np.uint8).reshape(n, -1)
    out.tofile(path)


def write_vectors(path, vectors: np.ndarray, fmt: str = "fvecs") -> None:
    if fmt not in ("fvecs", "bvecs"):
        raise ValueError(f"unknown vector format {fmt!r}")
    _write(path, np.asarray(vectors), fmt)


def write_ids(path, ids: np.ndarray) -> None:
    _write(path, np.asarray(ids), "ivecs")
