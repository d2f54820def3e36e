"""Kernel seam (drop-in for graphann.backend, backend.py:1-58).

The reference selects between a compiled CPU module and a numpy twin.  This
package has exactly one implementation, the sm_100a library behind
`_gpu_backend`; there is no CPU fallback and `use()` accepts only "cuda".
"""

from __future__ import annotations

import contextlib

from . import _gpu_backend

impl = _gpu_backend
BACKEND = "cuda"


def available() -> list[str]:
    return ["cuda"]


@contextlib.contextmanager
def use(name: str):
    """Select the backend for a block of code; only "cuda" exists."""
    if name != "cuda":
        raise ValueError(f"unknown backend {name!r} (this build has only the 'cuda' backend)")
    yield
