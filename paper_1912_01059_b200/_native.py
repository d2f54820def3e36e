"""ctypes binding of libggnn_b200.so (include/ggnn_b200.h).

torch is used only as the device allocator and stream provider: tensors are
passed to the C ABI as raw device pointers.  There is no fallback -- if the
library is missing or no CUDA device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
# GGNN_LIB overrides the library path (A/B experiments with alternative builds)
LIB_PATH = Path(__import__("os").environ.get("GGNN_LIB", PKG / "libggnn_b200.so"))

GGNN_F32 = 0
GGNN_U8 = 1
FLAG_DISTINCT = 1
FLAG_EXACT_DISTS = 2
FLAG_UNIQUE_ROWS = 4

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double


class Vectors(ctypes.Structure):
    _fields_ = [("d_data", P), ("n", I64), ("d", I32), ("dtype", I32)]


class Queries(ctypes.Structure):
    _fields_ = [("d_data", P), ("d_rows", P), ("m", I64), ("dtype", I32), ("pad_", I32)]


class Layer(ctypes.Structure):
    _fields_ = [("d_adj", P), ("d_to_row", P), ("d_down", P), ("node_count", I64), ("k", I32), ("k_nn", I32),
                ("slack", F64)]


class SearchParams(ctypes.Structure):
    _fields_ = [("k_out", I32), ("prioq_size", I32), ("visited_size", I32), ("flags", I32), ("tau", F64),
                ("max_iterations", I64)]


class Push(ctypes.Structure):  # ggnn_push (include/ggnn_p2p.h)
    _fields_ = [("d_peers", P * 8), ("nranks", I32), ("rank", I32), ("parity", I32), ("pad_", I32),
                ("d_gid_of_local", P), ("gid_size", I64)]


class NativeError(RuntimeError):
    pass


_lib = None

# name -> argtypes (restype is int unless listed in _RESTYPES)
_SIGS = {
    "ggnn_last_error": [],
    "ggnn_version": [],
    "ggnn_device_info": [P, P],
    "ggnn_search_workspace_bytes": [I64, P, I32],
    "ggnn_sanitize_layer": [P, P, I64, I32, I32, P, P],
    "ggnn_rows_unique": [P, I64, I32, P, P],
    "ggnn_query_batch": [P, P, P, I64, P, P, F64, P, P, P, P, ctypes.c_size_t, P],
    "ggnn_greedy_batch": [P, P, P, P, P, I32, P, F64, P, P, P, P, ctypes.c_size_t, P],
    "ggnn_descent_batch": [P, P, I32, I32, I32, P, P, P, P, P, P, P, P, ctypes.c_size_t, P],
    "ggnn_sym_check_batch": [P, P, P, P, P, I64, F64, F64, I32, I32, I32, I32, I32, P, P, P],
    "ggnn_exhaustive_topk": [P, P, I64, P, I32, P, P, P],
    "ggnn_exhaustive_topk_tc": [P, P, I32, P, P, P],
    "ggnn_bf_timeouts": [],
    "ggnn_squared_l2_many": [P, P, P, I32, P, P],
    "ggnn_f32_to_u8": [P, I64, P, P, P],
    "ggnn_leaf_knn": [P, P, P, P, I64, I64, I32, P, P, P, I32, P, P, P, P],
    "ggnn_leaf_knn_tc": [P, P, P, P, I64, I64, I32, P, P, P, I32, P, P, P, P],
    "ggnn_tc_timeouts": [],
    "ggnn_search_accounting": [P],
    "ggnn_query_schedule": [I64, F64],
    "ggnn_kernel_launches": [],
    "ggnn_query_schedule_large": [F64],
    "ggnn_merge_descent": [P, P, I32, I32, I32, P, I64, P, I32, I32, P, P, P, P, P],
    "ggnn_merge_rows": [I64, I32, I32, P, P, P, P, P, P, I32, P, P, P, P],
    "ggnn_merge_rows_range": [I64, I64, I32, I32, P, P, P, P, P, P, I32, P, P, P, P],
    "ggnn_sym_check_layer": [P, P, P, P, P, I32, F64, F64, I32, I32, I32, I32, I32, P, P, I64, P],
    "ggnn_sym_claim_round": [P, I64, I32, P, P, I32, I32, P, P, P, P, P, I32, P, P, P],
    "ggnn_sym_compact": [P, P, I64, P, P, P],
    "ggnn_sym_recheck": [P, P, P, I64, P, I32, F64, F64, I32, I32, I32, I32, I32, P, P],
    "ggnn_layer_stats": [P, I64, P, P, P],
    "ggnn_layer_stats_scratch_bytes": [],
    "ggnn_shard_block_bytes": [I64, I32],
    "ggnn_shard_block_dists_offset": [I64, I32],
    "ggnn_shard_block_counters_offset": [I64, I32],
    "ggnn_shard_globalize": [P, I64, P, I64, P],
    "ggnn_shard_merge": [P, I32, I64, I32, I32, P, P, P, P],
    "ggnn_p2p_bytes": [I32, I64, I32],
    "ggnn_p2p_alloc": [ctypes.c_size_t, P, P],
    "ggnn_p2p_open": [P, P],
    "ggnn_p2p_close": [P],
    "ggnn_p2p_free": [P],
    "ggnn_query_batch_push": [P, P, P, I64, P, P, F64, P, P, P, P, P],
    "ggnn_p2p_signal": [P, I64, I32, ctypes.c_uint32, P],
    "ggnn_shard_merge_wait": [P, I32, ctypes.c_uint32, I32, I64, I32, I32, P, P, P, P, P],
    "ggnn_query_batch_staged": [P, P, P, I64, P, I64, P, F64, P, I64, ctypes.c_uint32, I32, P, P, P, P, P],
    "ggnn_query_batch_host": [P, P, P, I64, P, I64, P, F64, P, P, P, I32, I32, P, P, P, P, P, P, P, P, P, P],
}
_RESTYPES = {"ggnn_last_error": ctypes.c_char_p, "ggnn_search_workspace_bytes": ctypes.c_size_t,
             "ggnn_layer_stats_scratch_bytes": ctypes.c_size_t, "ggnn_shard_block_bytes": ctypes.c_size_t,
             "ggnn_shard_block_dists_offset": ctypes.c_size_t, "ggnn_shard_block_counters_offset": ctypes.c_size_t,
             "ggnn_p2p_bytes": ctypes.c_size_t, "ggnn_kernel_launches": ctypes.c_ulonglong}
# entry points added by later translation units register themselves here
EXTRA_SIGS: dict = {}


def exported_symbols() -> list[str]:
    return sorted(list(_SIGS) + list(EXTRA_SIGS))


def load(require_gpu: bool = True):
    """Load the library (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeError(
            f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, args in {**_SIGS, **EXTRA_SIGS}.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().ggnn_last_error()
        msg = msg.decode() if msg else ""
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    check(rc, name)


# Tensor-core kernels bound their mbarrier waits (a lost MMA completion must
# not hang the GPU) and count the timeouts in a device counter instead;
# callers of those kernels check the counter after their results are on the
# host, so a stalled MMA raises instead of returning garbage lists.
_TC_SEEN: dict = {}


def check_tc_timeouts(which: str = "both") -> None:
    """Raise NativeError if a tensor-core kernel (leaf kNN: ggnn_tc_timeouts,
    brute force: ggnn_bf_timeouts) timed out since the last check on this
    device.  Reading the counters synchronises the device."""
    names = {"leaf": ("ggnn_tc_timeouts",), "bf": ("ggnn_bf_timeouts",),
             "both": ("ggnn_tc_timeouts", "ggnn_bf_timeouts")}[which]
    dev = torch().cuda.current_device()
    for name in names:
        v = int(getattr(load(), name)())
        if v < 0:
            raise NativeError(f"{name}: reading the device counter failed")
        seen = _TC_SEEN.get((name, dev), 0)
        if v != seen:
            _TC_SEEN[(name, dev)] = v
            raise NativeError(f"{name}: {v - seen} tensor-core MMA wait(s) timed out; results are invalid")


# ---------------------------------------------------------------- torch glue
_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        if not t.cuda.is_available():
            raise NativeError("no CUDA device visible: the GGNN B200 path has no CPU fallback")
        _torch = t
    return _torch


def device():
    return torch().device("cuda", torch().cuda.current_device())


def stream_ptr():
    return P(torch().cuda.current_stream().cuda_stream)


def ptr(t) -> P:
    return P(0) if t is None else P(t.data_ptr())


def to_dev(a: np.ndarray, dtype=None):
    import warnings

    t = torch()
    arr = np.ascontiguousarray(a if dtype is None else a.astype(dtype, copy=False))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # read-only arrays are only read
        return t.from_numpy(arr).to(device(), non_blocking=False)


def empty(shape, dtype):
    return torch().empty(shape, dtype=dtype, device=device())


def vectors_struct(data, dtype_code: int) -> Vectors:
    n, d = data.shape
    return Vectors(ptr(data), n, d, dtype_code)


def queries_struct(data=None, rows=None, dtype_code: int = GGNN_F32, m: int | None = None) -> Queries:
    if m is None:
        m = rows.shape[0] if rows is not None else data.shape[0]
    return Queries(ptr(data), ptr(rows), m, dtype_code, 0)


def search_params(k_out, prioq_size, visited_size, tau, max_iterations, flags=0) -> SearchParams:
    return SearchParams(int(k_out), int(prioq_size), int(visited_size), int(flags), float(tau), int(max_iterations))
