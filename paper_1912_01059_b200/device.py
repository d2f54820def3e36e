"""Device mirrors of datasets and hierarchies (HBM layout).

DeviceVectors   one (n, d) table per dataset and device: uint8 when every value
                is an integer in [0, 255] (lossless; distances stay exact and
                4x fewer bytes are gathered), float32 otherwise.
DeviceHierarchy per layer: the sanitized adjacency (slots the reference would
                skip set to -1), to_row (layer-local id -> dataset row), the
                down map (layer-local id -> local id one layer finer), the
                layer's slack bound, plus the top layer's rows and d_nn1_max.
"""

from __future__ import annotations

import weakref
import zlib

import numpy as np

from . import _native as N

_ARRAY_CACHE: dict = {}

# Host-resident hierarchies up to this many adjacency bytes are content-hashed
# on every device_hierarchy() call, so the reference's tests that write layer
# arrays in place (SURVEY 8b "host-object coherence") see their writes without
# a touch(); the hash costs well under a millisecond at this size.  Larger
# hierarchies are re-uploaded only on a version bump: after writing their
# numpy arrays directly call layer.touch() or Hierarchy.invalidate_caches().
_HASH_LIMIT = 1 << 20


class DeviceVectors:
    def __init__(self, dataset):
        t = N.torch()
        X = dataset.vectors if hasattr(dataset, "vectors") else np.ascontiguousarray(dataset, dtype=np.float32)
        self.n, self.d = X.shape
        f32 = N.to_dev(X)
        flag = t.ones(1, dtype=t.int32, device=f32.device)
        u8 = t.empty((self.n, self.d), dtype=t.uint8, device=f32.device)
        N.call("ggnn_f32_to_u8", N.ptr(f32), self.n * self.d, N.ptr(u8), N.ptr(flag), N.stream_ptr())
        if int(flag.item()) == 1:
            self.data, self.dtype = u8, N.GGNN_U8
            del f32
        else:
            self.data, self.dtype = f32, N.GGNN_F32
            del u8
        self.struct = N.vectors_struct(self.data, self.dtype)

    @property
    def exact_integers(self) -> bool:
        return self.dtype == N.GGNN_U8

    @classmethod
    def of(cls, dataset) -> "DeviceVectors":
        key = N.torch().cuda.current_device()
        dv = dataset._device.get(key)
        if dv is None:
            dv = cls(dataset)
            dataset._device[key] = dv
        return dv

    @classmethod
    def of_array(cls, X: np.ndarray) -> "DeviceVectors":
        """Device copy of a bare (n, d) array; cached while the array object is
        alive and read-only (Dataset vectors are)."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        if X.flags.writeable:
            return cls(X)
        key = (X.__array_interface__["data"][0], X.shape, N.torch().cuda.current_device())
        hit = _ARRAY_CACHE.get(key)
        if hit is not None and hit[0]() is X:
            return hit[1]
        dv = cls(X)
        if len(_ARRAY_CACHE) > 64:
            _ARRAY_CACHE.clear()
        _ARRAY_CACHE[key] = (weakref.ref(X), dv)
        return dv

    def queries(self, Q: np.ndarray):
        """Upload a (m, d) float32 query table; integral queries against a
        uint8 table are searched as uint8 (exact integer distances).  The
        check and the narrowing run on the device (ggnn_f32_to_u8): one
        float upload instead of a host-side scan of every value."""
        Q = np.ascontiguousarray(Q, dtype=np.float32)
        if Q.ndim != 2 or Q.shape[1] != self.d:
            raise ValueError(f"query shape {Q.shape} does not match index dimension {self.d}")
        dq = N.to_dev(Q)
        if self.dtype == N.GGNN_U8 and Q.size:
            t = N.torch()
            u8 = t.empty(Q.shape, dtype=t.uint8, device=dq.device)
            flag = t.ones(1, dtype=t.int32, device=dq.device)
            N.call("ggnn_f32_to_u8", N.ptr(dq), Q.size, N.ptr(u8), N.ptr(flag), N.stream_ptr())
            if int(flag.item()) == 1:
                return u8, N.queries_struct(data=u8, dtype_code=N.GGNN_U8)
        return dq, N.queries_struct(data=dq, dtype_code=N.GGNN_F32)


class DeviceLayer:
    __slots__ = ("adj", "to_row", "down", "node_count", "k", "k_nn", "slack", "struct")

    def __init__(self, adj, to_row, down, node_count, k, k_nn, slack):
        self.adj, self.to_row, self.down = adj, to_row, down
        self.node_count, self.k, self.k_nn, self.slack = int(node_count), int(k), int(k_nn), float(slack)
        self.struct = N.Layer(N.ptr(adj), N.ptr(to_row), N.ptr(down), self.node_count, self.k, self.k_nn,
                              self.slack)


def sanitize(adj_dev, symc_dev, node_count, k, k_nn):
    out = N.empty((node_count, k), N.torch().int32)
    N.call("ggnn_sanitize_layer", N.ptr(adj_dev), N.ptr(symc_dev), node_count, k, k_nn, N.ptr(out), N.stream_ptr())
    return out


def down_maps(to_bottom, n):
    """down[j][i] = local id in layer j-1 of node i of layer j (host numpy)."""
    out = [None]
    for j in range(1, len(to_bottom)):
        t = np.asarray(to_bottom[j], dtype=np.int32)
        if j == 1:
            out.append(t)
        else:
            inv = np.full(n, -1, dtype=np.int32)
            finer = np.asarray(to_bottom[j - 1], dtype=np.int32)
            inv[finer] = np.arange(len(finer), dtype=np.int32)
            out.append(inv[t])
    return out


class DeviceHierarchy:
    def __init__(self, h, slack_bounds=None):
        self.vectors = DeviceVectors.of(h.dataset)
        self.num_layers = h.num_layers
        downs = down_maps(h.to_bottom, h.n)
        self.layers = []
        for j, layer in enumerate(h.layers):
            dev = layer.device_arrays()
            if dev is not None:
                adj, symc = dev["adj"], dev["symc"]
            else:
                adj, symc = N.to_dev(layer.adjacency), N.to_dev(layer.sym_count)
            san = sanitize(adj, symc, layer.node_count, layer.k, layer.k_nn)
            to_row = None if j == 0 else N.to_dev(np.asarray(h.to_bottom[j], dtype=np.int32))
            down = None if j == 0 else N.to_dev(downs[j])
            slack = slack_bounds[j] if slack_bounds is not None else layer.live_d_nn1_max()
            self.layers.append(DeviceLayer(san, to_row, down, layer.node_count, layer.k, layer.k_nn, slack))
        top = self.layers[-1]
        self.top_rows = top.to_row  # None -> identity (single-layer hierarchy)
        self.ntop = top.node_count
        self.d_nn1_max = h.stats.d_nn1_max if h.stats is not None else self.layers[0].slack

    def layer_array(self):
        arr = (N.Layer * len(self.layers))()
        for j, L in enumerate(self.layers):
            arr[j] = L.struct
        return arr


def _token(h):
    parts = [id(h.dataset), h.num_layers, None if h.stats is None else (h.stats.d_nn1_max,)]
    total = sum(layer.node_count * layer.k * 4 for layer in h.layers)
    small = total <= _HASH_LIMIT
    for j, layer in enumerate(h.layers):
        parts.append((id(layer), layer._version, layer.device_authoritative))
        if small and not layer.device_authoritative:
            parts.append(zlib.crc32(layer.adjacency.tobytes()))
            parts.append(zlib.crc32(layer.sym_count.tobytes()))
            parts.append(zlib.crc32(layer.d_nn1.tobytes()))
        t = h.to_bottom[j]
        if t is not None:
            parts.append((id(t), len(t), zlib.crc32(np.ascontiguousarray(t).tobytes()) if small else 0))
    return tuple(parts)


def device_hierarchy(h) -> DeviceHierarchy:
    """The (cached) device mirror of `h`, rebuilt when `h` changed."""
    if h.dataset is None:
        raise RuntimeError("no dataset attached; call attach() after loading an index")
    tok = _token(h)
    cache = h._device_cache
    if cache is not None and cache[0] == tok:
        return cache[1]
    if all(L.device_authoritative and "rows_q" in L._dev for L in h.layers):
        from ._devgraph import device_hierarchy_from_build

        dh = device_hierarchy_from_build(h)  # layers already in searchable device form
    else:
        dh = DeviceHierarchy(h)
    h._device_cache = (tok, dh)
    return dh
