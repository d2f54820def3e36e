"""Device state of a hierarchy under construction.

Every layer of a Hierarchy being built or refined is device-authoritative:
its dev dict holds
    adj  (nc, k)    int32   -1 = empty slot; direct slots are a prefix and
                            inverse slots beyond sym_count are -1, so the
                            array is directly searchable (no sanitize pass)
    nnd  (nc, k_nn) float64 direct-slot distances (+inf = empty)
    symc (nc,)      int32   used inverse slots
    dnn1 (nc,)      float64 first-neighbour distance (+inf = none)
    to_row (nc,)    int32   dataset rows (absent for the bottom layer)
    down (nc,)      int32   local ids one layer finer (absent for the bottom)
    rows_q (nc,)    int32   rows used as self queries (arange at the bottom)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .device import DeviceHierarchy, DeviceLayer, DeviceVectors

INT32_MAX = 2**31 - 1


def new_layer_dev(nc: int, k: int, k_nn: int) -> dict:
    t = N.torch()
    dev = N.device()
    return {
        "adj": t.full((nc, k), -1, dtype=t.int32, device=dev),
        "nnd": t.full((nc, k_nn), float("inf"), dtype=t.float64, device=dev),
        "symc": t.zeros((nc,), dtype=t.int32, device=dev),
        "dnn1": t.full((nc,), float("inf"), dtype=t.float64, device=dev),
    }


def ensure_device(h) -> None:
    """Make every layer of `h` device-authoritative (uploading host arrays),
    and attach translation arrays."""
    from .device import down_maps

    t = N.torch()
    downs = None
    for j, layer in enumerate(h.layers):
        dev = layer.device_arrays()
        if dev is None:
            dev = {
                "adj": _sanitized_upload(layer),
                "nnd": N.to_dev(layer.nn_dists),
                "symc": N.to_dev(layer.sym_count),
                "dnn1": N.to_dev(layer.d_nn1),
            }
            layer._dev = dev
            layer._host = None
            layer._version += 1
        if j == 0:
            if "rows_q" not in dev:
                dev["rows_q"] = t.arange(layer.node_count, dtype=t.int32, device=N.device())
        elif "to_row" not in dev or "down" not in dev:
            if downs is None:
                downs = down_maps(h.to_bottom, h.n)
            dev["to_row"] = N.to_dev(np.asarray(h.to_bottom[j], dtype=np.int32))
            dev["down"] = N.to_dev(downs[j])
            dev["rows_q"] = dev["to_row"]


def _sanitized_upload(layer):
    from .device import sanitize

    adj = N.to_dev(layer.adjacency)
    symc = N.to_dev(layer.sym_count)
    return sanitize(adj, symc, layer.node_count, layer.k, layer.k_nn)


class Workspace:
    """Scratch buffers reused across the passes of one build."""

    def __init__(self, n: int):
        t = N.torch()
        dev = N.device()
        self.stats_scratch = t.empty((int(N.load().ggnn_layer_stats_scratch_bytes()) // 8,), dtype=t.float64,
                                     device=dev)
        self.stats_out = t.empty((4,), dtype=t.float64, device=dev)
        self.best = t.full((n,), INT32_MAX, dtype=t.int32, device=dev)
        self.first = t.full((n,), INT32_MAX, dtype=t.int32, device=dev)
        self.req_cap = 0
        self.req = self.stage = self.tgt = None
        self.req_count = t.zeros((1,), dtype=t.int32, device=dev)
        self.dropped = t.zeros((1,), dtype=t.int32, device=dev)
        self.reduced = t.zeros((1,), dtype=t.int32, device=dev)
        self.pending = t.zeros((1,), dtype=t.int32, device=dev)
        self.n_open = t.zeros((1,), dtype=t.int32, device=dev)

    def ensure_requests(self, cap: int, n_fallback: int):
        if cap > self.req_cap:
            t = N.torch()
            dev = N.device()
            self.req_cap = cap
            self.req = t.empty((cap, 5 + n_fallback), dtype=t.int32, device=dev)
            self.stage = t.empty((cap,), dtype=t.int32, device=dev)
            self.tgt = t.empty((cap,), dtype=t.int32, device=dev)
            self.open_idx = (t.empty((cap,), dtype=t.int32, device=dev), t.empty((cap,), dtype=t.int32, device=dev))

    def stats(self, values) -> tuple[float, float, int, int]:
        N.call("ggnn_layer_stats", N.ptr(values), values.numel(), N.ptr(self.stats_scratch), N.ptr(self.stats_out),
               N.stream_ptr())
        mx, s, cnt, bad = self.stats_out.cpu().tolist()
        return mx, s, int(cnt), int(bad)


def workspace(h) -> Workspace:
    ws = getattr(h, "_gpu_ws", None)
    if ws is None or ws.best.numel() < h.n:
        ws = Workspace(h.n)
        h._gpu_ws = ws
    return ws


def layer_struct(layer, slack: float) -> N.Layer:
    dev = layer._dev
    return N.Layer(N.ptr(dev["adj"]), N.ptr(dev.get("to_row")), N.ptr(dev.get("down")), layer.node_count, layer.k,
                   layer.k_nn, float(slack))


def live_max(h, layer) -> float:
    """live_d_nn1_max (graph.py:196-199) of a device layer."""
    return workspace(h).stats(layer._dev["dnn1"])[0]


def device_hierarchy_from_build(h) -> DeviceHierarchy:
    """DeviceHierarchy view of a device-authoritative hierarchy (no copies)."""
    dh = DeviceHierarchy.__new__(DeviceHierarchy)
    dh.vectors = DeviceVectors.of(h.dataset)
    dh.num_layers = h.num_layers
    dh.layers = []
    for j, layer in enumerate(h.layers):
        dev = layer._dev
        slack = h.stats.d_nn1_max if (j == 0 and h.stats is not None) else live_max(h, layer)
        dh.layers.append(DeviceLayer(dev["adj"], dev.get("to_row"), dev.get("down"), layer.node_count, layer.k,
                                     layer.k_nn, slack))
    top = dh.layers[-1]
    dh.top_rows = top.to_row
    dh.ntop = top.node_count
    dh.d_nn1_max = h.stats.d_nn1_max if h.stats is not None else dh.layers[0].slack
    return dh


def structs_array(structs):
    arr = (N.Layer * len(structs))()
    for j, s in enumerate(structs):
        arr[j] = s
    return arr


__all__ = ["ctypes", "ensure_device", "new_layer_dev", "workspace", "layer_struct", "live_max",
           "device_hierarchy_from_build", "structs_array"]
