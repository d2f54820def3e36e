"""Kernel time vs batch size on the C2 workload: single-warp step latency at
low load and how much of a 10k batch is drain (tools/latency_probe.py)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import _native as N  # noqa: E402
from paper_1912_01059_b200.device import device_hierarchy  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

import os  # noqa: E402

# FLOAT=1: the sift1m-f32 workload (non-integer float32 rows); D: dimension
base, Q = make_latent16(n=1_000_000, d=int(os.environ.get("D", 128)), m=10_000, seed=1234,
                        as_float=os.environ.get("FLOAT") == "1")
import time  # noqa: E402

ga.build(ga.Dataset(base[:50_000]), ga.BuildConfig(seed=7))  # warm-up (module loading, allocator growth)
t0 = time.perf_counter()
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
print(f"build {time.perf_counter() - t0:.2f} s", flush=True)
dh = device_hierarchy(h)
dv = dh.vectors
tau = float(sys.argv[1]) if len(sys.argv) > 1 else 0.6
import os  # noqa: E402

from paper_1912_01059_b200 import search as S  # noqa: E402

qflags = 0 if os.environ.get("GGNN_NO_UNIQUE") else S._qflags(dh, False)
print("flags", qflags)
params = N.search_params(10, 256, 512, tau, 1000, qflags)
if os.environ.get("LARGE_WAVES"):  # large-batch variant threshold (ggnn_query_schedule_large)
    N.call("ggnn_query_schedule_large", float(os.environ["LARGE_WAVES"]))
Qall = np.concatenate([Q, Q[::-1]])
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148, 592, 1184, 2368, 4144, 6000, 8000,
                                                                           10000, 20000]
for m in sizes:
    Qm = Qall[:m]
    dq, qs = dv.queries(Qm)
    ids = N.empty((m, 10), torch.int32)
    dd = N.empty((m, 10), torch.float64)
    cnt = N.empty((m, 5), torch.int32)

    def run():
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max, N.ptr(ids),
               N.ptr(dd), N.ptr(cnt), None, 0, N.stream_ptr())

    for _ in range(3):
        run()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    T = cnt[:, 1].cpu().numpy()
    t = float(np.median(ts))
    print(f"m={m:6d}  {t:7.3f} ms  {m / t / 1e3:6.2f} Mq/s  steps mean {T.mean():6.1f} p99 {np.percentile(T, 99):5.0f} "
          f"max {T.max():5d}  us/step(max chain) {t * 1e3 / T.max():6.2f}", flush=True)
