"""Host-to-host query path vs the device-resident kernel on any bench
workload: staged (one launch, overlapped upload) vs chunked two-stream path.
Usage: python tools/e2e_workload_probe.py gist1m [tau]"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import _native as N, search as S  # noqa: E402
from paper_1912_01059_b200.device import device_hierarchy  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gist1m"
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 0.6
n, d = bench.DEFAULT_SHAPE[wl]
args = argparse.Namespace(workload=wl, n=n, d=d, queries=10_000)
base, Q = bench.make_workload(args)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
cfg = ga.QueryConfig(k_out=10, tau=tau)
Qp = torch.empty(Q.shape, dtype=torch.float32, pin_memory=True)
Qp.copy_(torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float32)))
Qh = Qp.numpy()
dh = device_hierarchy(h)
dq, qs = dh.vectors.queries(np.ascontiguousarray(Q, dtype=np.float32))
params = S._params(cfg, S._flags(dh.vectors, False))
m = Q.shape[0]
ids = N.empty((m, 10), torch.int32)
dd = N.empty((m, 10), torch.float64)
cnt = N.empty((m, 5), torch.int32)


def plain():
    N.call("ggnn_query_batch", N.ctypes.byref(dh.vectors.struct), N.ctypes.byref(dh.layers[0].struct),
           N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max, N.ptr(ids),
           N.ptr(dd), N.ptr(cnt), None, 0, N.stream_ptr())


for _ in range(3):
    plain()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    plain()
b.record()
torch.cuda.synchronize()
print(f"{wl}: resident kernel {a.elapsed_time(b) / 5:.3f} ms", flush=True)
for staged in (True, False, True):
    S._STAGED = staged
    for _ in range(3):
        r = ga.query_arrays(h, Qh, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        r = ga.query_arrays(h, Qh, cfg)
    dt = (time.perf_counter() - t0) / 5
    print(f"  staged={staged}: {dt * 1e3:.3f} ms per batch", flush=True)
    if staged:
        st = S._STAGING[torch.cuda.current_device()]
        print("   status", int(st.status_pin[0]))
