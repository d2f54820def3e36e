"""Where the host-to-host query call spends its time beyond the kernel:
host timestamps around each stage of search._query_host_staged, plus CUDA
events on the search stream (C2 workload, 10k queries)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import _native as N, search as S  # noqa: E402
from paper_1912_01059_b200.device import device_hierarchy  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
cfg = ga.QueryConfig(k_out=10, tau=0.58)
Qp = torch.empty(Q.shape, dtype=torch.float32, pin_memory=True)
Qp.copy_(torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float32)))
Q = Qp.numpy()
dh = device_hierarchy(h)
for _ in range(5):
    ga.query_arrays(h, Q, cfg)
torch.cuda.synchronize()

t = torch
acc = {}
for it in range(30):
    T = [time.perf_counter()]
    dv = dh.vectors
    m, d = Q.shape
    st = S._STAGING[t.cuda.current_device()].ensure(m, d, 10)
    search_s, copy_s = S._STREAMS[t.cuda.current_device()]
    st.epoch += 1
    st.epoch_pin[0] = st.epoch
    params = S._params(cfg, S._qflags(dh, False))
    e0, e1 = (t.cuda.Event(enable_timing=True) for _ in range(2))
    e0.record(search_s)
    T.append(time.perf_counter())
    N.call("ggnn_query_batch_host", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
           N.ptr(dh.top_rows), dh.ntop, N.P(Q.ctypes.data), m, N.ctypes.byref(params), dh.d_nn1_max,
           N.ptr(st.q_f32), N.ptr(st.chunk_flags), N.ptr(st.epoch_pin), 8, 1, N.ptr(st.ids),
           N.ptr(st.dists), N.ptr(st.cnt), N.ptr(st.status), N.ptr(st.ids_pin), N.ptr(st.dists_pin),
           N.ptr(st.cnt_pin), N.ptr(st.status_pin), N.P(search_s.cuda_stream), N.P(copy_s.cuda_stream))
    e1.record(search_s)
    T.append(time.perf_counter())
    search_s.synchronize()
    copy_s.synchronize()
    T.append(time.perf_counter())
    ok = int(st.status_pin[0]) == 0
    r = S.BatchResult(st.ids_pin[:m].numpy().copy(), st.dists_pin[:m].numpy().copy(), st.cnt_pin[:m].numpy().copy())
    T.append(time.perf_counter())
    names = ["prelude", "native call (issue)", "sync", "numpy out"]
    for i, n_ in enumerate(names):
        acc.setdefault(n_, []).append((T[i + 1] - T[i]) * 1e3)
    acc.setdefault("total", []).append((T[-1] - T[0]) * 1e3)
    acc.setdefault("gpu: search + d2h (events)", []).append(e0.elapsed_time(e1))
    assert ok
for k, v in acc.items():
    print(f"{k:28s} {np.median(v):7.3f} ms")
t0 = time.perf_counter()
for _ in range(20):
    ga.query_arrays(h, Q, cfg)
print(f"query_arrays end to end      {(time.perf_counter() - t0) / 20 * 1e3:7.3f} ms")

# kernel cost of the staged variant itself: every chunk already published
st.chunk_flags.fill_(st.epoch)
torch.cuda.synchronize()
dq, qs = dh.vectors.queries(np.ascontiguousarray(Q))
params = S._params(cfg, S._qflags(dh, False))


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def staged():
    N.call("ggnn_query_batch_staged", N.ctypes.byref(dh.vectors.struct), N.ctypes.byref(dh.layers[0].struct),
           N.ptr(dh.top_rows), dh.ntop, N.ptr(st.q_f32), 10000, N.ctypes.byref(params), dh.d_nn1_max,
           N.ptr(st.chunk_flags), 1250, N.ctypes.c_uint32(st.epoch), 1, N.ptr(st.ids), N.ptr(st.dists),
           N.ptr(st.cnt), N.ptr(st.status), N.stream_ptr())


def plain():
    N.call("ggnn_query_batch", N.ctypes.byref(dh.vectors.struct), N.ctypes.byref(dh.layers[0].struct),
           N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max, N.ptr(st.ids),
           N.ptr(st.dists), N.ptr(st.cnt), None, 0, N.stream_ptr())


print(f"staged kernel, data resident {timed(staged):.3f} ms; plain kernel {timed(plain):.3f} ms")
