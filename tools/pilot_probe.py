"""Can a short pilot search (max_iterations = P) predict a query's full
search length?  If so, launching the batch longest-first shortens the drain."""
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

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
dh = device_hierarchy(h)
dv = dh.vectors
m = Q.shape[0]


def run(Qm, maxit, reps=5):
    dq, qs = dv.queries(Qm)
    mm = Qm.shape[0]
    ids = N.empty((mm, 10), torch.int32)
    dd = N.empty((mm, 10), torch.float64)
    cnt = N.empty((mm, 5), torch.int32)
    params = N.search_params(10, 256, 512, 0.6, maxit, 0)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max, N.ptr(ids),
               N.ptr(dd), N.ptr(cnt), None, 0, N.stream_ptr())
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), dd.cpu().numpy(), cnt.cpu().numpy()


def spear(a, b):
    return np.corrcoef(np.argsort(np.argsort(a)), np.argsort(np.argsort(b)))[0, 1]


t_full, d_full, c_full = run(Q, 1000)
T = c_full[:, 1]
print(f"full: {t_full:.3f} ms  T mean {T.mean():.1f} max {T.max()}")
for P in (4, 8, 16, 32):
    tp, dp, cp = run(Q, P)
    feats = {"d1": dp[:, 0], "d10": dp[:, 9], "d10/d1": dp[:, 9] / np.maximum(dp[:, 0], 1), "V": cp[:, 0]}
    print(f"pilot P={P}: {tp:.3f} ms  " + "  ".join(f"{k} {spear(T, v):+.3f}" for k, v in feats.items()), flush=True)
    for k, v in feats.items():
        for sgn in (1, -1):
            order = np.argsort(-sgn * v, kind="stable")
            to, _, _ = run(np.ascontiguousarray(Q[order]), 1000)
            print(f"   order by {'-' if sgn < 0 else '+'}{k}: {to:.3f} ms", flush=True)
oracle_order = np.argsort(-T, kind="stable")
to, _, _ = run(np.ascontiguousarray(Q[oracle_order]), 1000)
print(f"oracle longest-first order: {to:.3f} ms (upper bound of any predictor)")
