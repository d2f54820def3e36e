"""Kernel time of the C2 batch under different query orders (drain study):
orders by cheap pre-search features vs the oracle longest-first order."""
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


def run(Qm, maxit=1000, reps=7):
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


t0, _, c = run(Q)
T = c[:, 1]
print(f"given order {t0:.3f} ms", flush=True)
Qd = Q.astype(np.float64)
feats = {}
qn = (Qd ** 2).sum(1)
for li in range(h.num_layers - 1, 0, -1):
    rows = h.to_bottom[li]
    if len(rows) > 8192:
        break
    Xt = base[rows].astype(np.float64)
    dd = np.sort(qn[:, None] + (Xt ** 2).sum(1)[None] - 2 * Qd @ Xt.T, axis=1)
    feats[f"L{li}_d1"] = dd[:, 0]
    feats[f"L{li}_d10/d1"] = dd[:, 9] / np.maximum(dd[:, 0], 1)
mu = base[:200000].astype(np.float64).mean(0)
feats["|q-mu|"] = ((Qd - mu) ** 2).sum(1)
for k, v in feats.items():
    best = None
    for sgn in (1, -1):
        order = np.argsort(-sgn * v, kind="stable")
        to, _, _ = run(np.ascontiguousarray(Q[order]))
        best = min(best or 1e9, to)
        print(f"  {k:14s} spearman {spear(T, v):+.3f}  order {'desc' if sgn > 0 else 'asc '}: {to:.3f} ms", flush=True)
to, _, _ = run(np.ascontiguousarray(Q[np.argsort(-T, kind='stable')]))
print(f"oracle longest-first {to:.3f} ms")
