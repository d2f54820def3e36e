"""Dump the C2 batch's per-query search lengths (full search) and short-pilot
features (max_iterations = P) for the drain scheduling study: run with
GGNN_LIB=build/libggnn_dbgopen.so (-DGGNN_DEBUG_OPEN: counter column 3 is the
pilot's pending work, unexpanded ring entries within the stopping threshold)
-> gpurun_out/drain_data.npz."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import _native as N  # noqa: E402
from paper_1912_01059_b200.device import device_hierarchy  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16, make_latent16_queries  # noqa: E402

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
dh = device_hierarchy(h)
dv = dh.vectors


def run(Qm, maxit, tau=0.58, reps=3):
    dq, qs = dv.queries(Qm)
    mm = Qm.shape[0]
    ids = N.empty((mm, 10), torch.int32)
    dd = N.empty((mm, 10), torch.float64)
    cnt = N.empty((mm, 5), torch.int32)
    params = N.search_params(10, 256, 512, tau, maxit, 0)
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


out = {}
for bi in range(3):
    Qb = Q if bi == 0 else make_latent16_queries(10_000, 128, batch=bi, seed=1234)
    t, d, c = run(Qb, 1000)
    out[f"b{bi}_T"] = c[:, 1]
    out[f"b{bi}_V"] = c[:, 0]
    out[f"b{bi}_ms"] = t
    for P in (4, 8, 12, 16, 24, 32):
        tp, dp, cp = run(Qb, P)
        out[f"b{bi}_P{P}_open"] = cp[:, 3]
        out[f"b{bi}_P{P}_d1"] = dp[:, 0]
        out[f"b{bi}_P{P}_d10"] = dp[:, 9]
        out[f"b{bi}_P{P}_ms"] = tp
    ord_ = np.argsort(-c[:, 1], kind="stable")
    out[f"b{bi}_oracle_ms"] = run(np.ascontiguousarray(Qb[ord_]), 1000)[0]
    ord_ = np.argsort(-out[f"b{bi}_P16_d1"], kind="stable")
    out[f"b{bi}_p16d1_ms"] = run(np.ascontiguousarray(Qb[ord_]), 1000)[0]
    print(bi, t, out[f"b{bi}_oracle_ms"], out[f"b{bi}_p16d1_ms"], flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
np.savez("gpurun_out/drain_data.npz", **out)
