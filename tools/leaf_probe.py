"""Leaf kNN timing on one layer-0 batch set (C3 / C4 shapes): the tensor-core
path (tf32 for float rows) vs the CUDA-core path, same batches, bitwise equal.
Usage: python tools/leaf_probe.py [gist|deep] [n]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_01059_b200 import _native as N  # noqa: E402
from paper_1912_01059_b200.build import partition_bottom, plan_geometry  # noqa: E402
from paper_1912_01059_b200.device import DeviceVectors  # noqa: E402
from paper_1912_01059_b200.synthetic import make_deep_like, make_latent16  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "gist"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
X = make_latent16(n=n, d=960, m=1, as_float=True)[0] if kind == "gist" else make_deep_like(n, 1)[0]
X.setflags(write=False)
dv = DeviceVectors.of_array(X)
l, b = plan_geometry(n, 32, 4)
perm, offs = partition_bottom(n, b, np.random.default_rng(7))
k_nn = 12
mem, off = N.to_dev(perm), N.to_dev(offs)
out = {}
for name in ("ggnn_leaf_knn_tc", "ggnn_leaf_knn"):
    pos = N.empty((n, k_nn), torch.int32)
    dist = N.empty((n, k_nn), torch.float64)
    if name == "ggnn_leaf_knn":  # force the CUDA-core path: a max_batch above the tensor-core tile
        mb = 129
    else:
        mb = int(np.diff(offs).max())
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        N.call(name, N.ctypes.byref(dv.struct), N.ptr(mem), None, N.ptr(off), b, mb, k_nn, N.ptr(pos), N.ptr(dist),
               None, 0, None, None, None, N.stream_ptr())
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    out[name] = (pos.cpu().numpy(), dist.cpu().numpy())
    macs = float((np.diff(offs) ** 2).sum()) * X.shape[1]
    print(f"{kind} n={n} d={X.shape[1]} {name:18s} {dt * 1e3:8.2f} ms  ({2 * macs / dt / 1e12:.2f} TFLOP/s useful)")
N.check_tc_timeouts("leaf")
a, c = out["ggnn_leaf_knn_tc"], out["ggnn_leaf_knn"]
print("bitwise equal:", np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1]))
