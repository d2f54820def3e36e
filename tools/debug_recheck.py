import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1912_01059_b200 as ga
from paper_1912_01059_b200 import _native as N
from paper_1912_01059_b200.device import DeviceVectors, sanitize
from paper_1912_01059_b200.synthetic import make_sift_shaped
z = np.load("tools/_dbg/ref_leafsym.npz")
base, Q = make_sift_shaped()
ds = ga.Dataset(base)
dv = DeviceVectors.of(ds)
t = N.torch()
adj = sanitize(N.to_dev(z["adj"]), N.to_dev(z["symc"]), 10000, 24, 12)
layer = N.Layer(N.ptr(adj), None, None, 10000, 24, 12, float(z["dmax"]))
snap = z["snap"]
X64 = base.astype(np.float64)
recs = np.zeros((len(snap), 13), dtype=np.int32)
for i, (x, zz) in enumerate(snap):
    d = float(((X64[x] - X64[zz]) ** 2).sum())
    recs[i, 0] = i; recs[i, 1] = x; recs[i, 2] = zz
    recs[i, 3:5] = np.array([d]).view(np.int32)
req = N.to_dev(recs)
stage = t.zeros(len(snap), dtype=t.int32, device="cuda")
N.call("ggnn_sym_recheck", N.ctypes.byref(dv.struct), N.ctypes.byref(layer), N.ptr(req), len(snap), N.ptr(stage),
       10000, 0.5, float(z["dmax"]), 16, 12, 64, 128, 8, N.stream_ptr())
st = stage.cpu().numpy()
print("recheck on reference post-pass graph: settled", int((st == -3).sum()), "still-2", int((st == 0).sum()))
# explicit pairs API on the same graph
px = N.to_dev(snap[:, 0].copy()); pz = N.to_dev(snap[:, 1].copy())
pd = N.to_dev(np.array([((X64[x] - X64[zz]) ** 2).sum() for x, zz in snap]))
ver = t.empty(len(snap), dtype=t.int32, device="cuda"); fb = t.empty((len(snap), 8), dtype=t.int32, device="cuda")
N.call("ggnn_sym_check_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(layer), N.ptr(px), N.ptr(pz), N.ptr(pd),
       len(snap), 0.5, float(z["dmax"]), 16, 12, 64, 128, 8, N.ptr(ver), N.ptr(fb), N.stream_ptr())
print("pairs API verdicts", np.bincount(ver.cpu().numpy(), minlength=3))
