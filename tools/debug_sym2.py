import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import oracle as O
import paper_1912_01059_b200 as ga
from paper_1912_01059_b200 import _native as N
from paper_1912_01059_b200.device import DeviceVectors, sanitize
from conftest import load_golden, golden_hierarchy
from paper_1912_01059_b200.synthetic import make_sift_shaped

g = load_golden("sift10k.npz")
base, Q = make_sift_shaped()
h = golden_hierarchy(g, base)
L = h.layers[0]
X = h.vectors()
rng = np.random.default_rng(0)
xs = rng.choice(10000, 300, replace=False)
px, pz, pd = [], [], []
for x in xs:
    for t in range(L.k_nn):
        z = L.adjacency[x, t]
        if z >= 0:
            px.append(x); pz.append(z); pd.append(O.squared_l2(X[x], X[z]))
px, pz, pd = map(np.array, (px, pz, pd))
dmax = L.live_d_nn1_max()
want = np.array([O.sym_check_pair(X, h.rows_for(0), L.adjacency, L.k_nn, L.sym_count, int(x), int(z), d, 0.5, dmax,
                                  16, 12, 64, 128, 8)[0] for x, z, d in zip(px, pz, pd)])
dv = DeviceVectors.of(h.dataset)
t = N.torch()
adj = sanitize(N.to_dev(L.adjacency), N.to_dev(L.sym_count), L.node_count, L.k, L.k_nn)
layer = N.Layer(N.ptr(adj), None, None, L.node_count, L.k, L.k_nn, 0.0)
dx, dz, dd = N.to_dev(px.astype(np.int32)), N.to_dev(pz.astype(np.int32)), N.to_dev(pd.astype(np.float64))
ver = N.empty((len(px),), t.int32)
fb = N.empty((len(px), 8), t.int32)
N.call("ggnn_sym_check_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(layer), N.ptr(dx), N.ptr(dz), N.ptr(dd),
       len(px), 0.5, dmax, 16, 12, 64, 128, 8, N.ptr(ver), N.ptr(fb), N.stream_ptr())
got = ver.cpu().numpy()
print("pairs", len(px), "ref verdict counts", np.bincount(want, minlength=3), "gpu", np.bincount(got, minlength=3))
bad = np.nonzero(got != want)[0]
print("mismatches", len(bad), [(int(px[i]), int(pz[i]), int(want[i]), int(got[i])) for i in bad[:10]])
