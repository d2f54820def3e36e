"""Ground truth of the float brute force: tensor-core path (3xTF32 + exact
re-score) vs the CUDA-core scan (forced through a row subset = every row),
on the C4 generator.  Usage: python tools/gt_check.py [n] [m]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import _native as N  # noqa: E402
from paper_1912_01059_b200.device import DeviceVectors  # noqa: E402
from paper_1912_01059_b200.synthetic import make_deep_like  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
base, Q = make_deep_like(n, 10_000)
Q = Q[:m]
ds = ga.Dataset(base)
tc_ids, tc_d = ga.search.exact_knn(ds, Q, 10)
dv = DeviceVectors.of(ds)
t = N.torch()
rows = N.to_dev(np.arange(n, dtype=np.int32))
dq, qs = dv.queries(Q)
ids = N.empty((m, 10), t.int32)
dists = N.empty((m, 10), t.float64)
N.call("ggnn_exhaustive_topk", N.ctypes.byref(dv.struct), N.ptr(rows), n, N.ctypes.byref(qs), 10, N.ptr(ids),
       N.ptr(dists), N.stream_ptr())
w_ids, w_d = ids.cpu().numpy(), dists.cpu().numpy()
print("ids equal rows:", int((tc_ids == w_ids).all(axis=1).sum()), "of", m,
      " dists equal rows:", int((tc_d == w_d).all(axis=1).sum()))
bad = np.nonzero(~(tc_ids == w_ids).all(axis=1))[0][:5]
for i in bad:
    print(i, tc_ids[i], w_ids[i], tc_d[i] - w_d[i])
