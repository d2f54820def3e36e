import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1912_01059_b200 as ga
import importlib
from paper_1912_01059_b200 import _devgraph as G
B = importlib.import_module("paper_1912_01059_b200.build")
from paper_1912_01059_b200.graph import AdjacencyLayer, Hierarchy

ds = ga.Dataset(np.asarray([0.0, 1.0, 10.0], dtype=np.float32).reshape(-1, 1))
cfg = ga.BuildConfig(k=2, k_nn=1, k_sym=1, s=2, g=2, refinements=0, seed=0)
layer = AdjacencyLayer(3, 2, 1)
h = Hierarchy([layer], [None], s=2, g=2, config=cfg, dim=1)
h.attach(ds)
ga.build_base(layer, ds.vectors, h.rows_for(0), np.arange(3, dtype=np.int32))
print("adj", layer.adjacency.tolist(), "nnd", layer.nn_dists.tolist(), "symc", layer.sym_count.tolist())
impl = ga.backend.impl
for x, z in ((2, 1), (1, 0), (0, 1)):
    v, fb = impl.sym_check_pair(ds.vectors, h.rows_for(0), layer.adjacency, 1, layer.sym_count, x, z,
                                float(layer.nn_dists[x, 0]), 0.5, layer.live_d_nn1_max(), 16, 1, 64, 128, 8,
                                impl.SymScratch(3, 2, 65, 128, 16, 8))
    print("pair", x, z, "verdict", v, fb.tolist())
G.ensure_device(h)
ws = G.workspace(h)
dev = layer._dev
print("dev adj", dev["adj"].cpu().tolist(), "dnn1", dev["dnn1"].cpu().tolist(), "live", G.live_max(h, layer))
dropped = B._symmetrize_dev(h, 0, 0.5, None)
print("req_count", ws.req_count.item(), "req", ws.req[: max(1, ws.req_count.item())].cpu().tolist(), "dropped", dropped)
print("after adj", dev["adj"].cpu().tolist(), "symc", dev["symc"].cpu().tolist(), "best", ws.best.cpu().tolist())
