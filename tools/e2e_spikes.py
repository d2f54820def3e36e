"""Per-call wall times of the host-array query (C2, pinned 10k batches):
which calls spike, with and without the Python GC."""
import gc
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16, make_latent16_queries  # noqa: E402

base, _ = make_latent16(n=1_000_000, d=128, m=16, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
cfg = ga.QueryConfig(k_out=10, tau=0.58)
pinned = [torch.from_numpy(make_latent16_queries(10_000, 128, batch=b + 1, seed=1234).astype(np.float32)).pin_memory()
          .numpy() for b in range(8)]
for i in range(20):
    ga.query_arrays(h, pinned[i % 8], cfg)
torch.cuda.synchronize()
for mode in ("gc on", "gc off", "gc on"):
    if mode == "gc off":
        gc.disable()
    else:
        gc.enable()
    ts = []
    for i in range(200):
        c0 = time.perf_counter()
        out = ga.query_arrays(h, pinned[i % 8], cfg)
        ts.append((time.perf_counter() - c0) * 1e3)
    ts = np.array(ts)
    med = np.median(ts)
    sp = np.nonzero(ts > 1.3 * med)[0]
    print(f"{mode}: median {med:.3f} mean {ts.mean():.3f} max {ts.max():.3f}  spikes at {sp.tolist()[:30]} "
          f"values {[round(float(x), 2) for x in ts[sp][:30]]}", flush=True)
