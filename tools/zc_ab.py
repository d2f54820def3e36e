"""A/B of the host-to-host query call with and without zero copy
(GGNN_ZERO_COPY, read once per process): C2 workload, 8 pinned 10k-query
batches cycled, ms per call over many calls (host wall clock, synchronised)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16, make_latent16_queries  # noqa: E402

base, _ = make_latent16(n=1_000_000, d=128, m=16, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
cfg = ga.QueryConfig(k_out=10, tau=0.58)
batches = []
for b in range(8):
    Q = make_latent16_queries(10_000, 128, batch=b + 1, seed=1234)
    t = torch.empty(Q.shape, dtype=torch.float32, pin_memory=True)
    t.copy_(torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float32)))
    batches.append(t.numpy())
for i in range(10):
    ga.query_arrays(h, batches[i % 8], cfg)
torch.cuda.synchronize()
res = []
for rep in range(5):
    t0 = time.perf_counter()
    for i in range(100):
        ga.query_arrays(h, batches[i % 8], cfg)
    torch.cuda.synchronize()
    res.append((time.perf_counter() - t0) * 10)
print("zero_copy", os.environ.get("GGNN_ZERO_COPY", "1"), "ms/call", " ".join(f"{x:.3f}" for x in res),
      "best %.3f" % min(res))
