"""Host-array query calls with and without the longest-first schedule
(ggnn_query_schedule), page-locked vs pageable query rows, uint8 and float
tables (latent16 n x 128, 10k queries): ms per call."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import _native as N  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16, make_latent16_queries  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
base, _ = make_latent16(n=n, d=128, m=16, seed=1234)
Qs = [make_latent16_queries(10_000, 128, batch=b + 1, seed=1234) for b in range(4)]
for kind in ("u8", "f32"):
    X = base if kind == "u8" else (base / 255.0).astype(np.float32)
    h, _ = ga.build(ga.Dataset(X), ga.BuildConfig(seed=7))
    qs = [(q if kind == "u8" else q / 255.0).astype(np.float32) for q in Qs]
    pinned = [torch.from_numpy(q).pin_memory().numpy() for q in qs]
    cfg = ga.QueryConfig(k_out=10, tau=0.58)
    for P in (0, 20):
        N.call("ggnn_query_schedule", P, 1.5)
        for name, arrs in (("pageable", qs), ("pinned", pinned)):
            for i in range(8):
                ga.query_arrays(h, arrs[i % 4], cfg)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(40):
                ga.query_arrays(h, arrs[i % 4], cfg)
            torch.cuda.synchronize()
            print(f"{kind} P={P} {name:8s} {(time.perf_counter() - t0) / 40 * 1e3:.3f} ms/call", flush=True)
