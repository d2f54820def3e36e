"""ncu target for the scheduled C2 query path: builds the C2 index, runs a few
warm-up batches through query_arrays, then one batch between
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures exactly the
kernels of one scheduled 10k-query batch (query_kernel pilot, park_order,
resume rounds).  Usage: ncu --profile-from-start off ... python tools/ncu_sched.py"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16, make_latent16_queries  # noqa: E402

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
cfg = ga.QueryConfig(k_out=10, tau=float(sys.argv[1]) if len(sys.argv) > 1 else 0.58)
Qb = make_latent16_queries(10_000, 128, batch=3, seed=1234)
for _ in range(3):
    ga.query_arrays(h, Qb, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = ga.query_arrays(h, Qb, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("steps mean", r.counters[:, 1].mean(), "max", r.counters[:, 1].max())
