"""Query-kernel time (device-resident, CUDA events) on the C2 graph for the
default and a large query cache.  Usage: GGNN_LIB=... python tools/cache_probe.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
for pq, vs, tau in ((256, 512, 0.58), (1024, 2048, 0.58), (1024, 2048, 2.0), (2048, 4096, 1.0)):
    cfg = ga.QueryConfig(k_out=10, tau=tau, prioq_size=pq, visited_size=vs, max_iterations=4 * pq)
    for _ in range(3):
        ga.query_arrays(h, Q, cfg, out="device")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ids, d, c = ga.query_arrays(h, Q, cfg, out="device")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"prioq {pq} tau {tau}: {ms:.3f} ms per 10k (incl. upload)  V {c[:, 0].float().mean().item():.0f}", flush=True)
