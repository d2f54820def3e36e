"""Throughput of the reference-named batch_query (QueryResult objects, exact
distinct_touched) vs query_arrays on the C2 workload."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
cfg = ga.QueryConfig(k_out=10, tau=0.6)
for name, fn in (("query_arrays", lambda: ga.query_arrays(h, Q, cfg)),
                 ("query_arrays(distinct)", lambda: ga.query_arrays(h, Q, cfg, distinct=True)),
                 ("batch_query", lambda: ga.batch_query(h, Q, cfg))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name:24s} {dt * 1e3:8.2f} ms per 10k -> {10000 / dt / 1e3:8.1f} k QPS")
