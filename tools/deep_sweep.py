"""C4 (deep10m) recall vs the query cache size: one build, then R@10 for
(prioq_size, visited_size, tau) combinations on 1000 held-out queries, with
the query kernel time of a 10k batch.  Usage: python tools/deep_sweep.py [n]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_deep_like  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
base, Q = make_deep_like(n, 10_000)
ds = ga.Dataset(base)
t0 = time.perf_counter()
h, st = ga.build(ds, ga.BuildConfig(seed=7))
print(f"build {st.build_seconds:.1f} s", flush=True)
gt = ga.brute_force_oracle(ds, Q[:1000], 10).ids
for prioq, vis in ((256, 512), (512, 1024), (1024, 2048), (2048, 4096)):
    for tau in (0.6, 1.0, 2.0, 4.0):
        cfg = ga.QueryConfig(k_out=10, tau=tau, prioq_size=prioq, visited_size=vis, max_iterations=4000)
        r = ga.query_arrays(h, Q[:1000], cfg)
        rec = float(np.mean((r.ids[:, :10] == gt[:, :1]).any(axis=1)))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rr = ga.query_arrays(h, Q, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        term = np.bincount(r.counters[:, 2], minlength=3)
        print(f"prioq {prioq} vis {vis} tau {tau}: R@10 {rec:.4f} V {r.counters[:, 0].mean():.0f} "
              f"T {r.counters[:, 1].mean():.0f} term {term.tolist()} e2e {10000 / dt / 1e3:.0f} k q/s", flush=True)
