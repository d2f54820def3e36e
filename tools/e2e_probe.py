"""Time the host-to-host query path (query_arrays) for several chunk counts."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import search  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

base, Q = make_latent16(n=1_000_000, d=128, m=10_000, seed=1234)
h, _ = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
cfg = ga.QueryConfig(k_out=10, tau=0.6)
ref = None
if "--pinned" in sys.argv:  # the caller's batch lives in page-locked memory
    Qp = torch.empty(Q.shape, dtype=torch.float32, pin_memory=True)
    Qp.copy_(torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float32)))
    Q = Qp.numpy()
    print("pinned input", flush=True)
for staged, chunks, first in ((True, 2, 0.5), (False, 2, 0.5), (True, 2, 0.5), (False, 2, 0.5)):
    search._STAGED, search._CHUNKS, search._FIRST = staged, chunks, first
    for _ in range(3):
        r = ga.query_arrays(h, Q, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        r = ga.query_arrays(h, Q, cfg)
    dt = (time.perf_counter() - t0) / 20
    if ref is None:
        ref = r.ids
    assert np.array_equal(r.ids, ref)
    print(f"staged {staged} chunks {chunks} first {first}: {dt * 1e3:.3f} ms per 10k -> {10000 / dt / 1e6:.3f} M QPS e2e",
          flush=True)
for sc in (4, 8, 16, 32):
    search._STAGED, search._STAGED_CHUNKS = True, sc
    for _ in range(3):
        r = ga.query_arrays(h, Q, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        r = ga.query_arrays(h, Q, cfg)
    dt = (time.perf_counter() - t0) / 20
    assert np.array_equal(r.ids, ref)
    print(f"staged chunks {sc}: {dt * 1e3:.3f} ms per 10k -> {10000 / dt / 1e6:.3f} M QPS e2e", flush=True)
