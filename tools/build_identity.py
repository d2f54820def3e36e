"""Build C2-shaped latent16 (n points) twice -- claim-round compaction on and
off -- and check the graphs are identical; print both build times.
Usage: python tools/build_identity.py [n]"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200 import build as B  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
base = make_latent16(n=n, d=128, m=1)[0]
ga.build(ga.Dataset(base[:50000].copy()), ga.BuildConfig(seed=7))
out = {}
for flag in (True, False, True):
    B.CLAIM_COMPACT = flag
    h, st = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
    out[flag] = h
    print(f"compact={flag} build {st.build_seconds:.2f} s", flush=True)
same = all(np.array_equal(a.adjacency, b.adjacency) and np.array_equal(a.sym_count, b.sym_count)
           for a, b in zip(out[True].layers, out[False].layers))
print("identical graphs:", same)
import hashlib  # noqa: E402

hsh = hashlib.sha256()
for L in out[True].layers:
    hsh.update(L.adjacency.tobytes())
    hsh.update(L.sym_count.tobytes())
print("graph sha256:", hsh.hexdigest()[:16])
