"""Per-symmetrize-pass trace of a build (GGNN_TRACE): requests, claim rounds,
check vs claim-round seconds.  Usage: python tools/trace_build.py [sift10k|latent N]"""
import importlib
import json
import os
import sys
from pathlib import Path

os.environ["GGNN_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1912_01059_b200 as ga  # noqa: E402
from paper_1912_01059_b200.synthetic import make_latent16, make_sift_shaped  # noqa: E402

B = importlib.import_module("paper_1912_01059_b200.build")
if len(sys.argv) > 1 and sys.argv[1] == "latent":
    base = make_latent16(n=int(sys.argv[2]), d=128, m=1)[0]
else:
    base = make_sift_shaped()[0]
ga.build(ga.Dataset(base[:50000].copy()), ga.BuildConfig(seed=7))  # warm
B.TRACE.clear()
h, st = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
tot_check = sum(r["check_s"] for r in B.TRACE)
tot_claim = sum(r["claim_s"] for r in B.TRACE)
for r in B.TRACE:
    if r["nodes"] >= 100000:
        print(json.dumps(r))
print(f"passes {len(B.TRACE)} rounds {sum(r['rounds'] for r in B.TRACE)} check {tot_check:.2f}s claim {tot_claim:.2f}s "
      f"build {st.build_seconds:.2f}s (traced: syncs per pass)")
print("phases", sorted(st.phase_seconds.items(), key=lambda kv: -kv[1])[:8])
