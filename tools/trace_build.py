import os, sys, json
os.environ["GGNN_TRACE"] = "1"
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import importlib
import numpy as np
import paper_1912_01059_b200 as ga
from paper_1912_01059_b200.synthetic import make_sift_shaped
B = importlib.import_module("paper_1912_01059_b200.build")
base, Q = make_sift_shaped()
h, st = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
for r in B.TRACE:
    print(json.dumps(r))
print("mean_sym", st.mean_sym_used, "dropped", st.dropped_sym_links, "secs", st.build_seconds)
