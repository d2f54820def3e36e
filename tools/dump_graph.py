"""Build a GPU graph for a golden shape and save it (GGNN v1) under gpurun_out/."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "oracle")]
import paper_1912_01059_b200 as ga  # noqa: E402
from test_shapes import _data  # noqa: E402

for name in sys.argv[1:]:
    base, q = _data(name)
    h, st = ga.build(ga.Dataset(base), ga.BuildConfig(seed=7))
    ga.save_index(h, ROOT / "gpurun_out" / f"{name}_gpu.idx")
    print(name, st.phase_seconds.keys().__len__())
