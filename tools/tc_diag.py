"""Diagnostics for the tcgen05 leaf kNN: repeated launches vs the CPU checker."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import oracle as O  # noqa: E402
from paper_1912_01059_b200 import _native as N  # noqa: E402
from paper_1912_01059_b200.device import DeviceVectors  # noqa: E402


def run(d, seed, reps):
    rng = np.random.default_rng(seed)
    sizes = np.concatenate([[2, 3, 16, 17, 128, 127, 64], rng.integers(2, 129, size=33)])
    n = int(sizes.sum()) + 50
    X = rng.integers(0, 4 if d == 32 else 256, size=(n, d)).astype(np.float32)
    X.setflags(write=False)
    members = rng.permutation(n)[: sizes.sum()].astype(np.int32)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    dv = DeviceVectors.of_array(X)
    t = N.torch()
    ref = [O.batch_bruteforce(X, members[offsets[b]:offsets[b + 1]], 12) for b in range(len(sizes))]
    mem_d, off_d = N.to_dev(members), N.to_dev(offsets)
    bad_total = 0
    for r in range(reps):
        pos = N.empty((len(members), 12), t.int32)
        dist = N.empty((len(members), 12), t.float64)
        N.call("ggnn_leaf_knn_tc", N.ctypes.byref(dv.struct), N.ptr(mem_d), None, N.ptr(off_d), len(sizes),
               int(sizes.max()), 12, N.ptr(pos), N.ptr(dist), None, 0, None, None, None, N.stream_ptr())
        dist = dist.cpu().numpy()
        bad = [b for b in range(len(sizes)) if not np.array_equal(dist[offsets[b]:offsets[b + 1]], ref[b][1])]
        if bad:
            bad_total += 1
            print(f"d={d} rep={r}: bad batches {bad[:10]} sizes {[int(sizes[b]) for b in bad[:10]]}")
            b = bad[0]
            print("  got", dist[offsets[b]:offsets[b] + 2, :4].tolist(), "want", ref[b][1][:2, :4].tolist())
    print(f"d={d}: {bad_total}/{reps} launches with mismatches; timeouts={N.load().ggnn_tc_timeouts()}")


if __name__ == "__main__":
    N.torch().cuda.set_device(0)
    for d in (32, 128, 64, 256):
        run(d, d, int(sys.argv[1]) if len(sys.argv) > 1 else 20)
