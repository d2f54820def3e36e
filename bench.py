"""GGNN B200 benchmark: QPS at R@10 >= 0.99 on SIFT1M-shaped data + build seconds.

Workload (BASELINE.json configs[1], "C2", the default): synthetic SIFT1M-shaped
latent16 data (SURVEY.md 8d "G_B"), 1M x 128 integer-valued (stored losslessly
as uint8 on the device), 10k queries per step, k=10, BuildConfig(seed=7)
defaults (k=24, k_nn=12, s=32, g=4, refinements=2, tau_build=0.5).  tau is
chosen in the run: the smallest tau of a sweep whose R@10 (the reference's
`recall_at`, evaluate.py:60-76) against exact ground truth computed on the GPU
in the same run is >= the target (0.99; 0.95 for C5); a sweep that never gets
there says so (`recall_target_reached: false`) instead of quietly reporting its
last tau.

A "step" is one batch of 10k queries through the query kernel with inputs
resident in HBM; every step searches a FRESH batch (B distinct seeded batches,
cycled).  Other workloads (--workload): c1 (configs[0], the reference's own
10k test data), sift1m-f32 (C2's shape as non-integer fp32), gist1m (C3),
deep10m (C4), c5 (SIFT100M: 8 shards of 12.5M uint8) and c5shard (one of them).

Multi-GPU (one process per GPU, torchrun):
  * default / single-index workloads: query-parallel replicas -- every rank
    holds the whole index and answers its own fresh batches; queries are
    independent units, so there is no data-path collective (scaling "weak",
    value = queries delivered by all ranks per second);
  * c5: a FIXED 8-shard index, N ranks holding 8/N shards each; a step is the
    replicated batch searched on every shard, an NCCL all-gather of the
    per-shard top-10 and the GPU k-way merge (scaling "strong", value =
    delivered queries/s; N = 1 is one GPU searching all 8 shards in turn, the
    north star's QPS_1);
  * deep10m: C4 strong scaling, the 10M points as N shards on N GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload W] [--impl ggnn|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "queries/sec at R@10>=0.99 (SIFT1M-shape, k=10); index build seconds"
UNIT = "queries/s"
TAUS = [0.2, 0.25, 0.3, 0.35, 0.4, 0.45, 0.5, 0.55, 0.6, 0.7, 0.8, 1.0, 1.25, 1.5, 2.0]

# workload -> (n, d, queries, description, recall target, shards (None: one index))
WORKLOADS = {
    "c1": (10_000, 128, 1000, "configs[0]: the reference's SIFT stand-in make_sift_shaped (tests/conftest.py:79-87) "
           "{n}x{d} integer-valued", 0.99, None),
    "sift1m": (1_000_000, 128, 10_000, "SIFT1M-shaped latent16 (SURVEY.md 8d G_B) {n}x{d} integer-valued (uint8 on "
               "the device)", 0.99, None),
    "sift1m-f32": (1_000_000, 128, 10_000, "SIFT1M-shaped latent16 {n}x{d} as non-integer float32 (no rounding, /255; "
                   "fp32 table on the device)", 0.99, None),
    "gist1m": (1_000_000, 960, 10_000, "GIST1M-shaped float latent16 {n}x{d} (C3: no rounding, /255)", 0.99, None),
    "deep10m": (10_000_000, 96, 10_000, "Deep10M-shaped {n}x{d} clustered (1024 clusters), rows L2-normalised (C4)",
                0.99, "ranks"),
    "c5": (100_000_000, 128, 10_000, "SIFT100M-shaped latent16 {n}x{d} integer-valued, 8 shards (uint8 on the "
           "device)", 0.95, 8),
    "c5shard": (12_500_000, 128, 10_000, "one SIFT100M shard: latent16 {n}x{d} integer-valued (uint8 on the device; "
                "C5 is 8 such shards)", 0.99, None),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ggnn", choices=["ggnn", "reference"])
    ap.add_argument("--workload", default="sift1m", choices=sorted(WORKLOADS))
    ap.add_argument("--points", dest="n", type=int, default=None, help="override the workload's point count")
    ap.add_argument("--dim", dest="d", type=int, default=None, help="override the workload's dimension")
    ap.add_argument("--queries", type=int, default=None, help="queries per step (default: the workload's)")
    ap.add_argument("--batches", type=int, default=8, help="distinct query batches cycled over the steps")
    ap.add_argument("--gt-queries", type=int, default=None, help="ground-truth subsample (default: all of batch 0 "
                    "for c1 / sift1m, 1000 otherwise)")
    ap.add_argument("--tau", type=float, default=None, help="skip the sweep and use this tau")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ref-build", action="store_true", help="skip timing the reference's CPU build")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="sharded workloads, N > 1: NCCL all-gather after the search, or the fused peer-memory "
                         "exchange (one shard per rank)")
    ap.add_argument("--prep-reference", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    args = ap.parse_args()
    n0, d0, m0, _, target, shards = WORKLOADS[args.workload]
    args.n = args.n or n0
    args.d = args.d or d0
    args.queries = args.queries or m0
    args.target = target
    args.shards = shards
    return args


def workload_desc(args) -> str:
    return WORKLOADS[args.workload][3].format(n=args.n, d=args.d)


def config_of(args, tau, prioq=256, visited=512, max_it=1000) -> dict:
    """The `config` object of the JSON line -- identical in both arms."""
    return {"workload": f"{args.workload}: {workload_desc(args)}", "queries_per_step": args.queries, "k": 10,
            "k_build": 24, "tau": tau, "prioq_size": prioq, "visited_size": visited, "max_iterations": max_it,
            "recall_target": f"R@10>={args.target}", "queries": "a fresh seeded batch every step"}


# ------------------------------------------------------------------ data
def make_base(args, n=None):
    """Base vectors of a single-index workload (float32, host)."""
    from paper_1912_01059_b200.synthetic import make_deep_like, make_latent16, make_sift_shaped

    n = n or args.n
    w = args.workload
    if w == "c1":
        return make_sift_shaped(n=n, d=args.d, m=args.queries)[0]
    if w in ("sift1m", "c5shard"):
        return make_latent16(n=n, d=args.d, m=1, seed=1234)[0]
    if w in ("sift1m-f32", "gist1m"):
        return make_latent16(n=n, d=args.d, m=1, seed=1234, as_float=True)[0]
    if w == "deep10m":  # one draw with the held-out query rows (the generator's stream depends on its length)
        return make_deep_like(n, args.queries, d=args.d)[0]
    raise ValueError(w)


def make_queries(args, batch: int):
    """Query batch `batch` (0 = the workload's canonical query set)."""
    from paper_1912_01059_b200 import synthetic as S

    w, m, d = args.workload, args.queries, args.d
    if w == "c1":
        if batch == 0:
            return S.make_sift_shaped(n=args.n, d=d, m=m)[1]
        base = make_base(args)  # further noisy copies of base rows (the generator's query law)
        rng = np.random.default_rng((1234, 0xC1, batch))
        picks = rng.choice(base.shape[0], size=m, replace=False)
        return np.clip(np.rint(base[picks] + rng.normal(0, 12, (m, d))), 0, 255).astype(np.float32)
    if w in ("sift1m", "c5shard", "sift1m-f32", "gist1m", "c5"):
        as_float = w in ("sift1m-f32", "gist1m")
        if batch == 0 and w != "c5" and args.n <= S.CHUNK:
            return S.make_latent16(n=args.n, d=d, m=m, seed=1234, as_float=as_float)[1]
        if batch == 0:  # the chunked stream's query set (make_latent16, n > 1M)
            rng0 = np.random.default_rng(1234)
            A = rng0.standard_normal((16, d)) / 4.0
            C = rng0.standard_normal((64, 16)) * 2.0
            return S._latent_draw(np.random.default_rng((1234, 0x51E7)), A, C, m, d, as_float)
        return S.make_latent16_queries(m=m, d=d, batch=batch, seed=1234, as_float=as_float)
    if w == "deep10m":
        if batch == 0:
            return S.make_deep_like(args.n, m, d=d)[1]
        return S.make_deep_like_queries(m, d=d, batch=batch)
    raise ValueError(w)


def c5_shard_rows(args, i: int):
    """Shard i of the C5 index: n/8 latent16 rows from shard stream i (shard 0
    = make_latent16's chunked base); dataset ids i * n/8 ... (i + 1) * n/8 - 1."""
    from paper_1912_01059_b200.synthetic import make_latent16_shard

    per = args.n // args.shards
    return make_latent16_shard(n=per, d=args.d, shard=i, seed=1234), np.arange(i * per, (i + 1) * per,
                                                                                dtype=np.int32)


def recall_at(ids, gt_first, k):
    return float(np.mean((ids[:, :k] == gt_first[:, None]).any(axis=1)))


def k_recall_at(ids, gt, k):
    return float(np.mean([len(set(ids[i, :k].tolist()) & set(gt[i, :k].tolist())) / k for i in range(len(ids))]))


# the reference's QueryConfig cache (prioq_size, visited_size) first; larger
# ones only when no tau reaches the target with it (C4: the searches end on
# an empty queue, not on the stopping rule, so tau alone cannot get there)
CACHES = [(256, 512), (512, 1024), (1024, 2048), (2048, 4096)]
CACHE_TAUS = [0.6, 1.0, 1.5, 2.0]


def qconfig(row, ga):
    # the reference's max_iterations (1000) with its default cache; a larger
    # cache needs proportionally more steps (C4 at prioq 1024: mean T ~ 1050)
    return ga.QueryConfig(k_out=10, tau=row["tau"], prioq_size=row["prioq_size"], visited_size=row["visited_size"],
                          max_iterations=1000 if row["prioq_size"] <= 256 else 4 * row["prioq_size"])


def choose_tau(query_fn, gt_ids, fixed, target):
    """Smallest tau with R@10 >= target: the coarse sweep TAUS, then steps of
    0.01 between the last tau below the target and the first one above it
    ("finer steps near the R@10 = 0.99 crossing"); if the default
    cache never gets there, the next larger cache of CACHES.
    query_fn(tau, prioq, visited) -> (ids, counters).  Returns (row, sweep,
    reached); row carries tau, prioq_size and visited_size."""
    sweep = []

    def run(tau, pq, vs):
        ids, cnt = query_fn(tau, pq, vs)
        row = {"tau": tau, "prioq_size": pq, "visited_size": vs, "R@1": recall_at(ids, gt_ids[:, 0], 1),
               "R@10": recall_at(ids, gt_ids[:, 0], 10), "kR@10": k_recall_at(ids, gt_ids, 10),
               "V": float(cnt[:, 0].mean()), "T": float(cnt[:, 1].mean())}
        sweep.append(row)
        return row

    for ci, (pq, vs) in enumerate(CACHES if fixed is None else CACHES[:1]):
        prev = None
        for tau in ([fixed] if fixed is not None else (TAUS if ci == 0 else CACHE_TAUS)):
            row = run(tau, pq, vs)
            if row["R@10"] >= target:
                if prev is not None:
                    for k in range(1, int(round((tau - prev) * 100))):
                        fine = run(round(prev + 0.01 * k, 2), pq, vs)
                        if fine["R@10"] >= target:
                            return fine, sweep, True
                return row, sweep, True
            prev = tau
    best = max(sweep, key=lambda r: r["R@10"])
    return best, sweep, False


def recall_queries(args, batches):
    """The queries tau is chosen on (both arms): every query of every timed
    batch for the uint8 workloads (exact ground truth on the tensor cores is
    cheap), a subsample of batch 0 for the float ones."""
    m = batches[0].shape[0]
    if args.workload in ("c1", "sift1m"):
        gt_m = min(args.gt_queries or m, m)
        return np.ascontiguousarray(np.concatenate([b_[:gt_m] for b_ in batches]))
    return np.ascontiguousarray(batches[0][:min(args.gt_queries or 1000, m)])


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.first = threading.Event()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])
            self.first.set()

    def wait_first(self, timeout: float = 5.0):
        if self.proc is not None:
            self.first.wait(timeout)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ dist
class Dist:
    def __init__(self, torch):
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # GGNN_DIST_BACKEND=gloo lets several ranks share one GPU (functional
        # runs of the multi-rank paths on a 1-GPU box); the product path is NCCL
        self.backend = os.environ.get("GGNN_DIST_BACKEND", "nccl")
        self.device = self.local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(self.device)
        self.on = self.world > 1
        if self.on:
            import torch.distributed as dist

            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
            else:
                dist.init_process_group(self.backend)
            self.dist = dist

    def barrier(self):
        if self.on:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if not self.on:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, v):
        if not self.on:
            return [v]
        out = [None] * self.world
        self.dist.all_gather_object(out, v)
        return out

    def close(self):
        if self.on:
            self.dist.destroy_process_group()


def _peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        return float(json.loads(f.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return 6650.0, "fallback 6650 GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def _bytes(cnt, d, e, k, k_out=10):
    """Algorithmic bytes of a query batch from its V / T counters:
    sum over queries of V*d*e + T*(4k+4) + d*e + 8*k_out."""
    c = np.asarray(cnt, dtype=np.int64)
    return int((c[:, 0] * d * e + c[:, 1] * (4 * k + 4) + d * e + 8 * k_out).sum())


def _traffic(workload):
    """ncu dram__bytes (read + write) per launch of the query kernel of THIS
    workload, from the per-workload capture under profiles/ (or null)."""
    f = ROOT / "profiles" / f"query_kernel_ncu_{workload}.json"
    if f.exists():
        j = json.loads(f.read_text())
        return j.get("dram_bytes_per_launch"), str(f.relative_to(ROOT))
    return None, f"no ncu capture for {workload} under profiles/"


def _leaf_tensor_pipe():
    f = ROOT / "profiles" / "leaf_knn_tensor_pipe.json"
    return json.loads(f.read_text()) if f.exists() else None


# --------------------------------------------------------- CPU baseline
# The reference's own query path on this box's host cores, one process per
# core (threads do not scale under the GIL).  Every worker loads
# the GPU-built graph with the REFERENCE's load_index (GGNN v1 file written by
# this package's save_index) and imports nothing but graphann_ref and numpy.
_REF = None


def _ref_module():
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    import graphann_ref as R  # noqa: E402

    return R


def _ref_init(root):
    global _REF
    R = _ref_module()
    root = Path(root)
    meta = json.loads((root / "meta.json").read_text())
    h = R.load_index(root / "index.ggnn")
    h.attach(R.Dataset(np.load(root / "base.npy", mmap_mode="r")))
    _REF = (R, h, meta, np.load(root / "queries.npy", mmap_mode="r"))


def _ref_run(job):
    """The reference's batch_query on a query slice (timed inside the worker)."""
    lo, hi = job
    R, h, meta, Q = _REF
    q = np.ascontiguousarray(Q[lo:hi])
    t0 = time.perf_counter()
    res = R.batch_query(h, q, R.QueryConfig(k_out=10, tau=meta["tau"], prioq_size=meta["prioq_size"],
                                            visited_size=meta["visited_size"],
                                            max_iterations=meta["max_iterations"]), threads=1)
    dt = time.perf_counter() - t0
    ids = np.stack([np.pad(r.ids, (0, 10 - len(r.ids)), constant_values=-1) for r in res])
    return dt, ids


class RefPool:
    def __init__(self, root: Path, nq_total: int, procs=None):
        import multiprocessing as mp

        self.root, self.nq = root, nq_total
        self.procs = procs or os.cpu_count() or 1
        self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_ref_init, initargs=(str(root),))
        probe = min(20, nq_total)
        dt, _ = self.pool.map(_ref_run, [(0, probe)])[0]
        self.per_q = dt / probe
        self.tau = json.loads((root / "meta.json").read_text())["tau"]

    def sample(self, target_seconds: float) -> dict:
        per_proc = max(1, int(target_seconds / max(self.per_q, 1e-6)))
        per_proc = min(per_proc, max(1, self.nq // self.procs))
        jobs = [(i * per_proc, (i + 1) * per_proc) for i in range(self.procs) if (i + 1) * per_proc <= self.nq]
        out = self.pool.map(_ref_run, jobs, chunksize=1)
        inner = max(o[0] for o in out)
        nq = sum(hi - lo for lo, hi in jobs)
        return {"value": nq / inner, "unit": UNIT, "cores": len(jobs), "kind": "reference",
                "sample": f"{nq} queries ({len(jobs)} processes x {per_proc}) of batch 0 on the GPU-built graph "
                          f"(GGNN v1 file read by the reference's load_index), reference graphann.batch_query "
                          f"(compiled _core, threads=1 per process), tau={self.tau}",
                "ids": np.concatenate([o[1] for o in out]), "n": nq}

    def close(self):
        self.pool.terminate()
        self.pool.join()


def export_index(h, base, Q, meta: dict) -> Path:
    """GGNN v1 file + base / query arrays for the reference's worker processes."""
    import paper_1912_01059_b200 as ga

    root = Path(tempfile.mkdtemp(prefix="ggnn_ref_", dir="/dev/shm" if os.path.isdir("/dev/shm") else None))
    ga.save_index(h, root / "index.ggnn")
    np.save(root / "base.npy", np.ascontiguousarray(base, dtype=np.float32))
    np.save(root / "queries.npy", np.ascontiguousarray(Q, dtype=np.float32))
    (root / "meta.json").write_text(json.dumps(meta))
    return root


_REF_BUILD_SNIPPET = r"""
import sys, time, json, numpy as np
sys.path.insert(0, sys.argv[1])
import graphann_ref as R
X = np.load(sys.argv[2])
t0 = time.perf_counter()
h, st = R.build(R.Dataset(X), R.BuildConfig(seed=7), threads=1)
print(json.dumps({"seconds": time.perf_counter() - t0, "build_seconds": st.build_seconds, "n": int(X.shape[0])}))
"""


def start_reference_build(base_sub) -> tuple:
    """The reference's own CPU build (graphann.build, threads=1) of `base_sub`
    in a background process that imports only graphann_ref; returns a handle
    for finish_reference_build."""
    if not (ROOT / "oracle" / "_ref" / "graphann_ref").exists():
        return None
    f = tempfile.NamedTemporaryFile(suffix=".npy", delete=False)
    np.save(f, np.ascontiguousarray(base_sub, dtype=np.float32))
    f.close()
    p = subprocess.Popen([sys.executable, "-c", _REF_BUILD_SNIPPET, str(ROOT / "oracle" / "_ref"), f.name],
                         stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    return p, f.name


def finish_reference_build(handle, timeout=600):
    if handle is None:
        return None
    p, path = handle
    try:
        out, err = p.communicate(timeout=timeout)
        return json.loads(out.strip().splitlines()[-1]) if p.returncode == 0 else {"error": err[-300:]}
    except Exception as exc:  # noqa: BLE001 -- a baseline must never kill the bench
        p.kill()
        return {"error": repr(exc)}
    finally:
        os.unlink(path)


# ------------------------------------------------------------------ main
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)  # never imports torch or this package in this process
    import torch

    dist = Dist(torch)
    if args.prep_reference:
        return prep_reference(args, torch)
    if args.shards is not None and (args.workload == "c5" or dist.world > 1):
        return run_sharded(args, dist, torch)
    return run_index(args, dist, torch)


def build_index(ga, base, torch):
    """Warm process (a small build first loads the kernels and grows the
    allocators), then the timed index build."""
    cfg = ga.BuildConfig(seed=7)
    warm_n = min(base.shape[0] // 4, 50_000)
    t_w = time.perf_counter()
    ga.build(ga.Dataset(np.ascontiguousarray(base[:warm_n])), cfg)
    torch.cuda.synchronize()
    warm_s = time.perf_counter() - t_w
    h, bstats = ga.build(ga.Dataset(base), cfg, accounting=True)
    return h, bstats, warm_n, warm_s


def run_index(args, dist, torch):
    """One index per rank (N = 1: the headline; N > 1: query-parallel
    replicas, each rank answering its own fresh batches)."""
    import paper_1912_01059_b200 as ga
    from paper_1912_01059_b200 import _native as N
    from paper_1912_01059_b200.device import device_hierarchy
    from paper_1912_01059_b200.search import _qflags

    rank, G = dist.rank, dist.world
    m = args.queries
    base = make_base(args)
    B = max(1, min(args.batches, args.steps))
    batches = [make_queries(args, rank * B + b) for b in range(B)]
    Q = batches[0]
    dist.barrier()
    h, bstats, warm_n, warm_s = build_index(ga, base, torch)
    build_s = dist.max(bstats.build_seconds)
    ds = h.dataset

    # ---- recall: same-run exact ground truth on batch 0 -----------------
    torch.cuda.synchronize()
    t_gt = time.perf_counter()
    # tau is chosen on the canonical batches 0 .. B-1 on every rank (replicas
    # then all run the same tau; rank r > 0 times its own batches r*B ...)
    QG = recall_queries(args, batches if rank == 0 else [make_queries(args, b) for b in range(B)])
    gt_ids, _ = ga.search.exact_knn(ds, QG, 10)
    gt_s = time.perf_counter() - t_gt

    def qfn(tau, pq, vs):
        r = ga.query_arrays(h, QG, qconfig({"tau": tau, "prioq_size": pq, "visited_size": vs}, ga))
        return r.ids, r.counters

    chosen, sweep, reached = choose_tau(qfn, gt_ids, args.tau, args.target)
    tau = chosen["tau"]
    qcfg = qconfig(chosen, ga)

    # ---- device-resident kernel timing (value) ---------------------------
    dh = device_hierarchy(h)
    dv = dh.vectors
    dqs = [dv.queries(b_) for b_ in batches]  # every batch uploaded before timing (inputs resident in HBM)
    ids = N.empty((m, 10), torch.int32)
    dists = N.empty((m, 10), torch.float64)
    cnts = [N.empty((m, 5), torch.int32) for _ in range(B)]
    params = N.search_params(10, qcfg.prioq_size, qcfg.visited_size, tau, qcfg.max_iterations, _qflags(dh, False))

    def launch(i, stream_p, out=None):
        o = out or (ids, dists, cnts[i % B])
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(dqs[i % B][1]), N.ctypes.byref(params), dh.d_nn1_max,
               N.ptr(o[0]), N.ptr(o[1]), N.ptr(o[2]), None, 0, stream_p)

    stream = torch.cuda.current_stream()
    sp = N.P(stream.cuda_stream)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        clocks.wait_first()
        # warm-up: at least W steps and 0.5 s of load (the clock samples see
        # the GPU busy before the timed region starts)
        t_w = time.perf_counter()
        done = 0
        while done < args.warmup or time.perf_counter() - t_w < 0.5:
            launch(done, sp)
            done += 1
            if done % 8 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        n_launch0 = N.load().ggnn_kernel_launches()
        evs[0].record(stream)
        for i in range(args.steps):
            launch(i, sp)
            evs[i + 1].record(stream)
        n_launches = N.load().ggnn_kernel_launches() - n_launch0  # this library's kernels in the timed region
        torch.cuda.synchronize()
    dist.barrier()
    t_total = evs[0].elapsed_time(evs[-1]) / 1e3
    t_max = dist.max(t_total)
    per_launch = [evs[i].elapsed_time(evs[i + 1]) / 1e3 for i in range(args.steps)]
    value = G * m * args.steps / t_max
    e = 1 if dv.exact_integers else 4
    kk = dh.layers[0].k
    batch_bytes = [_bytes(c.cpu().numpy(), args.d, e, kk) for c in cnts]
    bytes_per_launch = float(np.mean([batch_bytes[i % B] for i in range(args.steps)]))
    avg_launch = float(np.mean(per_launch))
    peak, peak_src = _peak()
    achieved = bytes_per_launch / avg_launch / 1e9
    traffic, traffic_src = _traffic(args.workload)

    # serving-loop view (beside, not the headline): two batches in flight on
    # two streams, so batch i+1 fills the SMs while batch i's last wave drains
    pipe_streams = (torch.cuda.Stream(), torch.cuda.Stream())
    pipe_out = [(N.empty((m, 10), torch.int32), N.empty((m, 10), torch.float64), N.empty((m, 5), torch.int32))
                for _ in range(2)]
    for i in range(4):
        launch(i, N.P(pipe_streams[i & 1].cuda_stream), pipe_out[i & 1])
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for s_ in pipe_streams:
        s_.wait_stream(stream)
    for i in range(args.steps):
        launch(i, N.P(pipe_streams[i & 1].cuda_stream), pipe_out[i & 1])
    for s_ in pipe_streams:
        stream.wait_stream(s_)
    p1.record(stream)
    torch.cuda.synchronize()
    t_pipe = dist.max(p0.elapsed_time(p1) / 1e3)
    pipelined = {"qps": G * m * args.steps / t_pipe, "ms_per_batch": t_pipe / args.steps * 1e3,
                 "how": "the same fresh batches, two streams, two batches in flight (not the headline)"}

    # ---- end to end through the public API (host buffers) --------------
    # each step's batch sits in page-locked host memory; results come back as
    # fresh host arrays
    pinned = []
    for b_ in batches:
        t_ = torch.empty(b_.shape, dtype=torch.float32, pin_memory=True)
        t_.copy_(torch.from_numpy(np.ascontiguousarray(b_, dtype=np.float32)))
        pinned.append(t_.numpy())
    # (at least 20 untimed calls: the first few dozen host-side calls of a
    # process run measurably slower -- allocator and interpreter warm-up)
    for i in range(max(20, args.warmup)):  # as the timed loop: the previous result stays alive
        out = ga.query_arrays(h, pinned[i % B], qcfg)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    call_t = []
    for i in range(args.steps):
        c0 = time.perf_counter()
        out = ga.query_arrays(h, pinned[i % B], qcfg)
        call_t.append(time.perf_counter() - c0)
    torch.cuda.synchronize()
    e2e_t = dist.max(time.perf_counter() - t0)
    out0 = ga.query_arrays(h, pinned[0], qcfg)
    e2e = {"value": G * m * args.steps / e2e_t, "unit": UNIT, "h2d_bytes_per_step": int(pinned[0].nbytes),
           "d2h_bytes_per_step": int(out.ids.nbytes + out.dists.nbytes + out.counters.nbytes + 4),
           "api": "paper_1912_01059_b200.query_arrays(h, numpy float32 queries in pinned memory) -> host arrays",
           "call_ms": {"min": round(min(call_t) * 1e3, 3), "median": round(float(np.median(call_t)) * 1e3, 3),
                       "max": round(max(call_t) * 1e3, 3)}}

    # ---- CPU baselines (rank 0, N == 1) -------------------------------
    cpu, ref_build_res = None, None
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        if (ROOT / "oracle" / "_ref" / "graphann_ref").exists():
            import shutil

            root = export_index(h, base, Q, {"tau": tau, "prioq_size": qcfg.prioq_size,
                                             "visited_size": qcfg.visited_size,
                                             "max_iterations": qcfg.max_iterations})
            try:
                pool = RefPool(root, m)
                try:
                    cpu = pool.sample(args.cpu_seconds)
                finally:
                    pool.close()
            finally:
                shutil.rmtree(root, ignore_errors=True)
            ref_ids = cpu.pop("ids")
            cpu["ids_equal_to_gpu"] = float(np.mean(np.all(ref_ids == out0.ids[: cpu.pop("n")], axis=1)))
        else:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": "oracle/_ref not built on this box"}
    if rank == 0 and G == 1 and not args.no_ref_build:
        # the reference's CPU build of a 10k subsample, after every timed
        # section (it runs on one host core in a process of its own)
        ref_build_res = finish_reference_build(start_reference_build(base[:10_000]))
    ref_build_info = None
    if ref_build_res is not None:
        sub = ga.Dataset(np.ascontiguousarray(base[:10_000]))
        _, gst = ga.build(sub, ga.BuildConfig(seed=7))
        ref_build_info = {"reference_cpu_seconds": ref_build_res.get("build_seconds"),
                          "gpu_seconds_same_points": gst.build_seconds, "points": 10_000,
                          "how": "graphann.build(BuildConfig(seed=7), threads=1) of the workload's first 10k "
                                 "points in a background process (graphann_ref only) vs this package's build of "
                                 "the same points", **({"error": ref_build_res["error"]}
                                                      if "error" in ref_build_res else {})}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8" if dv.exact_integers else "f32",
        "data": f"synthetic, seed 1234: {workload_desc(args)}; {B} distinct query batches of {m}",
        "config": config_of(args, tau, qcfg.prioq_size, qcfg.visited_size, qcfg.max_iterations),
        "build_seconds": build_s,
        "e2e": e2e,
        "gpu_launches": int(n_launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": bytes_per_launch, "kernel_ms": avg_launch * 1e3,
                     "kernel": f"one ggnn_query_batch launch ({'uint8' if dv.exact_integers else 'float32'} table): "
                               "pilot query_kernel + park_order_kernel + resume_kernel rounds when the batch "
                               "is >= 1.5 waves (longest-first schedule), one query_kernel otherwise",
                     "peak_source": peak_src},
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "details": {
            "recall_queries": int(QG.shape[0]), "recall": {k: chosen[k] for k in ("R@1", "R@10", "kR@10")},
            "recall_target_reached": reached, "mean_visited": chosen["V"], "mean_steps": chosen["T"],
            "tau_sweep": sweep, "ground_truth_seconds": gt_s,
            "build_note": f"warm process: a {warm_n}-point build ran first ({warm_s:.2f} s, module loading and "
                          f"allocator growth); build_seconds = the full index build after it",
            "build_phase_seconds_top": dict(sorted(bstats.phase_seconds.items(), key=lambda kv: -kv[1])[:6]),
            "build_accounting": bstats.accounting_summary(args.d, e),
            "leaf_knn_tensor_pipe": _leaf_tensor_pipe(),
            "reference_build": ref_build_info,
            "two_batches_in_flight": pipelined,
            "parallelism": ("one index" if G == 1 else
                            f"query-parallel replicas x{G}: every rank holds the whole index and answers its own "
                            f"fresh batches (no data-path collective)"),
            "l2": f"inputs larger than L2 (vectors {base.nbytes // (4 if dv.exact_integers else 1) >> 20} MB + "
                  f"adjacency {args.n * 96 >> 20} MB on the device)" if args.n >= 1_000_000 else
                  "index smaller than L2 (c1)"},
    }
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            Path(args.out).write_text(s + "\n")
    dist.close()


def run_sharded(args, dist, torch):
    """Sharded workloads: c5 (a fixed 8-shard index over N ranks, any N) and
    deep10m with N > 1 (N shards on N GPUs).  A step = the replicated batch
    searched on every local shard into its block (ids globalized), one
    all-gather of the blocks (NCCL; none at N = 1), the GPU k-way merge."""
    import paper_1912_01059_b200 as ga
    from paper_1912_01059_b200 import _native as N
    from paper_1912_01059_b200.distributed import ShardGroup
    from paper_1912_01059_b200.search import _params, _qflags
    from paper_1912_01059_b200.device import device_hierarchy
    from paper_1912_01059_b200.shard import block_layout, block_pointers

    G, rank = dist.world, dist.rank
    m = args.queries
    n_shards = args.shards if args.shards != "ranks" else G
    if args.workload == "deep10m":
        base_all = make_base(args)
        perm = np.random.default_rng(7).permutation(args.n).astype(np.int32)  # shard.py:54-65, BuildConfig seed 7
        size = -(-args.n // n_shards)

        def loader(i):
            gid = perm[i * size:(i + 1) * size]
            return ga.Dataset(base_all[gid].copy()), gid
    else:
        def loader(i):
            rows, gid = c5_shard_rows(args, i)
            return ga.Dataset(rows), gid
    B = max(1, min(args.batches, args.steps))
    batches = [make_queries(args, b) for b in range(B)]  # replicated: every rank searches every batch
    Q = batches[0]
    # warm process (kernels loaded, allocators grown), then this rank's shard
    # builds; build_seconds = the builds alone (shard data generation excluded)
    from paper_1912_01059_b200.synthetic import make_deep_like, make_latent16

    warm = (make_deep_like(50_000, 1, d=args.d)[0] if args.workload == "deep10m"
            else make_latent16(n=50_000, d=args.d, m=1)[0])
    ga.build(ga.Dataset(warm), ga.BuildConfig(seed=7))
    torch.cuda.synchronize()
    dist.barrier()
    grp = ShardGroup.from_local_shards(loader, n_shards, ga.BuildConfig(seed=7))
    build_s = dist.max(sum(st.build_seconds for st in grp.build_stats))
    S = grp.per_rank
    gt_m = min(args.gt_queries or 1000, m)
    gt_ids, _ = grp.exact_arrays(Q[:gt_m], 10)

    def qfn(tau, pq, vs):
        r = grp.query_arrays(Q[:gt_m], qconfig({"tau": tau, "prioq_size": pq, "visited_size": vs}, ga))
        return r.ids, r.counters

    chosen, sweep, reached = choose_tau(qfn, gt_ids, args.tau, args.target)
    tau = chosen["tau"]
    qcfg = qconfig(chosen, ga)

    dhs = [device_hierarchy(h) for h, _ in grp.shards]
    dqs = [[dh.vectors.queries(b_) for dh in dhs] for b_ in batches]
    bb = block_layout(m, 10)[0]
    send = N.empty((S * bb,), torch.uint8)
    recv = N.empty((n_shards * bb,), torch.uint8) if G > 1 else send
    out_ids = N.empty((m, 10), torch.int32)
    out_d = N.empty((m, 10), torch.float64)
    out_c = N.empty((m, 5), torch.int32)
    params = [_params(qcfg, _qflags(dh, False)) for dh in dhs]
    stream = torch.cuda.current_stream()
    qev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    if args.exchange == "p2p" and G > 1 and S != 1:
        raise SystemExit("--exchange p2p needs one shard per rank (the fused exchange pushes one block per rank)")
    x = grp.p2p(m, 10) if (args.exchange == "p2p" and G > 1) else None

    def step(i, timed=False):
        if x is not None:  # fused: push search + signal, then wait + merge
            if timed:
                qev[2 * i].record(stream)
            x.search_push(grp.h, batches[i % B], qcfg)
            if timed:
                qev[2 * i + 1].record(stream)
            x.merge_into(out_ids, out_d, out_c)
            return
        if timed:
            qev[2 * i].record(stream)
        for s, dh in enumerate(dhs):
            ids_p, dists_p, cnt_p = block_pointers(send, s, m, 10)
            qs = dqs[i % B][s][1]
            N.call("ggnn_query_batch", N.ctypes.byref(dh.vectors.struct), N.ctypes.byref(dh.layers[0].struct),
                   N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params[s]), dh.d_nn1_max, ids_p,
                   dists_p, cnt_p, None, 0, N.stream_ptr())
            N.call("ggnn_shard_globalize", ids_p, m * 10, N.ptr(grp.gid_dev(s)), int(grp.shards[s][1].shape[0]),
                   N.stream_ptr())
        if timed:
            qev[2 * i + 1].record(stream)
        grp.exchange(send, recv)
        N.call("ggnn_shard_merge", N.ptr(recv), n_shards, m, 10, 10, N.ptr(out_ids), N.ptr(out_d), N.ptr(out_c),
               N.stream_ptr())

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        clocks.wait_first()
        for w in range(max(args.warmup, 8)):  # a FIXED count on every rank (each step is a collective)
            step(w)
            if w % 8 == 7:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        n_launch0 = N.load().ggnn_kernel_launches()
        evs[0].record(stream)
        for i in range(args.steps):
            step(i, timed=True)
            evs[i + 1].record(stream)
        n_launches = N.load().ggnn_kernel_launches() - n_launch0
        torch.cuda.synchronize()
    dist.barrier()
    if x is not None:
        x.check()
    t_max = dist.max(evs[0].elapsed_time(evs[-1]) / 1e3)
    value = m * args.steps / t_max  # delivered queries: every step answers m queries over the whole index
    search_s = float(np.mean([qev[2 * i].elapsed_time(qev[2 * i + 1]) for i in range(args.steps)])) / 1e3
    # QPS_1 estimate from this run: one GPU searching all n_shards shards in
    # turn = the sum of every shard's search time (each rank times its own)
    # plus this step's exchange-free merge
    all_search = dist.gather(search_s)
    qps1_est = m / sum(all_search) if G > 1 else value
    e = 1 if dhs[0].vectors.exact_integers else 4
    coff = block_layout(m, 10)[2]
    own = np.concatenate([send[s * bb + coff: s * bb + coff + m * 20].view(torch.int32).view(m, 5).cpu().numpy()
                          for s in range(S)]) if x is None else x.local_cnt.cpu().numpy()
    bpl = _bytes(own, args.d, e, dhs[0].layers[0].k) / S
    peak, peak_src = _peak()
    achieved = bpl / (search_s / S) / 1e9

    pinned = []
    for b_ in batches:
        t_ = torch.empty(b_.shape, dtype=torch.float32, pin_memory=True)
        t_.copy_(torch.from_numpy(np.ascontiguousarray(b_, dtype=np.float32)))
        pinned.append(t_.numpy())
    exch = args.exchange if G > 1 else "nccl"
    for i in range(max(1, args.warmup)):
        out = grp.query_arrays(pinned[i % B], qcfg, exchange=exch)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        out = grp.query_arrays(pinned[i % B], qcfg, exchange=exch)
    torch.cuda.synchronize()
    e2e_t = dist.max(time.perf_counter() - t0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8" if e == 1 else "f32",
        "data": f"synthetic, seed 1234: {workload_desc(args)}; {B} distinct query batches of {m} (replicated)",
        "config": config_of(args, tau, qcfg.prioq_size, qcfg.visited_size, qcfg.max_iterations),
        "build_seconds": build_s,
        "e2e": {"value": m * args.steps / e2e_t, "unit": UNIT, "h2d_bytes_per_step": int(pinned[0].nbytes),
                "d2h_bytes_per_step": int(out.ids.nbytes + out.dists.nbytes + out.counters.nbytes),
                "api": "ShardGroup.query_arrays(numpy queries) -> host arrays (every rank)"},
        "gpu_launches": int(n_launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "traffic_source": "per-shard query kernel (no ncu capture of this workload)",
                     "algorithmic_bytes_per_launch": bpl, "kernel_ms": search_s / S * 1e3,
                     "kernel": "query_kernel on one shard (rank 0 mean)", "peak_source": peak_src},
        "clocks": clocks.summary(),
        "cpu_baseline": None,
        "details": {
            "shards": n_shards, "shards_per_rank": S,
            "recall_queries": gt_m, "recall": {k: chosen[k] for k in ("R@1", "R@10", "kR@10")},
            "recall_target_reached": reached, "tau_sweep": sweep,
            "mean_visited_all_shards": chosen["V"], "mean_steps_all_shards": chosen["T"],
            "build_seconds_note": "this rank's shard builds, max over ranks (shards of a rank one after the other)",
            "qps_1_estimate": qps1_est,
            "efficiency_vs_qps_1_estimate": value / (G * qps1_est) if G > 1 else 1.0,
            "qps_1_note": ("one GPU searching all shards in turn, estimated in this run as m / (sum over every "
                           "shard's search time) -- the exchange and merge excluded" if G > 1 else
                           "this run IS QPS_1: one GPU searching all shards in turn"),
            "parallelism": (f"sharded {n_shards} over {G} GPUs: " +
                            (f"NCCL all_gather_into_tensor of {S * bb} B/rank + ggnn_shard_merge" if x is None else
                             "fused exchange (query kernel stores each finished row into every peer's receive "
                             "block over CUDA IPC) + ggnn_shard_merge_wait") if G > 1 else
                            f"one GPU, {n_shards} shards searched in turn + ggnn_shard_merge")},
    }
    if rank == 0:
        js = json.dumps(line)
        print(js, flush=True)
        if args.out:
            Path(args.out).write_text(js + "\n")
    grp.close()
    dist.close()


# ------------------------------------------------------------ reference arm
def prep_reference(args, torch):
    """Internal (a subprocess of --impl reference): build the index on the
    GPU, choose tau exactly like the GPU arm, write the GGNN v1 file and the
    arrays the reference's worker processes read, then exit."""
    import paper_1912_01059_b200 as ga

    root = Path(args.prep_reference)
    base = make_base(args)
    B = max(1, min(args.batches, args.steps))
    batches = [make_queries(args, b) for b in range(B)]  # the GPU arm's (rank 0's) batches
    Q = batches[0]
    h, _, _, _ = build_index(ga, base, torch)
    QG = recall_queries(args, batches)
    gt_ids, _ = ga.search.exact_knn(h.dataset, QG, 10)

    def qfn(tau, pq, vs):
        r = ga.query_arrays(h, QG, qconfig({"tau": tau, "prioq_size": pq, "visited_size": vs}, ga))
        return r.ids, r.counters

    chosen, sweep, reached = choose_tau(qfn, gt_ids, args.tau, args.target)
    qc = qconfig(chosen, ga)
    ga.save_index(h, root / "index.ggnn")
    np.save(root / "base.npy", np.ascontiguousarray(base, dtype=np.float32))
    np.save(root / "queries.npy", np.ascontiguousarray(Q, dtype=np.float32))
    (root / "meta.json").write_text(json.dumps({"tau": chosen["tau"], "prioq_size": qc.prioq_size,
                                                "visited_size": qc.visited_size,
                                                "max_iterations": qc.max_iterations, "reached": reached,
                                                "recall_gpu_same_tau": {k: chosen[k] for k in
                                                                        ("R@1", "R@10", "kR@10")}}))


def run_reference(args):
    """--impl reference: the reference's own CPU query path (graphann
    batch_query, compiled _core) on this box's host cores, process-parallel,
    a bounded sample of the same workload per step, on the same graph the
    GPU arm searches (built on the GPU by a preparation SUBPROCESS and read
    with the reference's load_index; this process imports only numpy and,
    in its workers, graphann_ref).  c1 (configs[0]): the reference's CPU
    build is timed end to end as well."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if args.shards is not None and args.workload == "c5":
        print(json.dumps({"impl": "reference", "unavailable": "the reference's query_sharded over a 100M-point "
                          "8-shard index does not fit a bounded CPU sample; use the sift1m arm"}))
        return
    if not (ROOT / "oracle" / "_ref" / "graphann_ref").exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (compiled reference) not present"}))
        return
    import shutil

    root = Path(tempfile.mkdtemp(prefix="ggnn_ref_", dir="/dev/shm" if os.path.isdir("/dev/shm") else None))
    try:
        cmd = [sys.executable, str(ROOT / "bench.py"), "--prep-reference", str(root), "--workload", args.workload,
               "--points", str(args.n), "--dim", str(args.d), "--queries", str(args.queries), "--steps",
               str(args.steps), "--batches", str(args.batches)]
        if args.tau is not None:
            cmd += ["--tau", str(args.tau)]
        if args.gt_queries is not None:
            cmd += ["--gt-queries", str(args.gt_queries)]
        env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
        subprocess.run(cmd, check=True, env=env, stdout=subprocess.DEVNULL)
        meta = json.loads((root / "meta.json").read_text())
        tau = meta["tau"]
        build_info = None
        if args.workload == "c1" or not args.no_ref_build:
            base = np.load(root / "base.npy", mmap_mode="r")
            sub = base if args.workload == "c1" else base[:10_000]
            res = finish_reference_build(start_reference_build(sub), timeout=1800)
            build_info = {"reference_cpu_seconds": (res or {}).get("build_seconds"), "points": int(sub.shape[0]),
                          "how": "graphann.build(BuildConfig(seed=7), threads=1) in a process that imports only "
                                 "graphann_ref" + ("" if args.workload == "c1" else
                                                   " (a 10k-point subsample: the 1M build takes hours on a CPU)")}
        per_step = max(2.0, min(args.cpu_seconds, 180.0 / max(1, args.steps + args.warmup)))
        vals, info, pool = [], None, None
        try:
            pool = RefPool(root, args.queries)
            for i in range(args.warmup + args.steps):
                r = pool.sample(per_step)
                r.pop("ids")
                r.pop("n")
                if i >= args.warmup:
                    vals.append(r["value"])
                    info = r
        finally:
            if pool is not None:
                pool.close()
    finally:
        shutil.rmtree(root, ignore_errors=True)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": args.queries / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic, seed 1234: {workload_desc(args)}",
        "config": config_of(args, tau, meta["prioq_size"], meta["visited_size"], meta["max_iterations"]),
        "build_seconds": (build_info or {}).get("reference_cpu_seconds") if args.workload == "c1" else None,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "reference",
                         "sample": info["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "details": {"recall_gpu_same_tau": meta["recall_gpu_same_tau"], "recall_target_reached": meta["reached"],
                    "reference_build": build_info,
                    "graph": "built on the GPU by a preparation subprocess (untimed), saved as GGNN v1, read by "
                             "graphann.load_index in every worker"},
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
