"""GGNN B200 benchmark: QPS at R@10 >= 0.99 on SIFT1M-shaped data + build seconds.

Workload (BASELINE.json configs[1], "C2"): synthetic SIFT1M-shaped latent16
data (SURVEY.md 8d "G_B"), 1M x 128 integer-valued (stored losslessly as
uint8 on the device), 10k queries, k=10, BuildConfig(seed=7) defaults
(k=24, k_nn=12, s=32, g=4, refinements=2, tau_build=0.5).  tau is chosen in
the run: the smallest tau of a sweep whose R@10 (reference `recall_at`,
evaluate.py:60-76) against exact ground truth computed on the GPU in the same
run is >= 0.99.

A "step" is one batch of 10k queries through the query kernel with inputs
resident in HBM.  Multi-GPU: one process per GPU, every rank holds the full
1M index and answers its own 10k-query batch (queries are independent units;
no data-path collective), so `scaling` is "weak".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ggnn|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "queries/sec at R@10>=0.99 (SIFT1M-shape, k=10); index build seconds"
UNIT = "queries/s"
TAUS = [0.2, 0.25, 0.3, 0.35, 0.4, 0.45, 0.5, 0.55, 0.6, 0.7, 0.8]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ggnn", choices=["ggnn", "reference"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--d", type=int, default=None)
    ap.add_argument("--queries", type=int, default=10_000)
    ap.add_argument("--workload", default="sift1m", choices=["sift1m", "gist1m", "deep10m", "c5shard"],
                    help="sift1m = configs[1] (the metric's workload, default); gist1m / deep10m = the C3 / C4 "
                         "shapes on one GPU (ground truth on a query subsample)")
    ap.add_argument("--gt-queries", type=int, default=None, help="ground-truth subsample (default: all for sift1m, "
                    "1000 otherwise)")
    ap.add_argument("--tau", type=float, default=None, help="skip the sweep and use this tau")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1: NCCL all-gather after the search, or the fused peer-memory exchange")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    return ap.parse_args()


# ------------------------------------------------------------------ dist
class Dist:
    def __init__(self, torch, n_gpus):
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # GGNN_DIST_BACKEND=gloo lets several ranks share one GPU (functional
        # tests of the sharded path on a 1-GPU box); the product path is NCCL
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

    def close(self):
        if self.on:
            self.dist.destroy_process_group()


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
        """Block until nvidia-smi has produced its first sample (it takes a
        few hundred ms to start), so the samples cover the timed region."""
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


# ------------------------------------------------------------------ data
WORKLOADS = {
    "sift1m": "SIFT1M-shaped latent16 (SURVEY.md 8d G_B) {n}x{d} integer-valued (uint8 on the device)",
    "gist1m": "GIST1M-shaped float latent16 {n}x{d} (C3: no rounding, /255)",
    "deep10m": "Deep10M-shaped {n}x{d} clustered (1024 clusters), rows L2-normalised (C4)",
    "c5shard": "one SIFT100M shard: latent16 {n}x{d} integer-valued (uint8 on the device; C5 is 8 such shards)",
}


def make_workload(args):
    """(base, queries) of the chosen workload; sizes default to the config's."""
    from paper_1912_01059_b200.synthetic import make_latent16

    if args.workload in ("sift1m", "c5shard"):
        return make_latent16(n=args.n, d=args.d, m=args.queries, seed=1234)
    if args.workload == "gist1m":
        return make_latent16(n=args.n, d=args.d, m=args.queries, seed=1234, as_float=True)
    from paper_1912_01059_b200.data import gen_synthetic

    X = gen_synthetic(args.n + args.queries, args.d, seed=1234, law="clustered", clusters=1024).vectors
    X = X.astype(np.float64)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X = X.astype(np.float32)
    return X[:args.n].copy(), X[args.n:].copy()


def recall_at(ids, gt_first, k):
    return float(np.mean((ids[:, :k] == gt_first[:, None]).any(axis=1)))


def k_recall_at(ids, gt, k):
    return float(np.mean([len(set(ids[i, :k].tolist()) & set(gt[i, :k].tolist())) / k for i in range(len(ids))]))


def choose_tau(ga, h, Q, gt_ids, fixed):
    sweep = []
    taus = [fixed] if fixed is not None else TAUS
    chosen = None
    for tau in taus:
        res = ga.query_arrays(h, Q, ga.QueryConfig(k_out=10, tau=tau))
        row = {"tau": tau, "R@1": recall_at(res.ids, gt_ids[:, 0], 1), "R@10": recall_at(res.ids, gt_ids[:, 0], 10),
               "kR@10": k_recall_at(res.ids, gt_ids, 10), "V": float(res.counters[:, 0].mean()),
               "T": float(res.counters[:, 1].mean())}
        sweep.append(row)
        if chosen is None and row["R@10"] >= 0.99:
            chosen = row
            if fixed is None:
                break
    if chosen is None:
        chosen = sweep[-1]
    return chosen, sweep


# --------------------------------------------------------- CPU baseline
def export_graph(h, base, Q, tau):
    """Dump the GPU-built graph + workload as .npy files (shared, memory-mapped
    by every CPU worker) -- the same arrays GGNN v1 persists."""
    import tempfile

    root = Path(tempfile.mkdtemp(prefix="ggnn_cpu_", dir="/dev/shm" if os.path.isdir("/dev/shm") else None))
    np.save(root / "base.npy", np.ascontiguousarray(base, dtype=np.float32))
    np.save(root / "queries.npy", np.ascontiguousarray(Q, dtype=np.float32))
    for j, L in enumerate(h.layers):
        np.save(root / f"adj{j}.npy", L.adjacency)
        np.save(root / f"nnd{j}.npy", L.nn_dists)
        np.save(root / f"sym{j}.npy", L.sym_count)
        np.save(root / f"dnn1_{j}.npy", L.d_nn1)
        if j:
            np.save(root / f"tob{j}.npy", h.to_bottom[j])
    c = h.config
    meta = {"layers": h.num_layers, "s": h.s, "g": h.g, "k": c.k, "k_nn": c.k_nn, "k_sym": c.k_sym,
            "refinements": c.refinements, "tau_build": c.tau_build, "seed": c.seed,
            "stats": [h.stats.d_nn1_mean, h.stats.d_nn1_max], "tau": tau}
    (root / "meta.json").write_text(json.dumps(meta))
    return root


def _load_ref_hierarchy(root: Path):
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    import graphann_ref as R  # noqa: E402

    meta = json.loads((root / "meta.json").read_text())
    cfg = R.BuildConfig(k=meta["k"], k_nn=meta["k_nn"], k_sym=meta["k_sym"], s=meta["s"], g=meta["g"],
                        refinements=meta["refinements"], tau_build=meta["tau_build"], seed=meta["seed"])
    layers, tob = [], [None]
    for j in range(meta["layers"]):
        adj = np.load(root / f"adj{j}.npy", mmap_mode="r")
        L = R.AdjacencyLayer.__new__(R.AdjacencyLayer)
        L.node_count, L.k, L.k_nn = adj.shape[0], meta["k"], meta["k_nn"]
        L.k_sym = L.k - L.k_nn
        L.adjacency = adj
        L.nn_dists = np.load(root / f"nnd{j}.npy", mmap_mode="r")
        L.sym_count = np.load(root / f"sym{j}.npy", mmap_mode="r")
        L.d_nn1 = np.load(root / f"dnn1_{j}.npy", mmap_mode="r")
        layers.append(L)
        if j:
            tob.append(np.load(root / f"tob{j}.npy"))
    h = R.Hierarchy(layers, tob, meta["s"], meta["g"], cfg, R.GraphStats(*meta["stats"]),
                    dim=int(np.load(root / "base.npy", mmap_mode="r").shape[1]))
    h.attach(R.Dataset(np.load(root / "base.npy", mmap_mode="r")))
    return R, h, meta


_REF = None


def _ref_init(root):
    """Worker initializer: load the reference package and the exported graph once."""
    global _REF
    R, h, meta = _load_ref_hierarchy(Path(root))
    _REF = (R, h, meta, np.load(Path(root) / "queries.npy", mmap_mode="r"))


def _ref_run(job):
    """The reference's own batch_query on a query slice (timed inside the worker)."""
    lo, hi = job
    R, h, meta, Q = _REF
    q = np.ascontiguousarray(Q[lo:hi])
    t0 = time.perf_counter()
    res = R.batch_query(h, q, R.QueryConfig(k_out=10, tau=meta["tau"]), threads=1)
    dt = time.perf_counter() - t0
    ids = np.stack([np.pad(r.ids, (0, 10 - len(r.ids)), constant_values=-1) for r in res])
    return dt, ids


class RefPool:
    """Process-parallel reference batch_query (threads do not scale under the
    GIL): one process per host core, each holding the exported
    GPU-built graph, answering bounded query samples of the workload."""

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
                "sample": f"{nq} queries ({len(jobs)} processes x {per_proc}) of the same workload on the GPU-built "
                          f"graph, reference graphann.batch_query (compiled _core), tau={self.tau}",
                "ids": np.concatenate([o[1] for o in out]), "n": nq}

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_reference_qps(root: Path, nq_total: int, target_seconds: float, max_procs=None):
    pool = RefPool(root, nq_total, max_procs)
    try:
        return pool.sample(target_seconds)
    finally:
        pool.close()


# ------------------------------------------------------------------ main
DEFAULT_SHAPE = {"sift1m": (1_000_000, 128), "gist1m": (1_000_000, 960), "deep10m": (10_000_000, 96),
                 "c5shard": (12_500_000, 128)}


def main():
    args = parse()
    n0, d0 = DEFAULT_SHAPE[args.workload]
    args.n = args.n or n0
    args.d = args.d or d0
    import torch

    dist = Dist(torch, args.gpus)
    import paper_1912_01059_b200 as ga
    from paper_1912_01059_b200 import _native as N

    if args.impl == "reference":
        return run_reference(args, dist, ga)
    if dist.world > 1:
        return run_sharded(args, dist, ga, torch)

    base, Q = make_workload(args)
    ds = ga.Dataset(base)
    cfg = ga.BuildConfig(seed=7)
    # warm process: one small build first loads the kernels and grows the
    # allocators, so build_seconds is the index build itself
    warm_n = min(args.n // 4, 50_000)
    t_w = time.perf_counter()
    ga.build(ga.Dataset(np.ascontiguousarray(base[:warm_n])), cfg)
    torch.cuda.synchronize()
    warmup_build_s = time.perf_counter() - t_w
    dist.barrier()
    h, bstats = ga.build(ds, cfg)
    build_s = dist.max(bstats.build_seconds)

    torch.cuda.synchronize()
    t_gt = time.perf_counter()
    gt_m = args.gt_queries or (Q.shape[0] if args.workload == "sift1m" else min(1000, Q.shape[0]))
    gt_ids, _ = ga.search.exact_knn(ds, Q[:gt_m], 10)  # tcgen05 brute force for uint8 data
    gt_s = time.perf_counter() - t_gt
    chosen, sweep = choose_tau(ga, h, Q[:gt_m], gt_ids, args.tau)
    tau = chosen["tau"]
    qcfg = ga.QueryConfig(k_out=10, tau=tau)

    # ---- device-resident kernel timing (value) ------------------------
    from paper_1912_01059_b200.device import device_hierarchy
    from paper_1912_01059_b200.search import _qflags

    dh = device_hierarchy(h)
    dv = dh.vectors
    dq, qs = dv.queries(Q)
    m = Q.shape[0]
    ids = N.empty((m, 10), torch.int32)
    dists = N.empty((m, 10), torch.float64)
    cnt = N.empty((m, 5), torch.int32)
    params = N.search_params(10, qcfg.prioq_size, qcfg.visited_size, tau, qcfg.max_iterations, _qflags(dh, False))

    def step():
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max, N.ptr(ids),
               N.ptr(dists), N.ptr(cnt), None, 0, N.stream_ptr())

    stream = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        clocks.wait_first()
        # warm-up: at least W steps, and at least 0.5 s of load so the clock
        # samples see the GPU busy before the timed region starts
        t_w = time.perf_counter()
        done = 0
        while done < args.warmup or time.perf_counter() - t_w < 0.5:
            step()
            done += 1
            if done % 8 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    t_total = evs[0].elapsed_time(evs[-1]) / 1e3
    t_max = dist.max(t_total)
    per_launch = [evs[i].elapsed_time(evs[i + 1]) / 1e3 for i in range(args.steps)]
    value = args.gpus * m * args.steps / t_max
    c = cnt.cpu().numpy().astype(np.int64)
    e = 1 if dv.exact_integers else 4
    d = base.shape[1]
    kk = dh.layers[0].k
    bytes_per_launch = int((c[:, 0] * d * e + c[:, 1] * (4 * kk + 4) + d * e + 8 * 10).sum())
    avg_launch = float(np.mean(per_launch))
    peak, peak_src = _peak()
    achieved = bytes_per_launch / avg_launch / 1e9
    # serving-loop view (reported beside, not as `value`): two independent
    # batches in flight on two streams, so batch i+1's searches fill the SMs
    # while batch i's last wave drains
    pipe_streams = (torch.cuda.Stream(), torch.cuda.Stream())
    pipe_out = [(N.empty((m, 10), torch.int32), N.empty((m, 10), torch.float64), N.empty((m, 5), torch.int32))
                for _ in range(2)]

    def pipe_step(i):
        s_ = pipe_streams[i & 1]
        o = pipe_out[i & 1]
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max,
               N.ptr(o[0]), N.ptr(o[1]), N.ptr(o[2]), None, 0, N.P(s_.cuda_stream))

    for i in range(4):
        pipe_step(i)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for s_ in pipe_streams:
        s_.wait_stream(stream)
    for i in range(args.steps):
        pipe_step(i)
    for s_ in pipe_streams:
        stream.wait_stream(s_)
    p1.record(stream)
    torch.cuda.synchronize()
    t_pipe = dist.max(p0.elapsed_time(p1) / 1e3)
    pipelined = {"qps": args.gpus * m * args.steps / t_pipe, "ms_per_batch": t_pipe / args.steps * 1e3,
                 "how": "same batches, two streams, two batches in flight (not the headline)"}

    traffic = None
    prof = ROOT / "profiles" / "query_kernel_ncu.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")

    # ---- end to end through the public API (host buffers) --------------
    # the step's input batch sits in page-locked host memory (the contract's
    # "host->device copy ... from pinned host memory"); results come back as
    # fresh host arrays
    Q_pin = torch.empty(Q.shape, dtype=torch.float32, pin_memory=True)
    Q_pin.copy_(torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float32)))
    Q_host = Q_pin.numpy()
    for _ in range(max(1, args.warmup)):
        ga.query_arrays(h, Q_host, qcfg)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = ga.query_arrays(h, Q_host, qcfg)
    torch.cuda.synchronize()
    e2e_t = dist.max(time.perf_counter() - t0)
    e2e = {"value": args.gpus * m * args.steps / e2e_t, "unit": UNIT,
           "h2d_bytes_per_step": int(Q_host.nbytes),
           "d2h_bytes_per_step": int(out.ids.nbytes + out.dists.nbytes + out.counters.nbytes + 4),
           "api": "paper_1912_01059_b200.query_arrays(h, numpy float32 queries in pinned memory) -> host arrays; "
                  "one search launch overlapped with the chunked upload (ggnn_query_batch_host), rows narrowed to "
                  "uint8 in the kernel"}

    # ---- CPU baseline (rank 0, N == 1) ---------------------------------
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        if (ROOT / "oracle" / "_ref" / "graphann_ref").exists():
            import shutil

            root = export_graph(h, base, Q, tau)
            try:
                cpu = cpu_reference_qps(root, m, args.cpu_seconds)
            finally:
                shutil.rmtree(root, ignore_errors=True)
            ref_ids = cpu.pop("ids")
            cpu["ids_equal_to_gpu"] = float(np.mean(np.all(ref_ids == out.ids[: cpu.pop("n")], axis=1)))
        else:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": "oracle/_ref not built on this box"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8" if dv.exact_integers else "f32",
        "data": f"synthetic, seed 1234: {WORKLOADS[args.workload].format(n=args.n, d=args.d)}",
        "config": {"workload": f"{args.workload}: {WORKLOADS[args.workload].format(n=args.n, d=args.d)}, "
                               f"{m} queries/rank, k=10, k_build=24",
                   "recall_queries": gt_m,
                   "tau": tau, "recall": {k: chosen[k] for k in ("R@1", "R@10", "kR@10")},
                   "mean_visited": chosen["V"], "mean_steps": chosen["T"], "tau_sweep": sweep,
                   "build_seconds": build_s, "ground_truth_seconds": gt_s,
                   "build_note": f"warm process: a {warm_n}-point build ran first ({warmup_build_s:.2f} s, module "
                                 f"loading and allocator growth); build_seconds = the full index build after it",
                   "build_phase_seconds_top": dict(sorted(
                       bstats.phase_seconds.items(), key=lambda kv: -kv[1])[:6]),
                   "two_batches_in_flight": pipelined,
                   "parallelism": f"replicas x{args.gpus} (independent query batches)",
                   "l2": f"inputs larger than L2 (vectors {base.nbytes // (4 if dv.exact_integers else 1) >> 20} MB "
                         f"+ adjacency {args.n * 96 >> 20} MB on the device)"},
        "build_seconds": build_s,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algorithmic_bytes_per_launch": bytes_per_launch,
                     "kernel_ms": avg_launch * 1e3, "peak_source": peak_src},
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    if dist.rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            Path(args.out).write_text(s + "\n")
    dist.close()


def _peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        return float(json.loads(f.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return 6650.0, "fallback 6650 GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def _bytes_per_launch(cnt, d, e, k, k_out):
    c = cnt.astype(np.int64)
    return int((c[:, 0] * d * e + c[:, 1] * (4 * k + 4) + d * e + 8 * k_out).sum())


def run_sharded(args, dist, ga, torch):
    """N > 1: one 1M-point shard per GPU of an N-million-point latent16 index
    (shard 0 = the C2 data), the 10k-query batch replicated on every rank,
    each step = search (query kernel into the shard block) + id globalization
    + NCCL all-gather + GPU G-way merge.  Weak scaling: per-GPU work is fixed
    (m queries on one 1M shard); value counts shard-queries (N * m per step)."""
    from paper_1912_01059_b200 import _native as N
    from paper_1912_01059_b200.device import device_hierarchy
    from paper_1912_01059_b200.distributed import ShardGroup
    from paper_1912_01059_b200.search import _qflags
    from paper_1912_01059_b200.shard import block_layout, block_pointers
    from paper_1912_01059_b200.synthetic import make_latent16, make_latent16_shard

    G, r = dist.world, dist.rank
    _, Q = make_latent16(n=args.n, d=args.d, m=args.queries, seed=1234)
    base = make_latent16_shard(n=args.n, d=args.d, shard=r, seed=1234)
    ds = ga.Dataset(base)
    ga.build(ga.Dataset(np.ascontiguousarray(base[:min(args.n // 4, 50_000)])), ga.BuildConfig(seed=7))  # warm
    torch.cuda.synchronize()
    dist.barrier()
    h, bstats = ga.build(ds, ga.BuildConfig(seed=7))
    build_s = dist.max(bstats.build_seconds)
    grp = ShardGroup(h, np.arange(r * args.n, (r + 1) * args.n, dtype=np.int32))
    gt_ids, _ = grp.exact_arrays(Q, 10)
    sweep, chosen = [], None
    for tau in ([args.tau] if args.tau is not None else TAUS):
        res = grp.query_arrays(Q, ga.QueryConfig(k_out=10, tau=tau))
        row = {"tau": tau, "R@1": recall_at(res.ids, gt_ids[:, 0], 1), "R@10": recall_at(res.ids, gt_ids[:, 0], 10),
               "kR@10": k_recall_at(res.ids, gt_ids, 10), "V": float(res.counters[:, 0].mean()) / G,
               "T": float(res.counters[:, 1].mean()) / G}
        sweep.append(row)
        if row["R@10"] >= 0.99:
            chosen = row
            break
    chosen = chosen or sweep[-1]
    tau = chosen["tau"]
    qcfg = ga.QueryConfig(k_out=10, tau=tau)

    dh = device_hierarchy(h)
    dv = dh.vectors
    dq, qs = dv.queries(Q)
    m = Q.shape[0]
    bb = block_layout(m, 10)[0]
    send = N.empty((bb,), torch.uint8)
    recv = N.empty((G * bb,), torch.uint8)
    ids_p, dists_p, cnt_p = block_pointers(send, 0, m, 10)
    out_ids = N.empty((m, 10), torch.int32)
    out_d = N.empty((m, 10), torch.float64)
    out_c = N.empty((m, 5), torch.int32)
    params = N.search_params(10, qcfg.prioq_size, qcfg.visited_size, tau, qcfg.max_iterations, _qflags(dh, False))
    gid = grp.gid_dev()
    stream = torch.cuda.current_stream()
    qev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]

    x = grp.p2p(m, 10) if args.exchange == "p2p" else None

    def step(i=None):
        if x is not None:  # fused: push search + signal, then wait + merge
            if i is not None:
                qev[2 * i].record(stream)
            x.search_push(h, Q, qcfg)
            if i is not None:
                qev[2 * i + 1].record(stream)
            x.merge_into(out_ids, out_d, out_c)
            return
        if i is not None:
            qev[2 * i].record(stream)
        N.call("ggnn_query_batch", N.ctypes.byref(dv.struct), N.ctypes.byref(dh.layers[0].struct),
               N.ptr(dh.top_rows), dh.ntop, N.ctypes.byref(qs), N.ctypes.byref(params), dh.d_nn1_max, ids_p, dists_p,
               cnt_p, None, 0, N.stream_ptr())
        if i is not None:
            qev[2 * i + 1].record(stream)
        N.call("ggnn_shard_globalize", ids_p, m * 10, N.ptr(gid), args.n, N.stream_ptr())
        grp.exchange(send, recv)
        N.call("ggnn_shard_merge", N.ptr(recv), G, m, 10, 10, N.ptr(out_ids), N.ptr(out_d), N.ptr(out_c),
               N.stream_ptr())

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        clocks.wait_first()
        # warm-up: a FIXED count on every rank (each step is a collective)
        for w in range(max(args.warmup, 16)):
            step()
            if w % 8 == 7:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(args.steps):
            step(i)
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    if x is not None:
        x.check()
    t_max = dist.max(evs[0].elapsed_time(evs[-1]) / 1e3)
    value = G * m * args.steps / t_max
    kern = float(np.mean([qev[2 * i].elapsed_time(qev[2 * i + 1]) for i in range(args.steps)])) / 1e3
    coff = block_layout(m, 10)[2]
    if x is not None:
        own = x.local_cnt.cpu().numpy()
    else:
        own = send[coff:coff + m * 20].view(torch.int32).view(m, 5).cpu().numpy()  # this rank's V, T counters
    e = 1 if dv.exact_integers else 4
    bpl = _bytes_per_launch(own, args.d, e, dh.layers[0].k, 10)
    peak, peak_src = _peak()
    achieved = bpl / kern / 1e9

    Q_pin = torch.empty(Q.shape, dtype=torch.float32, pin_memory=True)
    Q_pin.copy_(torch.from_numpy(np.ascontiguousarray(Q, dtype=np.float32)))
    Q_host = Q_pin.numpy()
    for _ in range(max(1, args.warmup)):
        grp.query_arrays(Q_host, qcfg, exchange=args.exchange)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = grp.query_arrays(Q_host, qcfg, exchange=args.exchange)
    torch.cuda.synchronize()
    e2e_t = dist.max(time.perf_counter() - t0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8" if dv.exact_integers else "f32",
        "data": "synthetic latent16 (SURVEY.md 8d G_B), seed 1234; shard r>0 from stream (1234, 0x5AD, r)",
        "config": {"workload": f"sharded latent16 {G}x{args.n}x{args.d} (one SIFT1M-shaped shard per GPU), "
                               f"{m} replicated queries, k=10, k_build=24",
                   "units": "shard-queries: each step searches all m queries on each of the N shards, then "
                            "all-gathers and merges the per-shard top-10 (value = N*m*steps/t)",
                   "tau": tau, "recall_merged": {k: chosen[k] for k in ("R@1", "R@10", "kR@10")},
                   "mean_visited_per_shard": chosen["V"], "mean_steps_per_shard": chosen["T"], "tau_sweep": sweep,
                   "build_seconds_max_over_ranks": build_s,
                   "parallelism": (f"sharded x{G}: NCCL all_gather_into_tensor of {bb} B/rank + ggnn_shard_merge"
                                   if x is None else f"sharded x{G}: fused exchange (query kernel stores each "
                                   f"finished row into every peer's receive block over CUDA IPC) + "
                                   f"ggnn_shard_merge_wait"),
                   "l2": "inputs larger than L2 (u8 shard 128 MB + adjacency 96 MB per GPU)"},
        "build_seconds": build_s,
        "e2e": {"value": G * m * args.steps / e2e_t, "unit": UNIT, "h2d_bytes_per_step": int(m * args.d * e),
                "d2h_bytes_per_step": int(out.ids.nbytes + out.dists.nbytes + out.counters.nbytes),
                "api": "ShardGroup.query_arrays(numpy queries) -> host arrays (every rank)"},
        "gpu_launches": 3 * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "algorithmic_bytes_per_launch": bpl, "kernel_ms": kern * 1e3,
                     "kernel": "query_kernel (rank 0)", "peak_source": peak_src},
        "clocks": clocks.summary(),
        "cpu_baseline": None,
    }
    if dist.rank == 0:
        js = json.dumps(line)
        print(js, flush=True)
        if args.out:
            Path(args.out).write_text(js + "\n")
    grp.close()
    dist.close()


def run_reference(args, dist, ga):
    """--impl reference: the reference's own CPU query path (graphann
    batch_query, compiled _core) on this box's host cores, process-parallel,
    on a bounded sample of the same workload per step."""
    if dist.rank != 0:
        dist.close()
        return
    base, Q = make_workload(args)
    ds = ga.Dataset(base)
    h, bstats = ga.build(ds, ga.BuildConfig(seed=7))  # index prep (untimed): the GPU-built graph
    gt_ids, _ = ga.search.exact_knn(ds, Q, 10)
    chosen, sweep = choose_tau(ga, h, Q, gt_ids, args.tau)
    tau = chosen["tau"]
    if not (ROOT / "oracle" / "_ref" / "graphann_ref").exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (compiled reference) not present"}))
        return
    import shutil

    root = export_graph(h, base, Q, tau)
    # one worker pool for the whole run; each step is a bounded sample
    per_step = max(2.0, min(args.cpu_seconds, 180.0 / max(1, args.steps + args.warmup)))
    vals = []
    info = None
    pool = None
    try:
        pool = RefPool(root, Q.shape[0])
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
        shutil.rmtree(root, ignore_errors=True)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic latent16 (SURVEY.md 8d G_B)",
        "config": {"workload": f"SIFT1M-shaped latent16 {args.n}x{args.d}, k=10, k_build=24", "tau": tau,
                   "recall_gpu_same_tau": {k: chosen[k] for k in ("R@1", "R@10", "kR@10")}},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "reference",
                         "sample": info["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
