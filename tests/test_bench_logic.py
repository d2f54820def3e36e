"""Host logic of bench.py (CPU): the tau / cache choice both arms share, the
recall query set, and the config object the driver compares between arms."""

import importlib.util
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["bench_mod"] = mod
    spec.loader.exec_module(mod)
    return mod


def _fake(recall_of):
    """query_fn whose R@10 is recall_of(tau, prioq): a fraction of queries
    return the true first neighbour in their top 10."""
    m = 1000
    gt = np.arange(m, dtype=np.int32)[:, None].repeat(10, axis=1)

    def fn(tau, pq, vs):
        hit = int(round(recall_of(tau, pq) * m))
        ids = np.full((m, 10), -1, dtype=np.int32)
        ids[:hit, 0] = np.arange(hit)
        cnt = np.zeros((m, 5), dtype=np.int32)
        cnt[:, 0] = int(1000 * tau * pq / 256)
        return ids, cnt
    return fn, gt


def test_choose_tau_refines_near_the_crossing():
    B = _bench()
    fn, gt = _fake(lambda tau, pq: min(1.0, 0.8 + 0.35 * tau))  # crosses 0.99 at tau ~0.543
    row, sweep, reached = B.choose_tau(fn, gt, None, 0.99)
    assert reached and row["tau"] == 0.55 and row["prioq_size"] == 256
    taus = [r["tau"] for r in sweep]
    assert taus[:8] == B.TAUS[:8] and 0.6 not in taus  # coarse sweep stopped at 0.55; no finer tau between 0.5 and 0.55 reached it
    fn, gt = _fake(lambda tau, pq: min(1.0, 0.9 + 0.2 * tau))  # crosses at 0.45 exactly
    row, sweep, reached = B.choose_tau(fn, gt, None, 0.99)
    assert reached and row["tau"] == 0.45


def test_choose_tau_escalates_the_cache_and_flags_failure():
    B = _bench()
    fn, gt = _fake(lambda tau, pq: 0.9 + (0.095 if pq >= 1024 else 0.0) * min(tau, 1.0))
    row, sweep, reached = B.choose_tau(fn, gt, None, 0.99)
    assert reached and row["prioq_size"] == 1024 and row["visited_size"] == 2048
    assert {r["prioq_size"] for r in sweep} == {256, 512, 1024}
    fn, gt = _fake(lambda tau, pq: 0.5)
    row, sweep, reached = B.choose_tau(fn, gt, None, 0.99)
    assert not reached and row["R@10"] == 0.5  # best row reported, flagged as not reached


def test_config_object_is_shared_and_caches_scale_iterations():
    B = _bench()

    class A:
        workload, n, d, queries, target = "sift1m", 1_000_000, 128, 10_000, 0.99

    c1 = B.config_of(A, 0.58)
    c2 = B.config_of(A, 0.58, 256, 512, 1000)
    assert c1 == c2 and c1["tau"] == 0.58 and c1["prioq_size"] == 256

    class GA:
        @staticmethod
        def QueryConfig(**kw):
            return kw

    assert B.qconfig({"tau": 0.6, "prioq_size": 256, "visited_size": 512}, GA)["max_iterations"] == 1000
    assert B.qconfig({"tau": 2.0, "prioq_size": 1024, "visited_size": 2048}, GA)["max_iterations"] == 4096


def test_recall_queries():
    B = _bench()

    class A:
        workload, gt_queries = "sift1m", None

    batches = [np.full((100, 4), b, dtype=np.float32) for b in range(3)]
    q = B.recall_queries(A, batches)
    assert q.shape == (300, 4) and (q[200:] == 2).all()
    A.workload = "gist1m"
    assert B.recall_queries(A, batches).shape == (100, 4)
