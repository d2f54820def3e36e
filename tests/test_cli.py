"""Batched CLI (paper_1912_01059_b200.cli): the reference CLI's sub-commands,
JSON-lines events and exit codes (reference tests/test_cli.py)."""

from __future__ import annotations

import json

import numpy as np
import pytest

import paper_1912_01059_b200 as ga
from paper_1912_01059_b200 import cli


def _events(capsys):
    out = capsys.readouterr().out
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def test_usage_errors_exit_2(capsys, tmp_path):
    assert cli.main([]) == 2
    assert cli.main(["build", "--data", str(tmp_path / "missing.fvecs"), "--out", str(tmp_path / "x")]) == 2
    err = json.loads(capsys.readouterr().err.strip().splitlines()[-1])
    assert err["exit_code"] == 2 and "not found" in err["error"]


def test_config_errors_exit_2(capsys, tmp_path):
    X = np.random.default_rng(0).random((64, 4)).astype(np.float32)
    ga.write_vectors(tmp_path / "d.fvecs", X)
    rc = cli.main(["build", "--data", str(tmp_path / "d.fvecs"), "--out", str(tmp_path / "i"), "--knn", "3"])
    assert rc == 2
    assert "k_nn" in json.loads(capsys.readouterr().err.strip().splitlines()[-1])["error"]


def test_sweep_spec():
    assert cli._sweep("0.3:0.8:0.1") == [0.3, 0.4, 0.5, 0.6, 0.7, 0.8]
    with pytest.raises(ValueError):
        cli._sweep("0.5:0.1:0.1")


@pytest.mark.gpu
def test_build_query_gt_bench_round_trip(capsys, tmp_path):
    from paper_1912_01059_b200.synthetic import make_latent16

    base, Q = make_latent16(n=3000, d=32, m=100, seed=5)
    ga.write_vectors(tmp_path / "b.fvecs", base)
    ga.write_vectors(tmp_path / "q.fvecs", Q)
    d, q = str(tmp_path / "b.fvecs"), str(tmp_path / "q.fvecs")
    assert cli.main(["build", "--data", d, "--out", str(tmp_path / "i.ggnn"), "--seed", "7"]) == 0
    ev = _events(capsys)
    assert [e["event"] for e in ev] == ["config", "build-stats"] and ev[1]["layers"][0] == 3000
    assert cli.main(["query", "--data", d, "--queries", q, "--index", str(tmp_path / "i.ggnn"), "--out",
                     str(tmp_path / "r.ivecs"), "--tau", "0.6"]) == 0
    ev = _events(capsys)
    assert ev[-1]["event"] == "query-stats" and ev[0]["mode"] == "batched"
    ids = ga.load_ids(tmp_path / "r.ivecs")
    h = ga.load_index(tmp_path / "i.ggnn").attach(ga.Dataset(base))
    np.testing.assert_array_equal(ids, ga.query_arrays(h, Q, ga.QueryConfig(k_out=10, tau=0.6)).ids)
    assert cli.main(["gt", "--data", d, "--queries", q, "--out", str(tmp_path / "gt.ivecs"), "--kout", "10"]) == 0
    gt = ga.load_ids(tmp_path / "gt.ivecs")
    np.testing.assert_array_equal(gt, ga.brute_force_oracle(ga.Dataset(base), Q, 10).ids)
    assert cli.main(["build", "--data", d, "--out", str(tmp_path / "sh"), "--shard-size", "1500"]) == 0
    assert cli.main(["query", "--data", d, "--queries", q, "--index", str(tmp_path / "sh"), "--out",
                     str(tmp_path / "rs.ivecs")]) == 0
    assert ga.load_ids(tmp_path / "rs.ivecs").shape == (100, 10)
    capsys.readouterr()
    assert cli.main(["bench", "--data", d, "--queries", q, "--tau-sweep", "0.3:0.6:0.3", "--refine-sweep", "0,1",
                     "--out", str(tmp_path / "rep"), "--repeats", "2"]) == 0
    ev = _events(capsys)
    rows = [e for e in ev if e["event"] == "bench-row"]
    assert len(rows) == 4 and all(0 <= r["recall_at_1"] <= 1 for r in rows)
    assert rows[0]["consensus_at_10"] is not None
    assert (tmp_path / "rep.json").exists() and (tmp_path / "rep.csv").exists()
