"""CLI and measurement module on the batched GPU path,
following the reference's cli.py / bench.py contracts."""

import csv
import json

import numpy as np
import pytest

import paper_2603_24919_b200 as T
from paper_2603_24919_b200 import cli, metrics


def test_recall_and_mre_definitions():
    # bench.py:47-91 semantics: set overlap over k; ascending-rank relative error,
    # zero true distances counted or skipped, missing ranks skipped
    assert metrics.recall(np.array([3, 1, -1]), np.array([1, 2, 3]), 3) == pytest.approx(2 / 3)
    v, sk = metrics.mre_with_skips([1.0, 2.2, np.inf], [1.0, 2.0, 3.0], 3)
    assert sk == 1 and v == pytest.approx(0.05)
    v, sk = metrics.mre_with_skips([0.0, 1.0], [0.0, 0.5], 2)
    assert sk == 0 and v == pytest.approx(0.5)
    v, sk = metrics.mre_with_skips([0.5], [0.0], 1)
    assert sk == 1 and v == 0.0
    with pytest.raises(T.ParameterError):
        metrics.recall([1], [1], 2)


def test_cli_usage_and_io_errors(tmp_path, capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["query"])
    assert e.value.code == 2
    rc = cli.main(["query", "--index", str(tmp_path / "none.taco"), "--dataset", "x", "--queries", "y",
                   "--ids-out", "a", "--dists-out", "b"])
    assert rc == 3
    bad = tmp_path / "bad.fvecs"
    bad.write_bytes(b"\x05\x00\x00\x00\x01")
    rc = cli.main(["groundtruth", "--dataset", str(bad), "--queries", str(bad), "--ids-out", "a",
                   "--dists-out", "b"])
    assert rc == 3
    assert "format" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_round_trip(tmp_path, capsys):
    f = lambda name: str(tmp_path / name)  # noqa: E731
    assert cli.main(["workload", "--config", "1", "--n", "4000", "--nq", "30", "--out", f("b.fvecs"),
                     "--queries-out", f("q.fvecs")]) == 0
    assert cli.main(["groundtruth", "--dataset", f("b.fvecs"), "--queries", f("q.fvecs"), "--k", "20",
                     "--ids-out", f("gt.ivecs"), "--dists-out", f("gt.fvecs")]) == 0
    assert cli.main(["build", "--dataset", f("b.fvecs"), "--index-out", f("x.taco"), "--subspaces", "4",
                     "--subspace-dim", "8", "--clusters", "64", "--kmeans-iters", "5"]) == 0
    assert cli.main(["query", "--index", f("x.taco"), "--dataset", f("b.fvecs"), "--queries", f("q.fvecs"),
                     "--alpha", "0.1", "--beta", "0.05", "--k", "10", "--ids-out", f("ids.ivecs"),
                     "--dists-out", f("d.fvecs"), "--candidates-out", f("c.csv")]) == 0
    ids = T.read_vectors(f("ids.ivecs"), "int32")
    X, Q = T.read_vectors(f("b.fvecs")), T.read_vectors(f("q.fvecs"))
    idx = T.load_index(f("x.taco"))
    want, _, num, _ = T.knn_query_batch(idx, X, Q, T.QueryParams(0.1, 0.05, 10))
    np.testing.assert_array_equal(ids, want)
    rows = list(csv.reader(open(f("c.csv"))))
    assert rows[0] == ["query", "candidates", "last_collision"] and int(rows[1][1]) == num[0]
    capsys.readouterr()
    assert cli.main(["bench", "--index", f("x.taco"), "--dataset", f("b.fvecs"), "--queries", f("q.fvecs"),
                     "--truth-ids", f("gt.ivecs"), "--truth-dists", f("gt.fvecs"), "--alphas", "0.05,0.2",
                     "--betas", "0.01", "--k", "10", "--repeats", "1", "--out", f("m.csv"),
                     "--records-out", f("r.csv")]) == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["rows"] == 2 and 0.0 <= out["best_recall"] <= 1.0
    m = list(csv.reader(open(f("m.csv"))))
    assert m[0][:4] == ["alpha", "beta", "k", "recall"] and len(m) == 3
    assert len(list(csv.reader(open(f("r.csv"))))) == 1 + 2 * 30
