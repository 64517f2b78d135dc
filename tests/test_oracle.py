"""Pins the CPU oracle against the golden vectors produced by running the
reference package (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import taco_oracle as O
from paper_2603_24919_b200.workloads import make_config

RIGS = ["rig1", "rig2", "rig3"]


def _digest(a):
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=16).hexdigest()


@pytest.fixture(scope="module", params=RIGS)
def rig(request, golden):
    g = golden(request.param)
    cfg, n, nq, d, ns, s, kp, it, seed = (int(v) for v in g["params"])
    X, Q, _ = make_config(cfg, n=n, nq=nq, d=d)
    idx = O.build_index(X, ns, s, kp * kp, it, seed)
    return g, X, Q, idx


def test_rig_build_bit_exact(rig):
    g, X, Q, idx = rig
    np.testing.assert_array_equal(idx.mean, g["mean"])
    np.testing.assert_array_equal(np.stack(idx.blocks), g["blocks"])
    for j in range(idx.n_sub):
        np.testing.assert_array_equal(idx.cb1[j], g[f"cb1_{j}"])
        np.testing.assert_array_equal(idx.cb2[j], g[f"cb2_{j}"])
        np.testing.assert_array_equal(idx.labels[j][0], g[f"lab1_{j}"])
        np.testing.assert_array_equal(idx.labels[j][1], g[f"lab2_{j}"])
    assert O.serialize(idx) == g["blob"].tobytes()
    np.testing.assert_array_equal(O.transform(idx.mean, idx.blocks, X[:200]), g["T_head"])
    np.testing.assert_array_equal(O.transform(idx.mean, idx.blocks, Q), g["QT"])


def test_rig_queries_bit_exact(rig):
    g, X, Q, idx = rig
    for gi, (alpha, beta, k) in enumerate(g["grid"]):
        k = int(k)
        ids, dists, num, lvl = O.knn_batch(idx, X, Q, alpha, beta, k)
        np.testing.assert_array_equal(ids, g[f"ids_{gi}"])
        np.testing.assert_array_equal(dists, g[f"dists_{gi}"])
        np.testing.assert_array_equal(num, g[f"num_{gi}"])
        np.testing.assert_array_equal(lvl, g[f"lvl_{gi}"])
        for qi in range(Q.shape[0]):
            assert _digest(O.query_scores(idx, Q[qi], alpha)) == g[f"scores_digest_{gi}"][qi]
        pops = g[f"pops_{gi}"]
        for qi in range(4):
            tr = []
            O.query_scores(idx, Q[qi], alpha, trace=tr)
            mine = [(qi, j, a, b, key, got) for j, (pp, got) in enumerate(tr) for key, a, b in pp]
            ref = pops[pops[:, 0] == qi]
            np.testing.assert_array_equal(np.array(mine, np.float64), ref)


def test_deserialize_round_trip(golden):
    g = golden("rig1")
    blob = g["blob"].tobytes()
    assert O.serialize(O.deserialize(blob)) == blob


def test_kmeans_units(golden):
    u = golden("units")
    c = 0
    while f"km{c}_cfg" in u:
        n, m, k, it, sd = (int(v) for v in u[f"km{c}_cfg"])
        X = np.random.default_rng(1000 + c).normal(size=(n, m)).astype(np.float32)
        if c == 3:
            X[100:300] = X[0]
        r = O.kmeans(X, k, it, sd)
        np.testing.assert_array_equal(r.centroids, u[f"km{c}_cent"])
        np.testing.assert_array_equal(r.labels, u[f"km{c}_lab"])
        np.testing.assert_array_equal(np.array(r.history), u[f"km{c}_hist"])
        c += 1
    assert c == 6


def test_jacobi_units(golden):
    u = golden("units")
    for c in range(6):
        w, V, _ = O.jacobi(u[f"jac{c}_A"])
        np.testing.assert_array_equal(w, u[f"jac{c}_w"])
        np.testing.assert_array_equal(V, u[f"jac{c}_V"])


def test_traversal_units(golden):
    u = golden("units")
    for c in range(int(u["n_trav"][0])):
        d1, d2, sizes = u[f"tr{c}_d1"], u[f"tr{c}_d2"], u[f"tr{c}_sizes"]
        kp = d1.size
        pops, got = O.traverse(float(u[f"tr{c}_alpha"][0]), int(sizes.sum()), kp, d1,
                               np.argsort(d1, kind="stable"), d2, np.argsort(d2, kind="stable"),
                               lambda a, b: int(sizes[a, b]))
        np.testing.assert_array_equal(np.array([(a, b) for _, a, b in pops]).reshape(-1, 2),
                                      u[f"tr{c}_pops"].reshape(-1, 2))
        assert got == int(u[f"tr{c}_ret"][0])


def test_select_units(golden):
    u = golden("units")
    rng = np.random.default_rng(0)
    for row in u["select"]:
        ns, beta, lvl, num = int(row[0]), row[1], int(row[2]), int(row[3])
        h = row[4:5 + ns].astype(np.int64)
        sc = np.repeat(np.arange(ns + 1), h).astype(np.uint8)
        rng.shuffle(sc)
        ids, got_num, got_lvl, _ = O.select(sc, beta, ns)
        assert (got_lvl, got_num) == (lvl, num)
        assert ids.size == num


def test_select_hand_traces():
    # reference tests: test_engine.py:55-70 (hand traces of Alg. 5)
    for hist, beta, ns, want in [([70, 20, 7, 3], 0.1, 3, (2, 10)),
                                 ([60, 20, 12, 8], 0.1, 3, (3, 8))]:
        sc = np.repeat(np.arange(len(hist)), hist).astype(np.uint8)
        _, num, lvl, _ = O.select(sc, beta, ns)
        assert (lvl, num) == want
    sc = np.zeros(10, np.uint8)
    sc[:2] = 1
    _, num, lvl, _ = O.select(sc, 0.99, 2)          # test_engine.py:78-83
    assert (lvl, num) == (0, 10)


def test_seeds(golden):
    for r, p, want in golden("units")["seeds"]:
        assert O.derive_seed(int(r), int(p)) == int(want)


def test_sc_linear_scores_vs_reference():
    """oracle.sc_linear_scores pinned to the reference's engine.sc_linear_scores."""
    import sys
    sys.path.insert(0, "tests/golden")
    from make_golden import SC_ALPHAS, SC_CASES, sc_inputs
    g = np.load("tests/golden/sclinear.npz")
    for ci, (seed, n, n_sub, s, ints) in enumerate(SC_CASES):
        T, q = sc_inputs(seed, n, n_sub, s, ints)
        for qi in range(q.shape[0]):
            for ai, a in enumerate(SC_ALPHAS):
                np.testing.assert_array_equal(O.sc_linear_scores(T, q[qi], n_sub, s, a), g[f"sc_{ci}_{qi}_{ai}"])


def _gt_inputs(n, d, nq, ints):
    """The inputs of tests/golden/make_golden.py gt_fixture (rng(n + d) draws)."""
    rng = np.random.default_rng(n + d)
    if ints:
        return (rng.integers(0, 4, (n, d)).astype(np.float32), rng.integers(0, 4, (nq, d)).astype(np.float32))
    return rng.standard_normal((n, d)).astype(np.float32), rng.standard_normal((nq, d)).astype(np.float32)


def test_ground_truth_vs_reference(golden):
    """O.ground_truth against dataio.compute_ground_truth's own outputs
    (dataio.py:142-172; integer data with exact distance ties, d up to 960, k = 100)."""
    g = golden("groundtruth")
    for ci, (n, d, nq, k, ints) in enumerate(g["cases"].tolist()):
        X, Q = _gt_inputs(n, d, nq, bool(ints))
        oi, od = O.ground_truth(X, Q, k)
        np.testing.assert_array_equal(oi, g[f"ids_{ci}"])
        np.testing.assert_array_equal(od, g[f"dists_{ci}"])
