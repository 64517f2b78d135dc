"""GPU parity of the query path: the reference-built index
(golden v1 bytes) imported onto the B200 must reproduce the reference's
scores, pop traces, candidate counts, thresholds, top-k ids and distances
bit-for-bit."""

import hashlib

import numpy as np
import pytest

import paper_2603_24919_b200 as T
from oracle import taco_oracle as O
from paper_2603_24919_b200.workloads import make_config

pytestmark = pytest.mark.gpu
RIGS = ["rig1", "rig2", "rig3"]


def _digest(a):
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=16).hexdigest()


@pytest.fixture(scope="module", params=RIGS)
def rig(request, golden):
    g = golden(request.param)
    cfg, n, nq, d, ns, s, kp, it, seed = (int(v) for v in g["params"])
    X, Q, _ = make_config(cfg, n=n, nq=nq, d=d)
    idx = T.deserialize_index(g["blob"].tobytes())
    return g, X, Q, idx


@pytest.mark.parametrize("walk", ["default", "smem", "heap", "pl"])
def test_batch_matches_reference(rig, walk, monkeypatch):
    if walk != "default":
        monkeypatch.setenv("TACO_TRAVERSE", walk)
    g, X, Q, idx = rig
    for gi, (alpha, beta, k) in enumerate(g["grid"]):
        qp = T.QueryParams(alpha=float(alpha), beta=float(beta), k=int(k))
        ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, qp)
        np.testing.assert_array_equal(num, g[f"num_{gi}"])
        np.testing.assert_array_equal(lvl, g[f"lvl_{gi}"])
        np.testing.assert_array_equal(ids, g[f"ids_{gi}"])
        np.testing.assert_array_equal(dists, g[f"dists_{gi}"])


@pytest.mark.parametrize("split", ["64", "300"])
def test_split_topk_matches_reference(rig, split, monkeypatch):
    """The two-step top-k of long partial lists (k_topk: ranges' best-k, then a merge
    launch), forced onto the rigs' short lists; large k keeps every candidate."""
    monkeypatch.setenv("TACO_TOPK_SPLIT", split)
    g, X, Q, idx = rig
    for gi, (alpha, beta, k) in enumerate(g["grid"]):
        qp = T.QueryParams(alpha=float(alpha), beta=float(beta), k=int(k))
        ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, qp)
        np.testing.assert_array_equal(ids, g[f"ids_{gi}"])
        np.testing.assert_array_equal(dists, g[f"dists_{gi}"])
    # k > 32: no per-tile filtering, every candidate reaches the top-k; against the oracle
    oidx = O.deserialize(g["blob"].tobytes())
    alpha, beta, _ = (float(v) for v in g["grid"][0])
    oi, od, on, ol = O.knn_batch(oidx, X, Q, alpha, max(beta, 0.05), 50, threads=4)
    ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, T.QueryParams(alpha, max(beta, 0.05), 50))
    np.testing.assert_array_equal(ids, oi)
    np.testing.assert_array_equal(dists, od)


def test_single_query_api(rig):
    g, X, Q, idx = rig
    alpha, beta, k = g["grid"][0]
    qp = T.QueryParams(alpha=float(alpha), beta=float(beta), k=int(k))
    for qi in range(min(4, Q.shape[0])):
        res = T.knn_query(idx, X, Q[qi], qp)
        want = g["ids_0"][qi]
        want = want[want >= 0]
        np.testing.assert_array_equal(res.ids, want)
        assert res.ids.dtype == np.int32 and res.dists.dtype == np.float32


def test_scores_and_traces(rig):
    g, X, Q, idx = rig
    for gi, (alpha, _, _) in enumerate(g["grid"]):
        for qi in range(Q.shape[0]):
            sc = T.count_collisions(idx, Q[qi], float(alpha))
            assert _digest(sc) == g[f"scores_digest_{gi}"][qi]
        pops = g[f"pops_{gi}"]
        s = idx.params.subspace_dim
        for qi in range(4):
            qt = T.transform_points(idx.transform, Q[qi][None, :])[0]
            for j, sub in enumerate(idx.subspaces):
                d1, i1, d2, i2 = T.sorted_centroid_distances(sub, qt[j * s:(j + 1) * s])
                act = T.scalable_dynamic_activation(float(alpha), idx.n, idx.params.clusters,
                                                    d1, i1, d2, i2, sub)
                ref = pops[(pops[:, 0] == qi) & (pops[:, 1] == j)]
                mine = np.array([(qi, j, a, b, key, act.retrieved_num) for key, a, b in act.pop_trace])
                np.testing.assert_array_equal(mine, ref)


def test_select_and_rerank_taps(rig):
    g, X, Q, idx = rig
    alpha, beta, k = g["grid"][0]
    for qi in range(3):
        sc = T.count_collisions(idx, Q[qi], float(alpha))
        cand = T.select_candidates(sc, float(beta), idx.params.n_subspaces, idx.n)
        ids, num, lvl, _ = O.select(sc, float(beta), idx.params.n_subspaces, idx.n)
        np.testing.assert_array_equal(cand.ids, ids)
        assert (cand.candidate_num, cand.last_collision) == (num, lvl)
        res = T.rerank(X, Q[qi], cand, int(k))
        rid, rd, _ = O.rerank(X, Q[qi], ids, int(k))
        np.testing.assert_array_equal(res.ids, rid)
        np.testing.assert_array_equal(res.dists, rd)


def test_transform_points_matches_reference(rig):
    g, X, Q, idx = rig
    np.testing.assert_array_equal(T.transform_points(idx.transform, X[:200]), g["T_head"])
    qt = T.transform_points(idx.transform, Q)
    # reference transforms one query at a time through dgemv (different fp64
    # summation order); after the f32 cast at most isolated 1-ulp flips remain
    diff = qt != g["QT"]
    assert diff.mean() < 1e-3
    np.testing.assert_allclose(qt, g["QT"], rtol=2e-7, atol=1e-6)


def test_select_edge_cases():
    rng = np.random.default_rng(0)
    for hist, beta, ns, want in [([70, 20, 7, 3], 0.1, 3, (2, 10)), ([60, 20, 12, 8], 0.1, 3, (3, 8))]:
        sc = np.repeat(np.arange(len(hist)), hist).astype(np.uint8)
        rng.shuffle(sc)
        c = T.select_candidates(sc, beta, ns)
        assert (c.last_collision, c.candidate_num) == want
        assert np.all(sc[c.ids] >= c.last_collision)
    sc = np.zeros(10, np.uint8)
    sc[:2] = 1
    c = T.select_candidates(sc, 0.99, 2)              # clamp at 0 -> everything
    assert (c.last_collision, c.candidate_num) == (0, 10)
    np.testing.assert_array_equal(c.ids, np.arange(10))
    big = rng.integers(0, 9, 300_000).astype(np.uint8)  # several 64 Ki chunks
    for beta in (0.001, 0.01, 0.2, 0.9):
        c = T.select_candidates(big, beta, 8)
        ids, num, lvl, _ = O.select(big, beta, 8)
        np.testing.assert_array_equal(c.ids, ids)
        assert (c.candidate_num, c.last_collision) == (num, lvl)


def test_rerank_edge_cases():
    rng = np.random.default_rng(1)
    X = rng.normal(size=(500, 7)).astype(np.float32)      # d not a multiple of 4
    X[10] = X[20]                                          # exact distance tie
    q = X[10].copy()
    ids = np.array([300, 20, 10, 5, 499], np.int64)       # unsorted input
    res = T.rerank(X, q, ids, 3)
    rid, rd, _ = O.rerank(X, q, ids, 3)
    np.testing.assert_array_equal(res.ids, rid)
    np.testing.assert_array_equal(res.dists, rd)
    assert list(res.ids[:2]) == [10, 20] and res.dists[0] == 0.0
    res = T.rerank(X, q, np.array([7], np.int64), 10)      # |C| < k
    assert res.ids.size == 1
    res = T.rerank(X, q, np.empty(0, np.int64), 10)
    assert res.ids.size == 0 and res.ids.dtype == np.int32


@pytest.mark.parametrize("walk", ["smem", "heap", "pl"])
def test_traversal_units(golden, walk, monkeypatch):
    """60 traversal instances with integer ties (reference pop traces), through
    the shared-memory fixed-depth heap (large batches) and the thread-local
    heap (small batches)."""
    monkeypatch.setenv("TACO_TRAVERSE", walk)
    u = golden("units")
    for c in range(int(u["n_trav"][0])):
        d1, d2, sizes = u[f"tr{c}_d1"], u[f"tr{c}_d2"], u[f"tr{c}_sizes"]
        kp = d1.size
        cells = {}
        base = 0
        for a in range(kp):
            for b in range(kp):
                if sizes[a, b]:
                    cells[(a, b)] = np.arange(base, base + sizes[a, b], dtype=np.uint32)
                    base += sizes[a, b]
        cb = T.KMeansModel(np.zeros((kp, 1), np.float32), None, 0.0)
        imi = T.InvertedMultiIndex(cb, cb, cells, kp, 1)
        act = T.scalable_dynamic_activation(float(u[f"tr{c}_alpha"][0]), int(sizes.sum()), kp * kp,
                                            d1, np.argsort(d1, kind="stable"), d2,
                                            np.argsort(d2, kind="stable"), imi)
        np.testing.assert_array_equal(np.array([(a, b) for _, a, b in act.pop_trace]).reshape(-1, 2),
                                      u[f"tr{c}_pops"].reshape(-1, 2))
        assert act.retrieved_num == int(u[f"tr{c}_ret"][0])


@pytest.mark.parametrize("fmt", [2, 1, 0])
def test_row_formats_bit_identical(fmt):
    """Lossless narrow row storage (u8 / f16 / f32, taco_b200.h) must not change
    a single bit of the answers: checked against the oracle on data that is
    exactly representable in each format, with non-representable queries."""
    from paper_2603_24919_b200 import _native as nat
    from paper_2603_24919_b200.engine import _device_of

    rng = np.random.default_rng(40 + fmt)
    n, d, nq = 4000, 32, 40
    if fmt == 2:
        X = rng.integers(0, 256, (n, d)).astype(np.float32)
    elif fmt == 1:
        X = (rng.integers(-1024, 1024, (n, d)) / 64.0).astype(np.float32)
    else:
        X = rng.standard_normal((n, d)).astype(np.float32) * 30
    Q = (X[rng.integers(0, n, nq)] + rng.standard_normal((nq, d)) * 3).astype(np.float32)
    idx = T.build_index(X, T.IndexParams(4, 8, 16, 10, 1 + fmt))
    assert nat.lib().taco_index_row_format(_device_of(idx).h) == fmt
    oidx = O.deserialize(T.serialize_index(idx))
    for a, b, k in [(0.05, 0.01, 10), (0.3, 0.2, 25)]:
        ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, T.QueryParams(a, b, k))
        oi, od, on, ol = O.knn_batch(oidx, X, Q, a, b, k)
        np.testing.assert_array_equal(num, on)
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(dists, od)


def test_sc_linear_scores_vs_reference():
    """SC-Linear exact collision counting on the GPU
    against the reference's engine.sc_linear_scores (tests/golden/sclinear.npz)."""
    import sys
    sys.path.insert(0, "tests/golden")
    from make_golden import SC_ALPHAS, SC_CASES, sc_inputs
    g = np.load("tests/golden/sclinear.npz")
    for ci, (seed, n, n_sub, s, ints) in enumerate(SC_CASES):
        T_, q = sc_inputs(seed, n, n_sub, s, ints)
        for qi in range(q.shape[0]):
            for ai, a in enumerate(SC_ALPHAS):
                np.testing.assert_array_equal(T.sc_linear_scores(T_, q[qi], n_sub, s, a), g[f"sc_{ci}_{qi}_{ai}"])


def test_sc_linear_query_vs_reference(golden):
    g = golden("rig1")
    cfg, n, nq, d, ns, s, kp, it, seed = (int(v) for v in g["params"])
    X, Q, _ = make_config(cfg, n=n, nq=nq, d=d)
    idx = T.deserialize_index(g["blob"].tobytes())
    with pytest.raises(T.StateError):
        T.sc_linear_query(idx, X, Q[0], T.QueryParams(0.05, 0.01, 10))
    T.attach_transformed(idx, X)
    gs = np.load("tests/golden/sclinear.npz")
    for qi in range(8):
        for gi, (a, b, k) in enumerate([(0.05, 0.01, 10), (0.2, 0.05, 15)]):
            r = T.sc_linear_query(idx, X, Q[qi], T.QueryParams(a, b, k))
            np.testing.assert_array_equal(r.ids, gs[f"q_{qi}_{gi}_ids"])
            np.testing.assert_array_equal(r.dists, gs[f"q_{qi}_{gi}_dists"])


def test_sc_linear_resident_matches_host():
    """The resident-matrix path (built index, keep_transformed) equals the
    host-matrix path."""
    X, Q, _ = make_config(1, n=3000, nq=4, d=32)
    idx = T.build_index(X, T.IndexParams(4, 8, 16, 5, 1), keep_transformed=True)
    assert getattr(idx.device, "transformed_key", None) is not None
    for qi in range(4):
        r1 = T.sc_linear_query(idx, X, Q[qi], T.QueryParams(0.1, 0.02, 10))
        qt = T.transform_points(idx.transform, Q[qi][None, :])[0]
        sc = T.sc_linear_scores(idx.transformed, qt, 4, 8, 0.1)
        cand = T.select_candidates(sc, 0.02, 4, 3000)
        r2 = T.rerank(X, Q[qi], cand, 10)
        np.testing.assert_array_equal(r1.ids, r2.ids)
        np.testing.assert_array_equal(r1.dists, r2.dists)


@pytest.mark.parametrize("int_queries", [True, False])
def test_integer_rerank_path(int_queries, monkeypatch):
    """u8 rows + u8-exact queries take the DP4A integer re-rank (exact by
    construction); it must agree bit-for-bit with the oracle, and so must the
    fp64 path on the same rows with non-integer queries."""
    rng = np.random.default_rng(77)
    n, d, nq = 5000, 64, 64
    X = rng.integers(0, 256, (n, d)).astype(np.float32)
    Q = X[rng.integers(0, n, nq)] + rng.integers(-6, 7, (nq, d))
    Q = np.clip(Q, 0, 255).astype(np.float32)
    if not int_queries:
        Q = (Q + rng.uniform(-0.5, 0.5, Q.shape)).astype(np.float32)
    Q[:3] = X[:3]   # exact duplicates: d2 == 0 ties broken by id
    idx = T.build_index(X, T.IndexParams(4, 16, 64, 5, 3))
    oidx = O.deserialize(T.serialize_index(idx))
    for a, b, k in [(0.05, 0.01, 10), (0.2, 0.05, 40)]:
        ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, T.QueryParams(a, b, k))
        oi, od, on, ol = O.knn_batch(oidx, X, Q, a, b, k)
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(dists, od)


def test_pipelined_batch_matches_oracle():
    """A batch >= 2 x 2048 queries runs as two tiles on two streams; every
    query's answer must still be the oracle's (and the same as unbatched)."""
    X, Q, _ = make_config(1, n=20000, nq=4500, d=32)
    idx = T.build_index(X, T.IndexParams(8, 4, 64, 5, 4))
    qp = T.QueryParams(0.05, 0.01, 10)
    ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, qp)
    oidx = O.deserialize(T.serialize_index(idx))
    sel = np.r_[0:40, 2240:2280, 4460:4500]   # both tiles and their seams
    oi, od, on, ol = O.knn_batch(oidx, X, Q[sel], qp.alpha, qp.beta, qp.k)
    np.testing.assert_array_equal(ids[sel], oi)
    np.testing.assert_array_equal(dists[sel], od)
    np.testing.assert_array_equal(num[sel], on)
    np.testing.assert_array_equal(lvl[sel], ol)
    i2, d2, n2, l2 = T.knn_query_batch(idx, X, Q[2250:2260], qp)   # a small unpipelined batch
    np.testing.assert_array_equal(i2, ids[2250:2260])


def test_assign_matches_reference_formula():
    """clustering.assign (clustering.py:118-127): nearest centroid by the fp64
    einsum distance, ties to the lowest index."""
    rng = np.random.default_rng(5)
    C = rng.normal(size=(40, 7)).astype(np.float32)
    C[17] = C[3]                                   # duplicate centroid: tie -> 3
    model = T.KMeansModel(C, None, 0.0)
    pts = np.vstack([rng.normal(size=(50, 7)), C[3:4], C[17:18]]).astype(np.float32)
    for p in pts:
        e = C.astype(np.float64) - p.astype(np.float64)
        want = int(np.argmin(np.einsum("ij,ij->i", e, e)))
        assert T.assign(model, p) == want
    with pytest.raises(T.DimensionMismatchError):
        T.assign(model, np.zeros(6, np.float32))


def test_knn_query_fills_scratch_and_pads_large_k(rig):
    """knn_query(scratch=...) leaves the query's collision counts in the
    buffer like engine.py:285; k beyond the device top-k limit is served when
    n fits under it (padding -1 / +inf like cli.py:155-164)."""
    g, X, Q, idx = rig
    alpha, beta, k = g["grid"][0]
    qp = T.QueryParams(float(alpha), float(beta), int(k))
    scratch = np.full(idx.n, 7, np.uint8)
    res = T.knn_query(idx, X, Q[0], qp, scratch=scratch)
    np.testing.assert_array_equal(scratch, T.count_collisions(idx, Q[0], float(alpha)))
    assert _digest(scratch) == g["scores_digest_0"][0]
    want = g["ids_0"][0]
    np.testing.assert_array_equal(res.ids, want[want >= 0])
    if idx.n <= T.engine.TOPK_MAX:
        return
    with pytest.raises(T.ParameterError):
        T.knn_query_batch(idx, X, Q[:2], T.QueryParams(float(alpha), float(beta), T.engine.TOPK_MAX + 1))


def test_large_k_on_small_index():
    X, Q, _ = make_config(1, n=1500, nq=6, d=32)
    idx = T.build_index(X, T.IndexParams(4, 8, 16, 5, 1))
    qp = T.QueryParams(0.5, 0.9, 3000)             # k > TK_MAX and k > n
    ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, qp)
    oidx = O.deserialize(T.serialize_index(idx))
    oi, od, on, ol = O.knn_batch(oidx, X, Q, qp.alpha, qp.beta, qp.k)
    np.testing.assert_array_equal(ids, oi)
    np.testing.assert_array_equal(dists, od)
    np.testing.assert_array_equal(num, on)
