"""GPU parity of the build path."""

import numpy as np
import pytest

import paper_2603_24919_b200 as T
from oracle import taco_oracle as O
from paper_2603_24919_b200.workloads import make_config

pytestmark = pytest.mark.gpu


def test_kmeans_units_bit_exact(golden):
    u = golden("units")
    for c in range(6):
        n, m, k, it, sd = (int(v) for v in u[f"km{c}_cfg"])
        X = np.random.default_rng(1000 + c).normal(size=(n, m)).astype(np.float32)
        if c == 3:
            X[100:300] = X[0]
        r = T.kmeans(X, k, it, sd)
        np.testing.assert_array_equal(r.assignments, u[f"km{c}_lab"])
        np.testing.assert_array_equal(r.centroids, u[f"km{c}_cent"])
        assert r.n_iter == len(u[f"km{c}_hist"])
        np.testing.assert_allclose(r.inertia_history, u[f"km{c}_hist"], rtol=1e-12, atol=1e-9)


def test_kmeans_reference_unit_cases():
    # clustering tests of the reference (test_clustering.py:12-86)
    data = np.array([[0.0], [1.0], [10.0], [11.0]], dtype=np.float32)
    m = T.kmeans(data, 2, max_iter=10, seed=3)
    assert sorted(m.centroids[:, 0].tolist()) == pytest.approx([0.5, 10.5])
    assert m.inertia == pytest.approx(1.0)
    rng = np.random.default_rng(0)
    data = rng.normal(size=(30, 4)).astype(np.float32)
    m = T.kmeans(data, 1, max_iter=5, seed=1)
    np.testing.assert_allclose(m.centroids[0], data.astype(np.float64).mean(axis=0), rtol=1e-5)
    assert np.all(m.assignments == 0)
    with pytest.raises(T.InsufficientDataError):
        T.kmeans(np.ones((2, 3), dtype=np.float32), 4)
    dup = np.zeros((20, 2), np.float32)      # all points identical -> D^2 total 0
    dup[:3] = [[1, 1], [2, 2], [3, 3]]
    r = T.kmeans(dup, 6, 5, 9)
    o = O.kmeans(dup, 6, 5, 9)
    np.testing.assert_array_equal(r.assignments, o.labels)
    np.testing.assert_array_equal(r.centroids, o.centroids)


@pytest.mark.parametrize("shape,k,seed", [((5000, 8), 64, 1), ((3000, 30), 50, 2),
                                          ((70000, 6), 128, 3), ((200, 2), 256 - 60, 4)])
def test_kmeans_vs_oracle(shape, k, seed):
    X = np.random.default_rng(seed).normal(size=shape).astype(np.float32)
    r = T.kmeans(X, k, 20, seed)
    o = O.kmeans(X, k, 20, seed)
    np.testing.assert_array_equal(r.assignments, o.labels)
    np.testing.assert_array_equal(r.centroids, o.centroids)


def test_build_subspace_index_vs_oracle():
    X = np.random.default_rng(7).normal(size=(4000, 7)).astype(np.float32)
    imi = T.build_subspace_index(X, 49, 10, 11)
    split = 4
    c1 = O.kmeans(X[:, :split], 7, 10, O.derive_seed(11, 0))
    c2 = O.kmeans(X[:, split:], 7, 10, O.derive_seed(11, 1))
    cells = O.cells_from_labels(c1.labels, c2.labels)
    assert imi.split == 4 and imi.codebook2.dim == 3
    assert sorted(imi.cells) == sorted(cells)
    for key in cells:
        np.testing.assert_array_equal(imi.cells[key], cells[key])


@pytest.fixture(scope="module", params=["rig1", "rig2", "rig3"])
def built(request, golden):
    g = golden(request.param)
    cfg, n, nq, d, ns, s, kp, it, seed = (int(v) for v in g["params"])
    X, Q, _ = make_config(cfg, n=n, nq=nq, d=d)
    idx = T.build_index(X, T.IndexParams(ns, s, kp * kp, it, seed))
    return g, X, Q, idx


def test_build_transform(built):
    g, X, Q, idx = built
    np.testing.assert_array_equal(idx.transform.mean, g["mean"])   # sequential fp64 mean
    blocks = np.stack(idx.transform.blocks)
    # covariance accumulates in a different fp64 order than OpenBLAS syrk:
    # blocks agree to a few f32 ulps
    np.testing.assert_allclose(blocks, g["blocks"], rtol=0, atol=2e-6)


def test_build_end_to_end(built):
    g, X, Q, idx = built
    blob = T.serialize_index(idx)
    same_model = np.array_equal(np.stack(idx.transform.blocks), g["blocks"])
    if same_model:
        assert blob == g["blob"].tobytes()
    # oracle reads the GPU-built index and must answer identically
    oidx = O.deserialize(blob)
    for gi, (alpha, beta, k) in enumerate(g["grid"]):
        qp = T.QueryParams(float(alpha), float(beta), int(k))
        ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, qp)
        oi, od, on, ol = O.knn_batch(oidx, X, Q, float(alpha), float(beta), int(k))
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(dists, od)
        np.testing.assert_array_equal(num, on)
        np.testing.assert_array_equal(lvl, ol)


def test_build_stagewise_kmeans_cells(built):
    """Given the GPU transform, every label / centroid / cell equals the
    oracle's k-means over the same T (P2, P3)."""
    g, X, Q, idx = built
    p = idx.params
    model = (idx.transform.mean, list(idx.transform.blocks))
    Tm = T.transform_points(idx.transform, X)
    o = O.build_index(X, p.n_subspaces, p.subspace_dim, p.clusters, p.kmeans_iters, p.seed,
                      T=Tm, model=model)
    for j, sub in enumerate(idx.subspaces):
        np.testing.assert_array_equal(sub.codebook1.assignments, o.labels[j][0])
        np.testing.assert_array_equal(sub.codebook2.assignments, o.labels[j][1])
        np.testing.assert_array_equal(sub.codebook1.centroids, o.cb1[j])
        np.testing.assert_array_equal(sub.codebook2.centroids, o.cb2[j])
        assert sorted(sub.cells) == sorted(o.cells[j])
    assert T.serialize_index(idx) == O.serialize(o)


def test_build_validation():
    X = np.random.default_rng(6).normal(size=(50, 6)).astype(np.float32)
    with pytest.raises(T.ParameterError) as err:
        T.build_index(X, T.IndexParams(n_subspaces=3, subspace_dim=4, clusters=4))
    assert "12" in str(err.value) and "6" in str(err.value)
    bad = X.copy()
    bad[7, 2] = np.nan
    with pytest.raises(T.NumericError):
        T.build_index(bad, T.IndexParams(n_subspaces=1, subspace_dim=4, clusters=4))
    one = T.build_index(X, T.IndexParams(n_subspaces=1, subspace_dim=4, clusters=1, kmeans_iters=3))
    (cells,) = [s.cells for s in one.subspaces]
    assert list(cells) == [(0, 0)] and cells[(0, 0)].size == 50


def test_kmeans_exact_replay_path():
    """Force every k-means++ draw through the exact numpy replay (taken in
    production only when the certified fast path is ambiguous)."""
    from paper_2603_24919_b200 import _native as nat
    nat.call("taco_debug_force_replay", 1)
    try:
        for shape, k, seed, iters in [((5000, 8), 64, 1, 10), ((3001, 5), 17, 4, 10), ((1000, 3), 40, 13, 10),
                                      ((200_000, 6), 16, 7, 10), ((1_500_000, 4), 8, 5, 2)]:
            X = np.random.default_rng(seed).normal(size=shape).astype(np.float32)
            if shape[0] > 100_000:
                X[::3] *= 1e-3   # wide value range: many binade changes inside the cumsum
            if shape[0] > 1_000_000:
                X[:40_000] *= 1e-6   # a long low head: the tile walk starts many binades down
            r = T.kmeans(X, k, iters, seed)
            o = O.kmeans(X, k, iters, seed)
            np.testing.assert_array_equal(r.assignments, o.labels)
            np.testing.assert_array_equal(r.centroids, o.centroids)
            # the multi-CTA tile walk (mode 1) == the one-CTA sequential chain
            # (mode 2) == the one-CTA binade scan (mode 3)
            for mode in (2, 3):
                nat.call("taco_debug_force_replay", mode)
                r2 = T.kmeans(X, k, iters, seed)
                nat.call("taco_debug_force_replay", 1)
                np.testing.assert_array_equal(r.assignments, r2.assignments)
                np.testing.assert_array_equal(r.centroids, r2.centroids)
    finally:
        nat.call("taco_debug_force_replay", 0)


def _jac(A, device, max_sweeps=100):
    from paper_2603_24919_b200 import _native as nat
    A = np.ascontiguousarray(A, dtype=np.float64).copy()
    d = A.shape[0]
    V = np.empty((d, d))
    sw = np.zeros(1, np.int32)
    res = np.zeros(1)
    tol = 1e-9 * float(np.linalg.norm(A, "fro"))
    if device:
        rc = nat.lib().taco_jacobi_sweeps_device(0, nat.ptr(A), nat.ptr(V), d, tol, max_sweeps,
                                                 nat.ptr(sw), nat.ptr(res))
    else:
        rc = nat.lib().taco_jacobi_sweeps(nat.ptr(A), nat.ptr(V), d, tol, max_sweeps, nat.ptr(sw),
                                          nat.ptr(res))
    return rc, A, V, int(sw[0]), float(res[0])


def test_device_jacobi_bit_identical_to_host():
    """eigen.cu (one cooperative kernel) == jacobi.cpp == the reference's sweeps,
    single-CTA (d <= 256) and multi-CTA (d > 256) paths, odd d, zero pairs."""
    rng = np.random.default_rng(11)
    for d in (2, 3, 17, 64, 128, 129, 300, 521):
        X = rng.normal(size=(max(4 * d, 64), d)) @ rng.normal(size=(d, d))
        A = X.T @ X
        A = (A + A.T) / 2.0
        if d == 17:
            A[3, :] = 0.0
            A[:, 3] = 0.0
            A[3, 3] = 2.0
        h = _jac(A, False)
        g = _jac(A, True)
        assert h[0] == 0 and g[0] == 0
        assert h[3] == g[3], (d, h[3], g[3])
        np.testing.assert_array_equal(g[1], h[1])
        np.testing.assert_array_equal(g[2], h[2])


def test_device_jacobi_golden_and_cap(golden):
    from paper_2603_24919_b200 import spectral as S
    u = golden("units")
    for c in range(6):
        w, V = S.jacobi_eigh(u[f"jac{c}_A"])   # device path on a GPU box
        np.testing.assert_array_equal(w, u[f"jac{c}_w"])
        np.testing.assert_array_equal(V, u[f"jac{c}_V"])
    A = np.random.default_rng(0).normal(size=(12, 12))
    rc, *_ , res = _jac(A + A.T, True, max_sweeps=1)
    assert rc == 5 and res > 0


def test_tensor_core_assign_matches_fp64_assign(tmp_path):
    """k_assign_tc (tcgen05 TF32x3 bound + exact fp64 recheck) and the
    all-fp64 k_assign (TACO_TC_ASSIGN=0) give bit-identical k-means runs,
    including duplicate points (seeds that clamp at distance 0), K' not a
    multiple of 16 (padded tensor-core N) and half widths 7, 12, 16, 30 (one,
    two and four TF32 k-blocks per product)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); import paper_2603_24919_b200 as T\n"
        "rng = np.random.default_rng(3)\n"
        "out, hist = [], []\n"
        "for m, k, it in ((7, 50, 6), (7, 64, 4), (7, 100, 3), (12, 64, 3), (16, 40, 3), (30, 64, 3)):\n"
        "    X = (rng.normal(size=(20000, m)) * 40).astype(np.float32)\n"
        "    X[500:900] = X[0]; X[900:950] = X[7]\n"
        "    r = T.kmeans(X, k, it, 11)\n"
        "    out += [r.assignments.astype(np.float64), r.centroids.ravel().astype(np.float64)]\n"
        "    hist.append(np.array(r.inertia_history))\n"
        "np.save(sys.argv[1], np.concatenate(out)); np.save(sys.argv[1] + '.h.npy', np.concatenate(hist))\n"
        % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    res = {}
    for tc in ("0", "1"):
        f = tmp_path / f"r{tc}.npy"
        subprocess.run([sys.executable, "-c", code, str(f)], check=True,
                       env=dict(os.environ, TACO_TC_ASSIGN=tc))
        res[tc] = (np.load(f), np.load(str(f) + ".h.npy"))
    np.testing.assert_array_equal(res["0"][0], res["1"][0])   # labels and centroids: bit-identical
    # the inertia history is a tree sum whose grouping follows the kernel's grid
    np.testing.assert_allclose(res["0"][1], res["1"][1], rtol=1e-12)
