"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/taco read-only under the module name
``taco_ref`` (no bytecode written) and stores its outputs on small seeded
inputs as compressed .npz files next to this script.  Inputs are
regenerated from seeds by ``paper_2603_24919_b200.workloads`` and the
``rng`` recipes below, so only outputs are committed.
"""

from __future__ import annotations

import hashlib
import importlib.util
import math
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from paper_2603_24919_b200.workloads import make_config  # noqa: E402

REF = "/root/reference/pkg/src/taco"

# (name, cfg, n, nq, d, n_sub, s, kprime, iters, seed, query grid [(alpha, beta, k)])
RIGS = [
    ("rig1", 1, 3000, 24, 32, 8, 4, 8, 10, 5, [(0.05, 0.01, 10), (0.1, 0.05, 20)]),
    ("rig2", 2, 20000, 16, 128, 8, 16, 16, 20, 0, [(0.03, 0.01, 10)]),
    ("rig3", 3, 4000, 12, 60, 4, 15, 6, 20, 3, [(0.05, 0.02, 10)]),
    # N_s = 16: 8-bit count tables with wide tallies (the config-3 count path)
    ("rig4", 3, 20000, 16, 64, 16, 4, 8, 10, 7, [(0.05, 0.01, 10), (0.2, 0.05, 10)]),
    # N_s = 20: levels above 16 (table-scan level histogram), half widths 2 / 1
    ("rig5", 4, 12000, 12, 64, 20, 3, 6, 10, 9, [(0.05, 0.01, 10), (0.3, 0.1, 12)]),
]


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "taco_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["taco_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def digest(a) -> str:
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=16).hexdigest()


def rig_fixture(ref, name, cfg, n, nq, d, n_sub, s, kp, iters, seed, grid):
    X, Q, _ = make_config(cfg, n=n, nq=nq, d=d)
    params = ref.IndexParams(n_subspaces=n_sub, subspace_dim=s, clusters=kp * kp,
                             kmeans_iters=iters, seed=seed)
    index = ref.build_index(X, params)
    out = {
        "params": np.array([cfg, n, nq, d, n_sub, s, kp, iters, seed], np.int64),
        "mean": index.transform.mean,
        "blocks": np.stack(index.transform.blocks),
        "blob": np.frombuffer(ref.serialize_index(index), np.uint8),
        "grid": np.array(grid, np.float64),
    }
    for j, sub in enumerate(index.subspaces):
        out[f"cb1_{j}"] = sub.codebook1.centroids
        out[f"cb2_{j}"] = sub.codebook2.centroids
        out[f"lab1_{j}"] = sub.codebook1.assignments
        out[f"lab2_{j}"] = sub.codebook2.assignments
        out[f"hist1_{j}"] = np.array(sub.codebook1.inertia_history)
        out[f"hist2_{j}"] = np.array(sub.codebook2.inertia_history)
    out["T_head"] = ref.transform_points(index.transform, X[:200])
    out["QT"] = ref.transform_points(index.transform, Q)
    for g, (alpha, beta, k) in enumerate(grid):
        ids = np.full((nq, k), -1, np.int32)
        dists = np.full((nq, k), np.inf, np.float32)
        num = np.zeros(nq, np.int64)
        lvl = np.zeros(nq, np.int32)
        sdig = []
        pops = []
        for qi in range(nq):
            sc = ref.count_collisions(index, Q[qi], alpha)
            cand = ref.select_candidates(sc, beta, n_sub, n)
            res = ref.rerank(X, Q[qi], cand, k)
            ids[qi, :res.ids.size] = res.ids
            dists[qi, :res.dists.size] = res.dists
            num[qi] = cand.candidate_num
            lvl[qi] = cand.last_collision
            sdig.append(digest(sc))
            if qi < 4:
                qt = ref.transform_points(index.transform, Q[qi][None, :])[0]
                for j, sub in enumerate(index.subspaces):
                    d1, i1, d2, i2 = ref.sorted_centroid_distances(sub, qt[j * s:(j + 1) * s])
                    act = ref.scalable_dynamic_activation(alpha, n, kp * kp, d1, i1, d2, i2, sub)
                    for key, a, b in act.pop_trace:
                        pops.append((qi, j, a, b, key, act.retrieved_num))
        out[f"ids_{g}"] = ids
        out[f"dists_{g}"] = dists
        out[f"num_{g}"] = num
        out[f"lvl_{g}"] = lvl
        out[f"scores_digest_{g}"] = np.array(sdig)
        out[f"pops_{g}"] = np.array(pops, np.float64)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "blob", len(out["blob"]), "bytes")


def unit_fixture(ref):
    out = {}
    rng = np.random.default_rng(77)
    # k-means cases: (n, m, k, iters, seed) on rng data (clustering.py:57-115)
    km = [(300, 5, 8, 25, 5), (200, 4, 10, 15, 7), (1000, 8, 16, 20, 11),
          (500, 3, 40, 6, 13), (64, 2, 64, 5, 17), (2000, 6, 30, 20, 19)]
    for c, (n, m, k, it, sd) in enumerate(km):
        X = np.random.default_rng(1000 + c).normal(size=(n, m)).astype(np.float32)
        if c == 3:
            X[100:300] = X[0]                  # duplicate points -> empty clusters
        r = ref.kmeans(X, k, it, sd)
        out[f"km{c}_cfg"] = np.array([n, m, k, it, sd], np.int64)
        out[f"km{c}_cent"] = r.centroids
        out[f"km{c}_lab"] = r.assignments
        out[f"km{c}_hist"] = np.array(r.inertia_history)
    # Jacobi eigensystems (spectral.py:139-195) on random SPD matrices
    for c, dd in enumerate([2, 3, 5, 8, 16, 33]):
        B = rng.normal(size=(dd, dd))
        A = B @ B.T + np.diag(rng.uniform(0, 1, dd))
        w, V = ref.jacobi_eigh(A)
        out[f"jac{c}_A"] = A
        out[f"jac{c}_w"] = w
        out[f"jac{c}_V"] = V
    # traversal instances with integer distances -> ties (helpers.py:33-62)
    trav = []
    for c in range(60):
        kp = int(rng.integers(2, 9))
        d1 = rng.integers(0, 6, kp).astype(np.float64) if c % 2 else rng.uniform(0, 10, kp)
        d2 = rng.integers(0, 6, kp).astype(np.float64) if c % 2 else rng.uniform(0, 10, kp)
        sizes = rng.integers(1, 7, size=(kp, kp))
        sizes[rng.random((kp, kp)) < 0.3] = 0
        if sizes.sum() == 0:
            sizes[0, 0] = 1
        tot = int(sizes.sum())
        alpha = float(rng.uniform(0.05, 1.0))
        flat = np.arange(tot, dtype=np.uint32)
        bounds = np.concatenate(([0], np.cumsum(sizes.ravel())))
        cells = {}
        for l1 in range(kp):
            for l2 in range(kp):
                slot = l1 * kp + l2
                if sizes[l1, l2]:
                    cells[(l1, l2)] = flat[bounds[slot]:bounds[slot + 1]]
        cb = ref.KMeansModel(centroids=np.zeros((kp, 1), np.float32), assignments=None, inertia=0.0)
        imi = ref.InvertedMultiIndex(codebook1=cb, codebook2=cb, cells=cells,
                                     codebook_size=kp, split=1)
        i1 = np.argsort(d1, kind="stable")
        i2 = np.argsort(d2, kind="stable")
        act = ref.scalable_dynamic_activation(alpha, tot, kp * kp, d1, i1, d2, i2, imi)
        out[f"tr{c}_d1"] = d1
        out[f"tr{c}_d2"] = d2
        out[f"tr{c}_sizes"] = sizes
        out[f"tr{c}_alpha"] = np.array([alpha])
        out[f"tr{c}_pops"] = np.array([(a, b) for _, a, b in act.pop_trace], np.int64)
        out[f"tr{c}_ret"] = np.array([act.retrieved_num])
        trav.append(c)
    out["n_trav"] = np.array([len(trav)])
    # Alg. 5 threshold scan on random histograms (engine.py:223-253)
    sel = []
    for c in range(300):
        ns = int(rng.integers(1, 17))
        h = rng.integers(0, 60, ns + 1)
        if h.sum() == 0:
            h[0] = 1
        sc = np.repeat(np.arange(ns + 1), h).astype(np.uint8)
        rng.shuffle(sc)
        beta = float(rng.uniform(0.001, 0.95))
        cs = ref.select_candidates(sc, beta, ns)
        sel.append([ns, beta, cs.last_collision, cs.candidate_num] + list(h) + [-1] * (16 - ns))
    out["select"] = np.array(sel, np.float64)
    # seeds (seeding.py:16-20)
    out["seeds"] = np.array([[r, p, ref.seeding.derive_seed(r, p)] for r in (0, 5, 123456789)
                             for p in range(4)], np.uint64)
    np.savez_compressed(os.path.join(HERE, "units.npz"), **out)
    print("units", len(out))


SC_CASES = [  # (seed, n, n_sub, s, integer-valued T)
    (11, 3000, 4, 8, False),
    (12, 2500, 8, 4, True),     # integer coordinates: many distance ties, decided by id
]
SC_ALPHAS = [0.01, 0.05, 0.3, 1.0]


def sc_inputs(seed, n, n_sub, s, ints):
    rng = np.random.default_rng([77, seed])
    if ints:
        T = rng.integers(-3, 4, (n, n_sub * s)).astype(np.float32)
        q = rng.integers(-3, 4, (6, n_sub * s)).astype(np.float32)
    else:
        T = rng.standard_normal((n, n_sub * s)).astype(np.float32)
        q = rng.standard_normal((6, n_sub * s)).astype(np.float32)
    return T, q


def sc_fixture(ref):
    """engine.sc_linear_scores on seeded transformed matrices, and
    sc_linear_query on the rig1 index (reference-built, transformed attached)."""
    out = {}
    for ci, (seed, n, n_sub, s, ints) in enumerate(SC_CASES):
        T, q = sc_inputs(seed, n, n_sub, s, ints)
        for qi in range(q.shape[0]):
            for ai, a in enumerate(SC_ALPHAS):
                out[f"sc_{ci}_{qi}_{ai}"] = ref.engine.sc_linear_scores(T, q[qi], n_sub, s, a)
    name, cfg, n, nq, d, n_sub, s, kp, iters, seed, grid = RIGS[0]
    X, Q, _ = make_config(cfg, n=n, nq=nq, d=d)
    blob = np.load(os.path.join(HERE, f"{name}.npz"))["blob"].tobytes()
    index = ref.engine.deserialize_index(blob) if hasattr(ref.engine, "deserialize_index") else None
    if index is None:
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".taco") as fh:
            fh.write(blob)
            fh.flush()
            index = ref.load_index(fh.name)
    ref.attach_transformed(index, X)
    for qi in range(8):
        for gi, (a, b, k) in enumerate([(0.05, 0.01, 10), (0.2, 0.05, 15)]):
            r = ref.engine.sc_linear_query(index, X, Q[qi], ref.QueryParams(alpha=a, beta=b, k=k))
            out[f"q_{qi}_{gi}_ids"] = r.ids
            out[f"q_{qi}_{gi}_dists"] = r.dists
    np.savez_compressed(os.path.join(HERE, "sclinear.npz"), **out)


# (n, d, nq, k, integer-valued) -- inputs are rng(n + d) draws as in tests/test_dataio.py
GT_CASES = [(5000, 32, 40, 10, False), (3000, 128, 33, 100, True), (2000, 37, 20, 7, False),
            (1500, 960, 5, 10, False)]


def gt_inputs(n, d, nq, ints):
    rng = np.random.default_rng(n + d)
    if ints:   # integer data: many exact distance ties -> id order decides
        return (rng.integers(0, 4, (n, d)).astype(np.float32), rng.integers(0, 4, (nq, d)).astype(np.float32))
    return rng.standard_normal((n, d)).astype(np.float32), rng.standard_normal((nq, d)).astype(np.float32)


def gt_fixture(ref):
    """dataio.compute_ground_truth (dataio.py:142-172) on small seeded inputs."""
    out = {"cases": np.array([[n, d, nq, k, int(i)] for n, d, nq, k, i in GT_CASES], np.int64)}
    for ci, (n, d, nq, k, ints) in enumerate(GT_CASES):
        X, Q = gt_inputs(n, d, nq, ints)
        gt = ref.dataio.compute_ground_truth(X, Q, k)
        out[f"ids_{ci}"] = gt.ids
        out[f"dists_{ci}"] = gt.dists
    np.savez_compressed(os.path.join(HERE, "groundtruth.npz"), **out)


def main():
    ref = load_reference()
    if sys.argv[1:] == ["sclinear"]:
        sc_fixture(ref)
        return
    if sys.argv[1:] == ["groundtruth"]:
        gt_fixture(ref)
        return
    if sys.argv[1:]:   # named rigs only, e.g. `make_golden.py rig4 rig5`
        for rig in RIGS:
            if rig[0] in sys.argv[1:]:
                rig_fixture(ref, *rig)
        return
    unit_fixture(ref)
    for rig in RIGS:
        rig_fixture(ref, *rig)
    sc_fixture(ref)
    gt_fixture(ref)


if __name__ == "__main__":
    main()
