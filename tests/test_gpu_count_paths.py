"""Every counting layout the product runs, against the reference's own
answers (golden fixtures from tests/golden/make_golden.py) and the oracle.

The batched count has three layouts:
  * cluster mode with ONE CTA per query (n small: all earlier rigs);
  * cluster mode with SEVERAL CTAs per query -- the config-2/3 path: per-CTA
    id chunks and candidate segments; the CTAs of a query are a software
    group of the persistent k_count_pg (level histograms exchanged through
    global slots; the default) or, with TACO_COUNT_PG=0, one hardware cluster
    of k_count_enc (histograms gathered over DSMEM, split cluster barrier).
    TACO_CLUSTER_IDS shrinks the chunk so a 20,000-point rig runs it with 10
    CTAs per query;
  * global mode (sharded / n > 1.5M, config 4): per-(query, chunk) CTAs,
    spilled score >= 2 records, emit sweep, recount list -- on the encoded
    CSR (4-entry units, k_count_genc) or, with TACO_COUNT_TMA=0, the
    unit-staged k_count.
and three table widths: 4-bit (N_s <= 15), 8-bit with wide tallies
(N_s = 16, config 3) and 8-bit with a table-scan level histogram (N_s > 16).
rig2 (N_s = 8), rig4 (N_s = 16) and rig5 (N_s = 20) cover the widths; the
modes below cover the layouts.  All must equal the reference bit-for-bit."""

import os

import numpy as np
import pytest

import paper_2603_24919_b200 as T
from oracle import taco_oracle as O
from paper_2603_24919_b200 import _native as nat
from paper_2603_24919_b200.engine import _device_of
from paper_2603_24919_b200.workloads import make_config

pytestmark = pytest.mark.gpu

# mode -> (environment at index creation, expected (cluster mode, min chunks))
MODES = {
    "cluster_1cta": ({}, (True, 1)),
    "cluster_multi": ({"TACO_CLUSTER_IDS": "2048"}, (True, 5)),
    "cluster_odd": ({"TACO_CLUSTER_IDS": "7000"}, (True, 2)),
    "global": ({"TACO_GLOBAL_MODE": "1"}, (False, 1)),
    "global_small_chunk": ({"TACO_GLOBAL_MODE": "1", "TACO_GLOBAL_CHUNK": "2048"}, (False, 5)),
    # the 128K-id chunks (64 KiB tables) global mode takes past 1024 chunks (n > 67M)
    "global_wide_chunk": ({"TACO_GLOBAL_MODE": "1", "TACO_GLOBAL_CHUNK": "131072"}, (False, 1)),
    # global mode without the encoded CSR (the unit-staged k_count sweep)
    "global_units": ({"TACO_GLOBAL_MODE": "1", "TACO_GLOBAL_CHUNK": "2048", "TACO_COUNT_TMA": "0"}, (False, 5)),
}


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.fixture(scope="module", params=["rig2", "rig4", "rig5"])
def rig(request, golden):
    g = golden(request.param)
    cfg, n, nq, d, ns, s, kp, it, seed = (int(v) for v in g["params"])
    X, Q, _ = make_config(cfg, n=n, nq=nq, d=d)
    return request.param, g, X, Q


@pytest.mark.parametrize("mode", list(MODES))
def test_count_layout_matches_reference(rig, mode):
    name, g, X, Q = rig
    env, (want_cluster, min_chunks) = MODES[mode]
    idx = _with_env(env, lambda: T.deserialize_index(g["blob"].tobytes()))
    chunk, nch, cluster = nat.index_layout(_device_of(idx).h)
    assert cluster == want_cluster and nch >= min_chunks, (chunk, nch, cluster)
    # cluster mode: the persistent software groups (default) and the hardware clusters
    for pg in (("1", "0") if want_cluster else ("1",)):
        for gi, (alpha, beta, k) in enumerate(g["grid"]):
            qp = T.QueryParams(alpha=float(alpha), beta=float(beta), k=int(k))
            ids, dists, num, lvl = _with_env({"TACO_COUNT_PG": pg}, lambda: T.knn_query_batch(idx, X, Q, qp))
            np.testing.assert_array_equal(num, g[f"num_{gi}"])
            np.testing.assert_array_equal(lvl, g[f"lvl_{gi}"])
            np.testing.assert_array_equal(ids, g[f"ids_{gi}"])
            np.testing.assert_array_equal(dists, g[f"dists_{gi}"])


def test_multi_cta_against_oracle_many_queries(rig):
    """More queries than the golden rig holds (the oracle answers them), both
    batch tiles, through the 10-CTA cluster path and global mode."""
    name, g, X, Q0 = rig
    cfg, n, nq, d, ns, s, kp, it, seed = (int(v) for v in g["params"])
    _, Q, _ = make_config(cfg, n=n, nq=96, d=d)
    oidx = O.deserialize(g["blob"].tobytes())
    alpha, beta, k = (float(v) for v in g["grid"][-1])
    oi, od, on, ol = O.knn_batch(oidx, X, Q, alpha, beta, int(k), threads=8)
    # 96 queries over 44 groups of 10 CTAs: the persistent groups walk several queries each
    for env, pg in ((MODES["cluster_multi"][0], "1"), (MODES["cluster_multi"][0], "0"),
                    (MODES["global_small_chunk"][0], "1")):
        idx = _with_env(env, lambda: T.deserialize_index(g["blob"].tobytes()))
        ids, dists, num, lvl = _with_env(
            {"TACO_COUNT_PG": pg}, lambda: T.knn_query_batch(idx, X, Q, T.QueryParams(alpha, beta, int(k))))
        np.testing.assert_array_equal(num, on)
        np.testing.assert_array_equal(lvl, ol)
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(dists, od)


def test_scores_tap_wide_levels(rig):
    """count_collisions (uint8 table) equals the reference's table digests,
    including N_s = 16 / 20 where scores exceed a nibble."""
    name, g, X, Q = rig
    idx = T.deserialize_index(g["blob"].tobytes())
    for gi, (alpha, _, _) in enumerate(g["grid"]):
        for qi in range(Q.shape[0]):
            sc = T.count_collisions(idx, Q[qi], float(alpha))
            import hashlib
            assert hashlib.blake2b(sc.tobytes(), digest_size=16).hexdigest() == g[f"scores_digest_{gi}"][qi]


@pytest.mark.parametrize("kernel", ["fused", "pg", "enc", "tma", "units"])
@pytest.mark.parametrize("layout", ["cluster_1cta", "cluster_multi"])
def test_cluster_count_kernels_extreme_budgets(kernel, layout, golden):
    """The cluster count kernels (the encoded, padded CSR with direct loads --
    as persistent software groups, as hardware clusters, or fused with the
    integer re-rank and top-k -- or the cp.async.bulk ring, and the
    unit-staged one) at budgets whose Alg. 5
    walk reaches level 1 (beta -> 1 with a small alpha: the level-1 count
    depends on the padding correction of the level-0 tally) and with almost
    every cell retrieved (alpha -> 1: slices far larger than a ring stage)."""
    g = golden("rig2")
    cfg, n, nq, d, ns, s, kp, it, seed = (int(v) for v in g["params"])
    X, Q, _ = make_config(cfg, n=n, nq=24, d=d)
    oidx = O.deserialize(g["blob"].tobytes())
    env = dict(MODES[layout][0], TACO_COUNT_TMA="0" if kernel == "units" else "1")
    idx = _with_env(env, lambda: T.deserialize_index(g["blob"].tobytes()))
    feed = {"TACO_COUNT_FEED": "tma" if kernel == "tma" else "enc",
            "TACO_FUSED": "1" if kernel == "fused" else "0",
            "TACO_COUNT_PG": "1" if kernel == "pg" else "0"}
    for alpha, beta, k in ((0.999, 0.999, 7), (0.5, 0.2, 10), (0.02, 0.999, 3), (0.999, 0.001, 5)):
        oi, od, on, ol = O.knn_batch(oidx, X, Q, alpha, beta, k, threads=8)
        ids, dists, num, lvl = _with_env(feed, lambda: T.knn_query_batch(idx, X, Q, T.QueryParams(alpha, beta, k)))
        np.testing.assert_array_equal(num, on)
        np.testing.assert_array_equal(lvl, ol)
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(dists, od)


@pytest.mark.parametrize("n_sub", [12, 15])
@pytest.mark.parametrize("layout", ["cluster_1cta", "cluster_multi"])
def test_wide_tallies_nibble_tables(n_sub, layout):
    """N_s 9..15: 4-bit tables with 16 tally levels (the encoded kernel's wide
    path); a GPU-built index answered by the GPU and by the oracle on the same
    v1 bytes (rigs 2/4/5 cover N_s = 8, 16 and 20)."""
    X, Q, _ = make_config(2, n=12000, nq=40, d=4 * n_sub)
    idx = _with_env(MODES[layout][0], lambda: T.build_index(
        X, T.IndexParams(n_subspaces=n_sub, subspace_dim=4, clusters=64, kmeans_iters=5, seed=3)))
    chunk, nch, cluster = nat.index_layout(_device_of(idx).h)
    assert cluster and nch >= MODES[layout][1][1]
    oidx = O.deserialize(T.serialize_index(idx))
    for alpha, beta, k in ((0.05, 0.01, 10), (0.3, 0.05, 7)):
        oi, od, on, ol = O.knn_batch(oidx, X, Q, alpha, beta, k, threads=8)
        ids, dists, num, lvl = T.knn_query_batch(idx, X, Q, T.QueryParams(alpha, beta, k))
        np.testing.assert_array_equal(num, on)
        np.testing.assert_array_equal(lvl, ol)
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(dists, od)
