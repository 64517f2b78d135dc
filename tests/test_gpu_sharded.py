"""CUDA shard backend on ONE GPU: two point shards counted separately, their
histograms summed (standing in for the NCCL all-reduce, no cross-kernel
waiting), Alg. 5 + rerank per shard, device merge -> must equal the
single-GPU batched path bit-for-bit."""

import numpy as np
import pytest
import torch

import paper_2603_24919_b200 as T
from paper_2603_24919_b200.distributed import CudaShardBackend, shard_range
from paper_2603_24919_b200.workloads import make_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chunk", [None, "1024"])
@pytest.mark.parametrize("world,alpha,beta,k", [(2, 0.05, 0.01, 10), (3, 0.2, 0.05, 25), (2, 0.6, 0.9, 5)])
def test_two_shards_match_single(world, alpha, beta, k, chunk, monkeypatch):
    """chunk=1024 cuts each shard into several id chunks whose spilled
    score >= 2 records (slot = 128) overflow at the larger alphas, so the
    emit sweep's record filter, its recount fallback and the L < 2 recount
    all run."""
    X, Q, _ = make_config(1, n=6000, nq=40, d=32)
    idx = T.build_index(X, T.IndexParams(8, 4, 64, 10, 2))
    ids0, d0, n0, l0 = T.knn_query_batch(idx, X, Q, T.QueryParams(alpha, beta, k))
    if chunk:
        monkeypatch.setenv("TACO_GLOBAL_CHUNK", chunk)
    bes = []
    for r in range(world):
        lo, hi = shard_range(X.shape[0], r, world)
        bes.append(CudaShardBackend(idx, X[lo:hi], lo, X.shape[0], 0))
    Qd = torch.from_numpy(Q).cuda()
    T_ = min(b.tile_size() for b in bes)
    outs = []
    for q0 in range(0, Q.shape[0], T_):
        Qt = Qd[q0:q0 + T_]
        m = Qt.shape[0]
        hist = sum(b.count(Qt, alpha) for b in bes)
        parts = [b.finish(m, hist, beta, k) for b in bes]
        d2_all = torch.stack([p[0] for p in parts])
        id_all = torch.stack([p[1] for p in parts])
        oi, od = bes[0].merge(d2_all, id_all, k)
        torch.cuda.synchronize()
        outs.append((oi.cpu().numpy(), od.cpu().numpy(), parts[0][2].cpu().numpy(), parts[0][3].cpu().numpy()))
        for p in parts[1:]:
            np.testing.assert_array_equal(p[2].cpu().numpy(), outs[-1][2])
    ids = np.concatenate([o[0] for o in outs])
    np.testing.assert_array_equal(ids, ids0)
    np.testing.assert_array_equal(np.concatenate([o[1] for o in outs]), d0)
    np.testing.assert_array_equal(np.concatenate([o[2] for o in outs]), n0)
    np.testing.assert_array_equal(np.concatenate([o[3] for o in outs]), l0)


@pytest.mark.parametrize("world,alpha,beta,k,cap", [(2, 0.05, 0.01, 10, 64), (3, 0.2, 0.05, 25, 4)])
def test_split_traversal_matches_single(world, alpha, beta, k, cap):
    """distributed._split_count on one GPU: every shard walks only its slice
    of the tile's queries (taco_query_front_device), the slices are copied
    into every shard's pop buffers (standing in for the in-place NCCL
    all_gather), each shard counts its ids (taco_query_count_popped_device).
    cap=4 forces the cap-overflow re-run at the measured need.  Must equal the
    single-GPU batch bit-for-bit."""
    X, Q, _ = make_config(1, n=6000, nq=40, d=32)
    idx = T.build_index(X, T.IndexParams(8, 4, 64, 10, 2))
    ids0, d0, n0, l0 = T.knn_query_batch(idx, X, Q, T.QueryParams(alpha, beta, k))
    bes = []
    for r in range(world):
        lo, hi = shard_range(X.shape[0], r, world)
        bes.append(CudaShardBackend(idx, X[lo:hi], lo, X.shape[0], 0))
        bes[-1].pop_cap = cap
    Qd = torch.from_numpy(Q).cuda()
    T_ = min(b.tile_size() for b in bes)
    outs = []
    raised = False
    for q0 in range(0, Q.shape[0], T_):
        Qt = Qd[q0:q0 + T_]
        m = Qt.shape[0]
        per = -(-m // world)
        rows = per * world
        for _ in range(2):
            need = max(b.front(Qt, alpha, min(m, r * per), min(m, r * per + per), rows) for r, b in enumerate(bes))
            if need == 0:
                break
            raised = True
            for b in bes:
                b.raise_pop_cap(need)
        views = [b.pop_views(rows) for b in bes]
        for r in range(world):              # all_gather: rank r's rows to every rank
            for dst in range(world):
                if dst != r:
                    for vd, vs in zip(views[dst], views[r]):
                        vd[r * per:(r + 1) * per].copy_(vs[r * per:(r + 1) * per])
        hist = sum(b.count_popped(m) for b in bes)
        parts = [b.finish(m, hist, beta, k) for b in bes]
        d2_all = torch.stack([p[0] for p in parts])
        id_all = torch.stack([p[1] for p in parts])
        oi, od = bes[0].merge(d2_all, id_all, k)
        torch.cuda.synchronize()
        outs.append((oi.cpu().numpy(), od.cpu().numpy(), parts[0][2].cpu().numpy(), parts[0][3].cpu().numpy()))
    assert raised == (cap < 64)
    np.testing.assert_array_equal(np.concatenate([o[0] for o in outs]), ids0)
    np.testing.assert_array_equal(np.concatenate([o[1] for o in outs]), d0)
    np.testing.assert_array_equal(np.concatenate([o[2] for o in outs]), n0)
    np.testing.assert_array_equal(np.concatenate([o[3] for o in outs]), l0)


@pytest.mark.parametrize("chunk", [None, "1024"])
def test_global_mode_matches_cluster_mode(chunk, monkeypatch):
    """One unsharded index counted both ways: cluster mode (DSMEM-fused
    count/select) and global mode (TACO_GLOBAL_MODE=1: per-chunk histograms,
    spilled score >= 2 records, warp record filter, persistent recount of the
    listed chunks).  chunk=1024 makes record slots overflow; beta=0.9 drives
    L below 2 (the recount path).  Results must be identical."""
    X, Q, _ = make_config(1, n=7000, nq=48, d=32)
    P = T.IndexParams(8, 4, 64, 10, 2)
    idx_c = T.build_index(X, P)
    monkeypatch.setenv("TACO_GLOBAL_MODE", "1")
    if chunk:
        monkeypatch.setenv("TACO_GLOBAL_CHUNK", chunk)
    idx_g = T.build_index(X, P)
    for alpha, beta, k in ((0.05, 0.01, 10), (0.3, 0.2, 16), (0.6, 0.9, 5)):
        qp = T.QueryParams(alpha, beta, k)
        a = T.knn_query_batch(idx_c, X, Q, qp)
        b = T.knn_query_batch(idx_g, X, Q, qp)
        for u, v in zip(a, b):
            np.testing.assert_array_equal(u, v)


def test_split_traversal_errors():
    """The split-traversal entry points fail loudly on bad slices / caps and on
    an unsharded (cluster-mode) index, like the reference's ParameterError."""
    import ctypes

    from paper_2603_24919_b200 import _native as nat
    from paper_2603_24919_b200.errors import ParameterError, StateError

    X, Q, _ = make_config(1, n=3000, nq=8, d=32)
    idx = T.build_index(X, T.IndexParams(8, 4, 64, 10, 2))
    be = CudaShardBackend(idx, X[:1500], 0, X.shape[0], 0)
    Qd = torch.from_numpy(Q).cuda()
    with pytest.raises(ParameterError):
        be.front(Qd, 0.1, 5, 3, 8)            # lo > hi
    with pytest.raises(ParameterError):
        be.front(Qd, 0.1, 0, 8, 4)            # rows < nq
    be.pop_cap = 10_000                        # above K'^2
    with pytest.raises(ParameterError):
        be.front(Qd, 0.1, 0, 8, 8)
    whole = T.build_index(X, T.IndexParams(8, 4, 64, 10, 2))   # unsharded: cluster mode
    need = ctypes.c_int64(0)
    with pytest.raises(StateError):
        nat.call("taco_query_front_device", T.engine._device_of(whole).h, Qd.data_ptr(), 8, 0, 8, 8, 0.1, 64,
                 ctypes.byref(need), None)
