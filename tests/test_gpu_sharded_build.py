"""The point-sharded collective build (distributed_build.py) and the sharded
query on ONE B200: 2 or 3 processes share the GPU and talk over gloo (CUDA
tensors staged through host memory; no kernel waits on another process), each
holding only its own rows.  The index assembled from the shards must be
byte-identical (v1 format) to the single-GPU build_index on the whole
matrix, and the sharded query must answer exactly like the single-GPU batch."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(cfg=1, n=20000, nq=64, d=32, params=(8, 4, 64, 10, 2), query=(0.05, 0.01, 10))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_24919_b200 as T
        from paper_2603_24919_b200.distributed import CudaShardBackend, sharded_query
        from paper_2603_24919_b200.distributed_build import (CudaShardBuilder, aligned_shard_range,
                                                             gather_serialized, sharded_build)
        from paper_2603_24919_b200.workloads import make_config
        torch.cuda.set_device(0)
        X, Q, _ = make_config(cfg["cfg"], n=cfg["n"], nq=cfg["nq"], d=cfg["d"])
        params = T.IndexParams(*cfg["params"])
        lo, hi = aligned_shard_range(X.shape[0], rank, world, int(T._native.lib().taco_gram_block_rows()))
        be = CudaShardBuilder(X[lo:hi], lo, X.shape[0], params, device=0)
        sh = sharded_build(be, params, X.shape[0])
        blob = gather_serialized(sh)
        a, b, k = cfg["query"]
        qb = CudaShardBackend.from_shard(sh)
        ids, dists, num, lvl = sharded_query(qb, torch.from_numpy(Q).cuda(), a, b, k)
        out_q.put((rank, blob, ids.cpu().numpy(), dists.cpu().numpy(), num.cpu().numpy(), lvl.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_build_and_query_match_single_gpu(world):
    import paper_2603_24919_b200 as T
    from paper_2603_24919_b200.workloads import make_config

    cfg = dict(CFG, n=20000 if world == 2 else 9000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        try:
            res.append(q.get(timeout=300))
        except Exception:
            break
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world
    X, Q, _ = make_config(cfg["cfg"], n=cfg["n"], nq=cfg["nq"], d=cfg["d"])
    idx = T.build_index(X, T.IndexParams(*cfg["params"]))
    want = T.serialize_index(idx)
    a, b, k = cfg["query"]
    i0, d0, n0, l0 = T.knn_query_batch(idx, X, Q, T.QueryParams(a, b, k))
    for rank, blob, ids, dists, num, lvl in res:
        assert blob == want, f"rank {rank}: sharded index bytes differ from the single-GPU build"
        np.testing.assert_array_equal(ids, i0)
        np.testing.assert_array_equal(dists, d0)
        np.testing.assert_array_equal(num, n0)
        np.testing.assert_array_equal(lvl, l0)
