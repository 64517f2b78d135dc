"""Point-sharded collective build (distributed_build.py) with
gloo on CPU: column-sum and Gram chains in rank order, the k-means halves run
by their subspace owners after an all-to-all of the transformed columns, the
labels sent back, the cell sizes all-reduced.  The v1 bytes of the index
assembled from the shards must not depend on the number of ranks, and every
rank's global size table must equal the whole index's cell sizes."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_24919_b200.workloads import make_config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["TACO_EIG"] = "host"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_24919_b200 as T
        from paper_2603_24919_b200.distributed_build import aligned_shard_range, gather_serialized, sharded_build
        from tests.shard_oracle import OracleShardBuilder
        X, _, _ = make_config(1, n=cfg["n"], nq=1, d=32)
        params = T.IndexParams(cfg["n_sub"], cfg["s"], cfg["clusters"], 6, 3)
        lo, hi = aligned_shard_range(X.shape[0], rank, world, 256)
        be = OracleShardBuilder(X[lo:hi], lo, X.shape[0], params, block=256)
        sh = sharded_build(be, params, X.shape[0])
        blob = gather_serialized(sh)
        out_q.put((rank, blob, be.global_sizes, sh.histories[0][0]))
    finally:
        dist.destroy_process_group()


def _run(world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        try:
            res.append(q.get(timeout=240))
        except Exception:
            break
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("cfg", [dict(n=1500, n_sub=4, s=8, clusters=16),
                                 dict(n=1100, n_sub=8, s=4, clusters=9)])
def test_sharded_build_independent_of_world(cfg):
    one = _run(1, cfg)
    for world in (2, 3):
        many = _run(world, cfg)
        for r in many:
            assert r[1] == one[0][1], f"world {world} rank {r[0]}: v1 bytes differ"
            np.testing.assert_array_equal(r[2], one[0][2])
            assert r[3] == one[0][3]


def test_aligned_shards_partition():
    from paper_2603_24919_b200.distributed_build import aligned_shard_range, owned_subspaces
    for n in (1, 1000, 4097, 10_000_000):
        for w in (1, 2, 3, 8):
            parts = [aligned_shard_range(n, r, w, 4096) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            assert all(lo % 4096 == 0 or lo == n for lo, _ in parts)
    for ns in (1, 8, 16):
        for w in (1, 2, 3, 8):
            got = sum((owned_subspaces(ns, r, w) for r in range(w)), [])
            assert got == list(range(ns))
