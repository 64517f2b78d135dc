"""world_size-2 gloo run of the sharded query orchestration (CPU): traversal
split by query + all-gather of the popped cells (with the cap-overflow
re-run), histogram all-reduce, Alg. 5 on the global histogram, top-k
all-gather + merge must equal the single-process result bit-for-bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import taco_oracle as O
from paper_2603_24919_b200.distributed import shard_range, sharded_query
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
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.shard_oracle import OracleShardBackend
    X, Q, _ = make_config(1, n=cfg["n"], nq=cfg["nq"], d=32)
    oidx = O.build_index(X, 8, 4, 64, 8, 3)
    lo, hi = shard_range(X.shape[0], rank, world)
    be = OracleShardBackend(oidx, X[lo:hi], lo, X.shape[0], tile=cfg.get("tiles", (5, 5))[rank])
    ids, dists, num, lvl = sharded_query(be, torch.from_numpy(Q), cfg["alpha"], cfg["beta"], cfg["k"])
    out_q.put((rank, ids.numpy(), dists.numpy(), num.numpy(), lvl.numpy(), be.pop_cap))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [dict(n=1500, nq=12, alpha=0.05, beta=0.02, k=10),
                                 dict(n=1201, nq=9, alpha=0.3, beta=0.9, k=7),
                                 # ranks whose own tile sizes differ must agree on one
                                 dict(n=1500, nq=11, alpha=0.05, beta=0.02, k=10, tiles=(5, 3))])
def test_sharded_equals_single(cfg):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        try:
            res.append(q.get(timeout=120))
        except Exception:
            break
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert len(res) == world
    X, Q, _ = make_config(1, n=cfg["n"], nq=cfg["nq"], d=32)
    oidx = O.build_index(X, 8, 4, 64, 8, 3)
    oi, od, on, ol = O.knn_batch(oidx, X, Q, cfg["alpha"], cfg["beta"], cfg["k"])
    # the split traversal's cap-overflow re-run (cap 6 -> the all-reduced need) ran with equal caps
    assert all(r[5] > 6 for r in res) and len({r[5] for r in res}) == 1, [r[5] for r in res]
    for _, ids, dists, num, lvl, _ in res:
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(dists, od)
        np.testing.assert_array_equal(num, on)
        np.testing.assert_array_equal(lvl, ol)


def test_shard_range_partitions():
    for n in (1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
