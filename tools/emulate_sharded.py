"""Point-sharded build + query at config scale on ONE GPU (run on the GPU box).

    python tools/emulate_sharded.py --config 4 --world 2 --out gpurun_out/shard_emul.json

`world` processes share cuda:0 and talk over gloo (CUDA tensors staged
through host memory; no kernel waits on another process, so this checks the
protocol, not multi-GPU speed).  Each rank generates only its own rows
(workloads.make_shard), builds collectively (distributed_build.sharded_build)
and answers the query batch through distributed.sharded_query.  Rank 0 then
builds the single-GPU index on the whole matrix and compares the v1 bytes and
every answer.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(rank, world, port, args, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_24919_b200 as T
    from paper_2603_24919_b200.distributed import CudaShardBackend, sharded_query
    from paper_2603_24919_b200.distributed_build import (CudaShardBuilder, aligned_shard_range,
                                                         gather_serialized, sharded_build)
    from paper_2603_24919_b200.workloads import CONFIGS, make_shard
    torch.cuda.set_device(0)
    n = args.n or CONFIGS[args.config]["n"]
    lo, hi = aligned_shard_range(n, rank, world, int(T._native.lib().taco_gram_block_rows()))
    X, Q, meta = make_shard(args.config, lo, hi, n=n, nq=args.nq)
    params = T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"])
    dist.barrier()
    t = time.perf_counter()
    sh = sharded_build(CudaShardBuilder(X, lo, n, params, device=0), params, n)
    build_s = time.perf_counter() - t
    blob = gather_serialized(sh)
    be = CudaShardBackend.from_shard(sh)
    t = time.perf_counter()
    ids, dists, num, lvl = sharded_query(be, torch.from_numpy(Q).cuda(), meta["alpha"], meta["beta"], meta["k"])
    torch.cuda.synchronize()
    q_s = time.perf_counter() - t
    res = dict(rank=rank, rows=[lo, hi], build_seconds=build_s, query_seconds=q_s, blob=blob,
               ids=ids.cpu().numpy(), dists=dists.cpu().numpy(), num=num.cpu().numpy(), lvl=lvl.cpu().numpy())
    q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def main():
    import numpy as np
    import torch.multiprocessing as mp

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, args.world, port, args, q)) for r in range(args.world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=3600) for _ in range(args.world)], key=lambda r: r["rank"])
    for p in procs:
        p.join(timeout=600)
    import paper_2603_24919_b200 as T
    from paper_2603_24919_b200.workloads import make_config
    X, Q, meta = make_config(args.config, n=args.n, nq=args.nq)
    params = T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"])
    t = time.perf_counter()
    idx = T.build_index(X, params)
    single_build = time.perf_counter() - t
    want = T.serialize_index(idx)
    i0, d0, n0, l0 = T.knn_query_batch(idx, X, Q, T.QueryParams(meta["alpha"], meta["beta"], meta["k"]))
    out = {"config": args.config, "n": meta["n"], "world": args.world, "batch": int(Q.shape[0]),
           "emulation": f"{args.world} processes on one GPU, gloo (host-staged) collectives",
           "single_gpu_build_seconds": single_build, "ranks": []}
    for r in res:
        out["ranks"].append({
            "rank": r["rank"], "rows": r["rows"], "build_seconds": r["build_seconds"],
            "query_seconds": r["query_seconds"],
            "index_bytes_identical": r["blob"] == want,
            "ids_identical": bool(np.array_equal(r["ids"], i0)),
            "dists_identical": bool(np.array_equal(r["dists"], d0)),
            "candidate_num_identical": bool(np.array_equal(r["num"], n0)),
            "last_collision_identical": bool(np.array_equal(r["lvl"], l0))})
    out["identical"] = all(all(v for k, v in rk.items() if k.endswith("identical")) for rk in out["ranks"])
    print(json.dumps(out))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
