"""Per-rank work of the point-sharded query path at G ranks, measured on one
GPU: shard 0 of G runs count -> (histogram = local, standing in for the
all-reduce) -> finish on the config-2 batch.  Compare with the single-GPU batch."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200.distributed import CudaShardBackend, shard_range  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

X, Q, meta = make_config(2)
idx = T.build_index(X, T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"]))
Qd = torch.from_numpy(Q).cuda()
a, b, k = meta["alpha"], meta["beta"], meta["k"]
n = X.shape[0]
for G in (2, 4, 8):
    lo, hi = shard_range(n, 0, G)
    be = CudaShardBackend(idx, X[lo:hi], lo, n, 0)
    T_ = be.tile_size()
    def run():
        for q0 in range(0, Q.shape[0], T_):
            Qt = Qd[q0:q0 + T_]
            h = be.count(Qt, a)
            d2, ids, num, lvl = be.finish(Qt.shape[0], h, b, k)
    run(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 3 * 1000
    print(f"G={G} shard0 [{lo},{hi}) per-rank ms {ms:.2f}  (implied {Q.shape[0] / ms * 1000:.0f} QPS if ranks scale)")
    del be
    # per-kernel split of one more pass (CUDA events on the launching stream)
    from paper_2603_24919_b200 import _native as nat  # noqa: E402
    be = CudaShardBackend(idx, X[lo:hi], lo, n, 0)
    run(); torch.cuda.synchronize()
    nat.profile_enable(True)
    nat.profile_read(reset=True)
    run(); torch.cuda.synchronize()
    prof, _ = nat.profile_read(reset=True)
    nat.profile_enable(False)
    print("   ", {k: round(v[0], 3) for k, v in prof.items() if v[0] > 0.02})
    del be
