"""Per-rank work of the point-sharded query path at G ranks, measured on one
GPU: shard 0 of G runs stage 1 -> (histogram = G x local, standing in for the
all-reduce) -> finish on the config-2 batch.  Stage 1 two ways: every rank
walks all queries (`count`), or the split traversal (`front` on rank 0's
slice, all_gather omitted, `count_popped`).  Compare with the single-GPU batch."""
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200 import _native as nat  # noqa: E402
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

    def run(split):
        for q0 in range(0, Q.shape[0], T_):
            Qt = Qd[q0:q0 + T_]
            m = Qt.shape[0]
            if split:
                per = -(-m // G)
                need = be.front(Qt, a, 0, min(m, per), per * G)
                if need:   # (first batch only: the raised cap is kept)
                    be.raise_pop_cap(need)
                    assert be.front(Qt, a, 0, min(m, per), per * G) == 0
                h = be.count_popped(m)
            else:
                h = be.count(Qt, a)
            # G x the local histogram stands in for the all-reduced one (points are sharded at random
            # with respect to the clusters, so the shards' histograms are alike); the local one alone
            # would put Alg. 5 a level deeper and re-rank several times the real candidates
            be.finish(m, h * G, b, k)

    for split in (False, True):
        if split:   # settle the cap, then walk every row once so the rows rank 0 skips hold valid cells
            for q0 in range(0, Q.shape[0], T_):
                Qt = Qd[q0:q0 + T_]
                m = Qt.shape[0]
                rows = -(-m // G) * G
                need = be.front(Qt, a, 0, m, rows)
                if need:
                    be.raise_pop_cap(need)
                    assert be.front(Qt, a, 0, m, rows) == 0
        run(split)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            run(split)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / 3 * 1000
        nat.profile_enable(True)
        nat.profile_read(reset=True)
        run(split)
        torch.cuda.synchronize()
        prof, _ = nat.profile_read(reset=True)
        nat.profile_enable(False)
        print(f"G={G} shard0 [{lo},{hi}) {'split' if split else 'full '} walk: per-rank ms {ms:.2f} "
              f"(implied {Q.shape[0] / ms * 1000:.0f} QPS if ranks scale)")
        print("   ", {kk: round(v[0], 3) for kk, v in prof.items() if v[0] > 0.02}, "pop_cap", be.pop_cap)
    del be
