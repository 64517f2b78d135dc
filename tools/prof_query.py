"""Build config CFG once, run the query batch REPS times (ncu target).

    python tools/prof_query.py CFG NQ [REPS]
"""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

cfg, nq = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
X, Q, m = make_config(cfg, nq=nq)
idx = T.build_index(X, T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], 0))
qp = T.QueryParams(m["alpha"], m["beta"], m["k"])
for r in range(reps):
    t = time.perf_counter()
    ids, d, num, lvl = T.knn_query_batch(idx, X, Q, qp)
    print(f"rep {r}: {nq / (time.perf_counter() - t):.0f} QPS (host wall), mean |C| {num.mean():.1f}, "
          f"levels {np.bincount(lvl).tolist()}", flush=True)
