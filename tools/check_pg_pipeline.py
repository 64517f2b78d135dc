"""k_count_pg under the two-stream tile pipeline (f32/f16 rows, >= 2 tiles): answers
equal to the hardware-cluster kernel's, no hang.   python tools/check_pg_pipeline.py"""
import os
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

X, Q, m = make_config(1, nq=20000)
idx = T.build_index(X, T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], 0))
qp = T.QueryParams(m["alpha"], m["beta"], m["k"])
out = {}
for pg in ("1", "0"):
    os.environ["TACO_COUNT_PG"] = pg
    for rep in range(3):
        t = time.perf_counter()
        out[pg] = T.knn_query_batch(idx, X, Q, qp)
        dt = time.perf_counter() - t
    print(f"TACO_COUNT_PG={pg}: {Q.shape[0] / dt:.0f} QPS (host wall)", flush=True)
same = all(np.array_equal(a, b) for a, b in zip(out["1"], out["0"]))
print("identical:", same)
sys.exit(0 if same else 1)
