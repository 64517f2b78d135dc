"""Score-level statistics of config 2 queries (count-kernel design study)."""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
X, Q, meta = make_config(cfg)
idx = T.build_index(X, T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"]))
ns = meta["n_sub"]
ge = []
Ls = []
for i in range(200):
    sc = T.count_collisions(idx, Q[i], meta["alpha"])
    h = np.bincount(sc, minlength=ns + 1)
    ge.append(np.cumsum(h[::-1])[::-1])
    Ls.append(T.select_candidates(sc, meta["beta"], ns).last_collision)
ge = np.array(ge)
print("L distribution", np.bincount(Ls, minlength=ns + 1))
print("mean #ids with score >= l:", {l: int(ge[:, l].mean()) for l in range(1, ns + 1)})
print("p95 #ids with score >= l:", {l: int(np.percentile(ge[:, l], 95)) for l in range(1, ns + 1)})
