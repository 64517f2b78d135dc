"""Per-kernel times of one config-2 batch at a chosen k (k > 32 keeps every candidate in the
partial lists, the config-5 top-k regime).   python tools/prof_topk_k.py [k] [nq]"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200 import _native as nat  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 100
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
X, Q, m = make_config(2, nq=nq)
idx = T.build_index(X, T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], 0))
qp = T.QueryParams(m["alpha"], m["beta"], k)
out = T.knn_query_batch(idx, X, Q, qp)
nat.profile_enable(True)
nat.profile_read(reset=True)
out = T.knn_query_batch(idx, X, Q, qp)
prof, _ = nat.profile_read(reset=True)
print(f"k={k} nq={nq}", {kk: round(v[0], 3) for kk, v in prof.items() if v[0] > 0.005})
print("ids checksum", int(np.asarray(out[0], np.int64).sum()))
