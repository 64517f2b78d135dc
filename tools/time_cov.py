"""Host-side split of the covariance stage of build_index (tools/)."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200 import _native as nat  # noqa: E402
from paper_2603_24919_b200.engine import _data_key  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

X, Q, meta = make_config(2, nq=16)
P = T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"])
T.build_index(X, P)
for rep in range(3):
    t = [time.perf_counter()]
    dev = nat.DeviceIndex(X.shape[0], X.shape[1], P.n_subspaces, P.subspace_dim, P.clusters, P.kmeans_iters)
    t.append(time.perf_counter())
    nat.call("taco_index_set_data", dev.h, nat.ptr(X))
    t.append(time.perf_counter())
    _data_key(X)
    t.append(time.perf_counter())
    mean = np.empty(X.shape[1]); gram = np.empty((X.shape[1],) * 2); bad = np.zeros(1, np.int64)
    nat.call("taco_fit_covariance", dev.h, nat.ptr(mean), nat.ptr(gram), nat.ptr(bad))
    t.append(time.perf_counter())
    print("create %.2f  set_data %.2f  data_key %.2f  fit_cov %.2f ms" % tuple(1e3 * (t[i + 1] - t[i]) for i in range(4)))
    del dev
