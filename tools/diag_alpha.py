import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2603_24919_b200 as T
from oracle import taco_oracle as O
from paper_2603_24919_b200.workloads import make_config
X, Q, _ = make_config(1, n=6000, nq=40, d=32)
idx = T.build_index(X, T.IndexParams(8, 4, 64, 10, 2))
oidx = O.deserialize(T.serialize_index(idx))
for a, b, k in [(0.05, 0.01, 10), (0.2, 0.05, 25), (0.6, 0.9, 5), (0.6, 0.05, 5), (0.3, 0.9, 5)]:
    ids0, d0, n0, l0 = T.knn_query_batch(idx, X, Q, T.QueryParams(a, b, k))
    oi, od, on, ol = O.knn_batch(oidx, X, Q, a, b, k)
    bad = np.flatnonzero(n0 != on)
    print(a, b, k, 'ids eq', np.array_equal(ids0, oi), 'num eq', np.array_equal(n0, on), 'lvl eq', np.array_equal(l0, ol), bad[:5])
    if bad.size:
        q = bad[0]
        sc = T.count_collisions(idx, Q[q], a)
        so = O.query_scores(oidx, Q[q], a)
        print('  scores eq', np.array_equal(sc, so), np.bincount(sc, minlength=9), np.bincount(so, minlength=9), n0[q], on[q], l0[q], ol[q])
