import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2603_24919_b200 as T
from oracle import taco_oracle as O
from paper_2603_24919_b200.distributed import CudaShardBackend, shard_range
from paper_2603_24919_b200.workloads import make_config
X, Q, _ = make_config(1, n=6000, nq=40, d=32)
idx = T.build_index(X, T.IndexParams(8, 4, 64, 10, 2))
oidx = O.deserialize(T.serialize_index(idx))
Qd = torch.from_numpy(Q).cuda()
for a in (0.2, 0.6):
    for r in range(2):
        lo, hi = shard_range(6000, r, 2)
        be = CudaShardBackend(idx, X[lo:hi], lo, 6000, 0)
        h = be.count(Qd, a).cpu().numpy()
        ho = np.array([np.bincount(O.query_scores(oidx, q, a)[lo:hi], minlength=9) for q in Q])
        bad = np.flatnonzero((h != ho).any(1))
        print(a, r, 'hist eq', np.array_equal(h, ho), bad[:4])
        if bad.size:
            print('  gpu', h[bad[0]], '\n  ora', ho[bad[0]])
    full = np.array([np.bincount(O.query_scores(oidx, q, a), minlength=9) for q in Q])
    sc = T.count_collisions(idx, Q[0], a)
    print(' single tap eq', np.array_equal(np.bincount(sc, minlength=9), full[0]))
