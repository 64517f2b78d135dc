import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2603_24919_b200 as T
from oracle import taco_oracle as O
from paper_2603_24919_b200.distributed import CudaShardBackend, shard_range
from paper_2603_24919_b200.workloads import make_config
X, Q, _ = make_config(1, n=6000, nq=40, d=32)
idx = T.build_index(X, T.IndexParams(8, 4, 64, 10, 2))
oidx = O.deserialize(T.serialize_index(idx))
a, b, k = 0.6, 0.9, 5
ids0, d0, n0, l0 = T.knn_query_batch(idx, X, Q, T.QueryParams(a, b, k))
full = np.array([np.bincount(O.query_scores(oidx, q, a), minlength=9) for q in Q])
bes = [CudaShardBackend(idx, X[lo:hi], lo, 6000, 0) for lo, hi in (shard_range(6000, r, 2) for r in range(2))]
Qd = torch.from_numpy(Q).cuda()
hs = [be.count(Qd, a) for be in bes]
hist = hs[0] + hs[1]
torch.cuda.synchronize()
print('ghist eq oracle', np.array_equal(hist.cpu().numpy(), full))
parts = [be.finish(40, hist, b, k) for be in bes]
torch.cuda.synchronize()
print('ghist after finish eq', np.array_equal(hist.cpu().numpy(), full))
for p in parts:
    print('cnum eq', np.array_equal(p[2].cpu().numpy(), n0), 'lvl eq', np.array_equal(p[3].cpu().numpy(), l0), p[2][:4].tolist(), n0[:4], p[3][:4].tolist(), l0[:4])
budget = b * 6000
q = 0
h = full[q]; L = 8; c = 0
for j in range(8, -1, -1):
    c += int(h[j])
    if h[j] <= budget - c: L -= 1
    else: break
print('python alg5', max(L, 0), c, h)
