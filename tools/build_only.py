"""Build one index (for launch-list profiling of the build path)."""
import sys, time
sys.path.insert(0, '/root/repo')
import paper_2603_24919_b200 as T
from paper_2603_24919_b200.workloads import make_config
cfg = int(sys.argv[1]); n = int(sys.argv[2])
X, Q, m = make_config(cfg, n=n, nq=10)
t = time.perf_counter()
idx = T.build_index(X, T.IndexParams(m['n_sub'], m['s'], m['clusters'], m['kmeans_iters'], 0))
print('build', time.perf_counter() - t, idx.metadata)
