"""Per-half k-means++ / Lloyd split (TACO_DEBUG_TIMING) of one warm build."""
import os, sys
sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T
from paper_2603_24919_b200.workloads import make_config
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
X, Q, m = make_config(cfg, nq=16)
P = T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], m["seed"])
T.build_index(X, P)
os.environ["TACO_DEBUG_TIMING"] = "1"
T.build_index(X, P)
