"""Back-to-back config-2 builds: the staged upload's host-copy time with and
without a pause before each build (finds host threads left spinning by the
previous build)."""
import os, sys, time
os.environ["TACO_DEBUG_UPLOAD"] = "1"
sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T
from paper_2603_24919_b200.workloads import make_config
X, Q, m = make_config(2, nq=16)
P = T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], m["seed"])
idx = T.build_index(X, P)
for pause in (0, 0, 0, 0.3, 0.3, 0.3, 0, 0):
    time.sleep(pause)
    t = time.perf_counter(); idx = T.build_index(X, P)
    print(f"pause {pause}: build {1e3*(time.perf_counter()-t):.1f} ms", file=sys.stderr, flush=True)
