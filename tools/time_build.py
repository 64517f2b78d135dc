"""Cold + warm build timings with the stage split (run on the GPU box).

    python tools/time_build.py CFG [N] [WARM]
"""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
X, Q, m = make_config(cfg, n=n, nq=10)
P = T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], 0)
for i in range(1 + warm):
    t = time.perf_counter()
    idx = T.build_index(X, P)
    w = time.perf_counter() - t
    md = {k: round(v, 4) for k, v in idx.metadata.items() if k.endswith("_seconds")}
    print(json.dumps({"cfg": cfg, "run": "cold" if i == 0 else "warm", "wall": round(w, 4), **md}), flush=True)
    del idx
