"""Which (k, iters) case differs between the tensor-core and fp64 assignment (tools/)."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
if len(sys.argv) > 2:
    import paper_2603_24919_b200 as T
    rng = np.random.default_rng(3)
    X = (rng.normal(size=(20000, 7)) * 40).astype(np.float32)
    if sys.argv[3] == "dup":
        X[500:900] = X[0]
        X[900:950] = X[7]
    k, it = int(sys.argv[1]), int(sys.argv[2])
    r = T.kmeans(X, k, it, 11)
    np.save(sys.argv[4], np.concatenate([r.assignments.astype(np.float64), r.centroids.ravel().astype(np.float64)]))
    sys.exit(0)
for dup in ("nodup", "dup"):
    for k in (50, 64, 100):
        for it in (1, 2):
            res = {}
            for tc in ("0", "1"):
                f = f"/tmp/d{tc}.npy"
                subprocess.run([sys.executable, __file__, str(k), str(it), dup, f], check=True,
                               env=dict(os.environ, TACO_TC_ASSIGN=tc))
                res[tc] = np.load(f)
            a0, a1 = res["0"][:20000], res["1"][:20000]
            bad = np.flatnonzero(a0 != a1)
            print(dup, k, it, "label diffs", bad.size, bad[:8], a0[bad[:4]], a1[bad[:4]],
                  "cent eq", np.array_equal(res["0"][20000:], res["1"][20000:]))
