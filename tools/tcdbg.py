"""k_assign_tc vs k_assign (tools/, not a test)."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
if len(sys.argv) > 1:   # child: one k-means, labels to stdout file
    import paper_2603_24919_b200 as T
    X = np.random.default_rng(1).normal(size=(5000, 8)).astype(np.float32)
    r = T.kmeans(X, 64, int(sys.argv[2]), 1)
    np.save(sys.argv[1], np.concatenate([r.assignments.astype(np.float64), r.centroids.ravel().astype(np.float64),
                                         np.array(r.inertia_history)]))
    sys.exit(0)
from oracle import taco_oracle as O  # noqa: E402
X = np.random.default_rng(1).normal(size=(5000, 8)).astype(np.float32)
for it in (1, 2, 3):
    res = {}
    for tc in ("0", "1"):
        env = dict(os.environ, TACO_TC_ASSIGN=tc)
        subprocess.run([sys.executable, __file__, f"/tmp/tc{tc}.npy", str(it)], env=env, check=True)
        res[tc] = np.load(f"/tmp/tc{tc}.npy")
    o = O.kmeans(X, 64, it, 1)
    a0, a1 = res["0"][:5000], res["1"][:5000]
    c0, c1 = res["0"][5000:5000 + 512], res["1"][5000:5000 + 512]
    print(it, "labels tc0==tc1", np.array_equal(a0, a1), int((a0 != a1).sum()), "tc0==oracle",
          np.array_equal(a0, o.labels), "tc1==oracle", np.array_equal(a1, o.labels),
          "cent eq", np.array_equal(c0, c1), "hist", res["0"][5512:], res["1"][5512:])
    d = np.abs(c0 - c1).reshape(64, 8).max(axis=1)
    print("  clusters differing:", np.flatnonzero(d > 0)[:20], "max diff", d.max(),
          "sizes", np.bincount(a0.astype(int), minlength=64)[np.flatnonzero(d > 0)[:10]])
