"""Cost of the exact k-means++ replay (tools/, not a test): kmeans on n points
with every draw forced through the replay vs the certified fast path."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200 import _native as nat  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
k = 9
X = np.random.default_rng(0).normal(size=(n, 6)).astype(np.float32)
T.kmeans(X, k, 1, 1)
for mode in (0, 1, 2, 0):
    nat.call("taco_debug_force_replay", mode)
    t = time.perf_counter()
    r = T.kmeans(X, k, 1, 1)
    dt = time.perf_counter() - t
    print(f"n={n} mode={mode} {dt * 1e3:.1f} ms ({dt * 1e3 / (k - 1):.2f} ms per draw)")
nat.call("taco_debug_force_replay", 0)
