"""Device vs host Jacobi sweeps: time and bit-identity (tools/, not a test)."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from tests.test_gpu_build import _jac  # noqa: E402

rng = np.random.default_rng(1)
for d in [int(x) for x in (sys.argv[1:] or (128, 257, 300, 600, 960))]:
    X = rng.normal(size=(4 * d, d)) @ rng.normal(size=(d, d))
    A = X.T @ X
    A = (A + A.T) / 2
    _jac(A, True)
    t = time.perf_counter()
    g = _jac(A, True)
    tg = time.perf_counter() - t
    g2 = _jac(A, True)
    t = time.perf_counter()
    h = _jac(A, False)
    th = time.perf_counter() - t
    eq = np.array_equal(g[1], h[1]) and np.array_equal(g[2], h[2])
    rep = np.array_equal(g[1], g2[1]) and np.array_equal(g[2], g2[2])
    print(f"d={d} device {tg * 1e3:.1f} ms host {th * 1e3:.1f} ms sweeps {g[3]}/{h[3]} "
          f"equal {eq} repeatable {rep} maxdiffV {np.abs(g[2] - h[2]).max():.3g}")
