"""How often is a Lloyd centroid sum order-free?  For each (half, cluster,
column): u = smallest f32 ulp among the cluster's nonzero values, S = sum of
|x|; if S < 2^53 u every fp64 partial sum is exact, so a parallel sum equals
np.add.at's sequential one (Lloyd update)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T
from paper_2603_24919_b200.workloads import make_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
X, Q, m = make_config(cfg, nq=4)
idx = T.build_index(X, T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], 0), keep_transformed=True)
Tm = idx.transformed
s = m["s"]
tot = ok = 0
worst = []
for j, sub in enumerate(idx.subspaces):
    for h, cb in enumerate((sub.codebook1, sub.codebook2)):
        lo = j * s + (0 if h == 0 else (s + 1) // 2)
        hi = lo + cb.dim
        lab = np.asarray(cb.assignments)
        for c in range(m["kprime"]):
            pts = Tm[lab == c, lo:hi].astype(np.float64)
            if pts.shape[0] == 0:
                continue
            a = np.abs(pts)
            for t in range(pts.shape[1]):
                col = a[:, t]
                nz = col[col > 0]
                tot += 1
                if nz.size == 0:
                    ok += 1
                    continue
                e = np.frexp(nz.astype(np.float32))[1]          # value in [2^(e-1), 2^e)
                u = np.ldexp(1.0, int(e.min()) - 24)             # f32 ulp of the smallest value
                S = col.sum()
                good = S * (1 + 1e-9) < np.ldexp(u, 53)
                ok += good
                worst.append(np.log2(S / u))
print(f"cfg {cfg}: {ok}/{tot} (cluster, column) sums certified order-free; "
      f"log2(S/u) median {np.median(worst):.1f}, p90 {np.percentile(worst, 90):.1f}, max {max(worst):.1f} (need < 53)")
