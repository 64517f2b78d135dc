"""How much do the candidate sets of a batch's queries overlap?  (rerank L2-reuse study)

Collects the candidate sets of the first NQ queries of config 2 through the
single-query taps, then reports the Jaccard similarity of neighbours in several
orders and the best achievable (max over all other queries).
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

NQ = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
X, Q, meta = make_config(2)
idx = T.build_index(X, T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"]))
n = X.shape[0]
t0 = time.time()
sets = []
for i in range(NQ):
    sc = T.count_collisions(idx, Q[i], meta["alpha"])
    cs = T.select_candidates(sc, meta["beta"], meta["n_sub"])
    sets.append(cs.ids)
print("collected", NQ, "sets in", round(time.time() - t0, 1), "s; mean size", np.mean([s.size for s in sets]))
M = torch.zeros((NQ, n), dtype=torch.bfloat16, device="cuda")
print("all-batch union/sum", round(torch.unique(torch.cat([torch.from_numpy(x).cuda() for x in sets])).numel() / sum(x.size for x in sets), 4))
for i, s in enumerate(sets):
    M[i, torch.from_numpy(s).cuda()] = 1
sizes = M.float().sum(1)
inter = (M @ M.T).float()
union = sizes[:, None] + sizes[None, :] - inter
J = inter / union
J.fill_diagonal_(0)
best = J.max(1).values
print("max-Jaccard over others: mean %.3f median %.3f p90 %.3f" % (best.mean(), best.median(), best.quantile(0.9)))
print("mean Jaccard of random pairs: %.4f" % J.mean())
# fraction of each query's candidates seen by ANY of the previous w queries in an order
def reuse(order, w):
    seen = torch.zeros(n, dtype=torch.int32, device="cuda")
    hits = 0
    tot = 0
    for pos, q in enumerate(order):
        s = torch.from_numpy(sets[q]).cuda()
        hits += int((seen[s] > 0).sum()) if pos else 0
        tot += s.numel()
        seen[s] += 1
        if pos >= w:
            seen[torch.from_numpy(sets[order[pos - w]]).cuda()] -= 1
    return hits / tot
keys = {
    "batch": list(range(NQ)),
    "minid": sorted(range(NQ), key=lambda q: (int(sets[q][0]) if sets[q].size else 1 << 40, q)),
}
# greedy nearest-neighbour chain (upper-bound-ish ordering)
Jc = J.clone()
cur, left, chain = 0, set(range(1, NQ)), [0]
Jn = Jc.cpu().numpy()
while left:
    l = np.fromiter(left, int)
    nxt = int(l[np.argmax(Jn[cur, l])])
    chain.append(nxt)
    left.remove(nxt)
    cur = nxt
keys["greedy"] = chain
def group_union(order, G):
    tot = uni = 0
    for g0 in range(0, NQ, G):
        qs = order[g0:g0 + G]
        u = torch.unique(torch.cat([torch.from_numpy(sets[q]).cuda() for q in qs]))
        uni += u.numel()
        tot += sum(sets[q].size for q in qs)
    return uni / tot
for name, order in keys.items():
    print(name, {w: round(reuse(order, w), 3) for w in (1, 4, 16)},
          "union/sum", {G: round(group_union(order, G), 3) for G in (16, 64, 256, 1024)})
