"""CPU stand-in for CudaShardBackend (TEST INFRASTRUCTURE): the per-rank
stages computed with the oracle so the sharded orchestration in
paper_2603_24919_b200.distributed can be exercised with gloo on CPU."""

import numpy as np
import torch

from oracle import taco_oracle as O


class OracleShardBackend:
    def __init__(self, oidx, X_shard, id_base, n_global, tile=7):
        self.o = oidx
        self.X = np.asarray(X_shard, np.float32)
        self.lo = id_base
        self.n = n_global
        self.tile = tile
        self.scores = None

    def tile_size(self):
        return self.tile

    # ---- split traversal (distributed._split_count); small cap so the
    # overflow -> re-run path is exercised too
    pop_cap = 6

    def front(self, Qt, alpha, lo, hi, rows):
        o = self.o
        Q = Qt.numpy()
        self.Q = Q
        if getattr(self, "_rows", None) != (rows, self.pop_cap):
            self._rows = (rows, self.pop_cap)
            self.pops = np.zeros((rows, o.n_sub, self.pop_cap), np.uint16)
            self.npop = np.zeros((rows, o.n_sub), np.int32)
            self.ret = np.zeros((rows, o.n_sub), np.int64)
        need = 0
        s, kp = o.s, o.kprime
        for r in range(lo, hi):
            qt = O.transform(o.mean, o.blocks, Q[r][None, :])[0]
            for j in range(o.n_sub):
                cells = o.cells[j]
                d1, i1, d2, i2 = O.centroid_order(o.cb1[j], o.cb2[j], qt[j * s:(j + 1) * s], o.split)
                pops, got = O.traverse(alpha, o.n, kp, d1, i1, d2, i2,
                                       lambda a, b: cells[(a, b)].size if (a, b) in cells else 0)
                self.npop[r, j] = len(pops)
                self.ret[r, j] = got
                if len(pops) > self.pop_cap:
                    need = max(need, len(pops))
                for t, (_, a, b) in enumerate(pops[:self.pop_cap]):
                    self.pops[r, j, t] = a * kp + b
        return need

    def front_async(self, Qt, alpha, lo, hi, rows):
        """distributed._split_count's protocol: the slice's longest walk as a
        tensor (the caller checks it against the cap once per batch)."""
        self.front(Qt, alpha, lo, hi, rows)
        return torch.tensor([int(self.npop[lo:hi].max()) if hi > lo else 0], dtype=torch.int64)

    def raise_pop_cap(self, need):
        self.pop_cap = min(self.o.kprime ** 2, need + 1)

    def pop_views(self, rows):
        return [torch.from_numpy(a.reshape(rows, -1).view(np.uint8)) for a in (self.pops, self.npop, self.ret)]

    def count_popped(self, nq):
        o = self.o
        hi = self.lo + self.X.shape[0]
        self.scores = []
        for r in range(nq):
            sc = np.zeros(o.n, np.uint8)
            for j in range(o.n_sub):
                for cell in self.pops[r, j, :self.npop[r, j]]:
                    key = divmod(int(cell), o.kprime)
                    if key in o.cells[j]:
                        sc[o.cells[j][key]] += 1
            self.scores.append(sc[self.lo:hi])
        h = [np.bincount(s, minlength=o.n_sub + 1) for s in self.scores]
        return torch.tensor(np.array(h, np.int64))

    def count(self, Qt, alpha):
        Q = Qt.numpy()
        hi = self.lo + self.X.shape[0]
        self.scores = [O.query_scores(self.o, q, alpha)[self.lo:hi] for q in Q]
        self.Q = Q
        h = [np.bincount(s, minlength=self.o.n_sub + 1) for s in self.scores]
        return torch.tensor(np.array(h, np.int64))

    def finish(self, nq, ghist, beta, k):
        g = ghist.numpy()
        ns = self.o.n_sub
        d2 = np.full((nq, k), np.inf)
        ids = np.full((nq, k), -1, np.int64)
        num = np.zeros(nq, np.int64)
        lvl = np.zeros(nq, np.int32)
        budget = beta * self.n
        for r in range(nq):
            L, cand = ns, 0
            for j in range(ns, -1, -1):       # engine.py:243-249 on the global histogram
                cand += int(g[r, j])
                if g[r, j] <= budget - cand:
                    L -= 1
                else:
                    break
            L = max(L, 0)
            num[r], lvl[r] = cand, L
            loc = np.flatnonzero(self.scores[r] >= L)
            if loc.size:
                e = self.X[loc].astype(np.float64) - self.Q[r].astype(np.float64)
                dd = np.einsum("ij,ij->i", e, e)
                gid = loc + self.lo
                o = np.lexsort((gid, dd))[:k]
                d2[r, :o.size] = dd[o]
                ids[r, :o.size] = gid[o]
        return torch.tensor(d2), torch.tensor(ids), torch.tensor(num), torch.tensor(lvl)

    def merge(self, d2_all, ids_all, k):
        d2a, ida = d2_all.numpy(), ids_all.numpy()
        R, nq = d2a.shape[0], d2a.shape[1]
        out_i = np.full((nq, k), -1, np.int32)
        out_d = np.full((nq, k), np.inf, np.float32)
        for q in range(nq):
            items = [(d2a[r, q, t], ida[r, q, t]) for r in range(R) for t in range(k) if ida[r, q, t] >= 0]
            items.sort()
            for t, (dv, iv) in enumerate(items[:k]):
                out_i[q, t] = iv
                out_d[q, t] = np.float32(np.sqrt(dv))
        return torch.tensor(out_i), torch.tensor(out_d)


class OracleShardBuilder:
    """CPU stand-in for distributed_build.CudaShardBuilder (TEST
    INFRASTRUCTURE): each build stage of one rank restated with numpy /
    the oracle, so the collective orchestration of
    paper_2603_24919_b200.distributed_build runs with gloo on CPU.  The
    covariance follows the same chains as the device (sequential column sums;
    Gram partials over fixed row blocks added in order)."""

    comm_device = "cpu"

    def __init__(self, X_local, id_base, n_global, params, block=256):
        self.X = np.ascontiguousarray(X_local, np.float32)
        self.n_local, self.d = self.X.shape
        self.id_base, self.n_global, self.params, self.block = id_base, n_global, params, block

    def gram_block_rows(self):
        return self.block

    def colsum(self, carry):
        X64 = self.X.astype(np.float64)
        bad = np.flatnonzero(~np.isfinite(self.X).all(axis=1))
        acc = X64[0].copy() if carry is None else np.array(carry, np.float64)
        for row in (X64[1:] if carry is None else X64):
            acc += row
        return acc, int(bad[0]) if bad.size else -1

    def gram(self, mean, block, carry):
        acc = np.zeros((self.d, self.d)) if carry is None else np.array(carry, np.float64)
        for b0 in range(0, self.n_local, block):
            xc = self.X[b0:b0 + block].astype(np.float64) - mean
            acc = acc + xc.T @ xc
        return acc

    def transform(self, model):
        T = O.transform(np.asarray(model.mean, np.float32), list(model.blocks), self.X)
        return torch.from_numpy(np.ascontiguousarray(T.T))

    def kmeans(self, subspaces, T_cols, n_global, params):
        p = params
        s, sp = p.subspace_dim, (p.subspace_dim + 1) // 2
        Tc = T_cols.numpy()
        labs, cbs, hist = [], [], []
        for jj, j in enumerate(subspaces):
            blk = np.ascontiguousarray(Tc[jj * s:(jj + 1) * s].T)
            sj = O.derive_seed(p.seed, j)
            r1 = O.kmeans(blk[:, :sp], p.codebook_size, p.kmeans_iters, O.derive_seed(sj, 0))
            r2 = O.kmeans(blk[:, sp:], p.codebook_size, p.kmeans_iters, O.derive_seed(sj, 1))
            labs += [r1.labels, r2.labels]
            cbs.append((r1.centroids, r2.centroids))
            hist.append((tuple(r1.history), tuple(r2.history)))
        return {"labels": torch.from_numpy(np.array(labs, np.int32)), "codebooks": cbs, "histories": hist}

    def finish(self, codebooks, labels_loc):
        p = self.params
        L = labels_loc.numpy()
        kp = p.codebook_size
        self.cells = [O.cells_from_labels(L[2 * j], L[2 * j + 1]) for j in range(p.n_subspaces)]
        sizes = np.zeros((p.n_subspaces, p.clusters), np.int64)
        for j, cells in enumerate(self.cells):
            for (a, b), ids in cells.items():
                sizes[j, a * kp + b] = ids.size
        return sizes

    def set_global_sizes(self, sizes):
        self.global_sizes = np.asarray(sizes)

    def local_cells(self):
        kp = self.params.codebook_size
        out = []
        for cells in self.cells:
            off = np.zeros(kp * kp + 1, np.int64)
            parts = []
            for c in range(kp * kp):
                ids = cells.get((c // kp, c % kp))
                off[c + 1] = off[c] + (0 if ids is None else ids.size)
                if ids is not None:
                    parts.append(ids)
            out.append((off, np.concatenate(parts) if parts else np.empty(0, np.uint32)))
        return out
