"""CPU oracle for the TaCo build + batched k-ANN hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module.  It is imported by ``tests/`` (as the parity checker), by
``__graft_entry__.smoke()`` (to check one small GPU run) and by
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg (as the timed
CPU baseline, kind "port").

It is a numpy restatement of the reference package's algorithm
(``/root/reference/pkg/src/taco``, which is Python/numpy; every function
cites the file:line it follows).  Because the reference's arithmetic *is*
numpy, the restatement keeps the exact numpy primitive for every floating
point reduction whose summation order decides bits:

* ``np.einsum('ij,ij->i')``  -- SSE2 two-lane order (measured, see
  DESIGN.md "numerics"), used for squared norms / distances;
* ``X @ C.T`` with >= 2 columns -- OpenBLAS dgemm, a sequential FMA chain;
  with 1 column it is dgemv (order not restated: see DESIGN.md);
* ``ndarray.sum()`` -- numpy pairwise summation;
* ``mean(axis=0)``, ``cumsum``, ``np.add.at`` -- sequential.

Pinned against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``; checked by ``tests/test_oracle.py``).
"""

from __future__ import annotations

import hashlib
import heapq
import math
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_SEED_MASK = (1 << 63) - 1
ZERO_EIG_REL = 1e-12          # spectral.py:25
JACOBI_TOL = 1e-9             # spectral.py:28
JACOBI_SWEEPS = 100           # spectral.py:29


class OracleError(Exception):
    """Raised where the reference raises one of its TacoError subclasses;
    ``kind`` names the reference class (errors.py:4-45)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# ----------------------------------------------------------------- seeding
def derive_seed(root: int, *path: int) -> int:
    """seeding.py:16-20 -- SeedSequence fold of (root, *path) to one u64."""
    words = [int(root) & _SEED_MASK]
    words += [int(p) & _SEED_MASK for p in path]
    return int(np.random.SeedSequence(words).generate_state(1, np.uint64)[0])


# ---------------------------------------------------------------- spectral
def fit_covariance(X):
    """spectral.py:94-111: fp64 mean (sequential over rows) and
    (X-mu)^T (X-mu)/(n-1), symmetrised."""
    X = np.asarray(X)
    n = X.shape[0]
    if n < 2:
        raise OracleError("InsufficientDataError", f"covariance needs >= 2 rows, got {n}")
    ok = np.isfinite(X).all(axis=1)
    if not ok.all():
        raise OracleError("NumericError", f"non-finite value in row {int(np.argmin(ok))}")
    X64 = X.astype(np.float64)
    mu = X64.mean(axis=0)
    C = X64 - mu
    gram = C.T @ C / (n - 1)
    return mu, (gram + gram.T) / 2.0


def circle_schedule(d: int):
    """spectral.py:114-131 -- round-robin (circle method) pairing."""
    m = d + (d & 1)
    ring = list(range(m))
    out = []
    for _ in range(m - 1):
        rnd = []
        for i in range(m // 2):
            a, b = ring[i], ring[m - 1 - i]
            if a < d and b < d:
                rnd.append((a, b) if a < b else (b, a))
        out.append(rnd)
        ring = [ring[0], ring[-1]] + ring[1:-1]
    return out


def _offdiag_max(A):
    """spectral.py:134-136."""
    if A.size == 0:
        return 0.0
    return float(np.abs(A - np.diag(np.diag(A))).max())


def jacobi(matrix, tol_rel=JACOBI_TOL, max_sweeps=JACOBI_SWEEPS):
    """spectral.py:139-195 -- cyclic Jacobi, one batched rotation per round.

    Returns (eigenvalues unsorted, V, sweeps_run)."""
    A = np.array(matrix, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise OracleError("ParameterError", f"expected a square matrix, got shape {A.shape}")
    d = A.shape[0]
    big = max(1.0, float(np.abs(A).max()) if A.size else 1.0)
    if A.size and float(np.abs(A - A.T).max()) > 1e-6 * big:
        raise OracleError("ParameterError", "matrix is not symmetric")
    A = (A + A.T) / 2.0
    V = np.eye(d)
    if d <= 1:
        return np.diag(A).copy(), V, 0
    tol = tol_rel * float(np.linalg.norm(A, "fro"))
    rounds = [(np.array([p for p, _ in r], dtype=np.intp),
               np.array([q for _, q in r], dtype=np.intp)) for r in circle_schedule(d)]
    sweeps = 0
    converged = False
    for _ in range(max_sweeps):
        if _offdiag_max(A) <= tol:
            converged = True
            break
        sweeps += 1
        for P0, Q0 in rounds:
            a_pq = A[P0, Q0]
            keep = a_pq != 0.0
            if not keep.any():
                continue
            P, Q, a_pq = P0[keep], Q0[keep], a_pq[keep]
            tau = (A[Q, Q] - A[P, P]) / (2.0 * a_pq)
            sgn = np.where(tau < 0.0, -1.0, 1.0)
            t = sgn / (np.abs(tau) + np.sqrt(1.0 + tau * tau))
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = t * c
            rp, rq = A[P, :].copy(), A[Q, :].copy()
            A[P, :] = c[:, None] * rp - s[:, None] * rq
            A[Q, :] = s[:, None] * rp + c[:, None] * rq
            cp_, cq_ = A[:, P].copy(), A[:, Q].copy()
            A[:, P] = cp_ * c - cq_ * s
            A[:, Q] = cp_ * s + cq_ * c
            A[P, Q] = 0.0
            A[Q, P] = 0.0
            vp, vq = V[:, P].copy(), V[:, Q].copy()
            V[:, P] = vp * c - vq * s
            V[:, Q] = vp * s + vq * c
    if not converged:
        resid = _offdiag_max(A)
        if resid > tol:
            raise OracleError("ConvergenceError",
                              f"eigensolver hit the {max_sweeps}-sweep cap with "
                              f"off-diagonal residual {resid:.3e} above tolerance {tol:.3e}")
    return np.diag(A).copy(), V, sweeps


def eigensystem(cov):
    """spectral.py:198-231 -- sort desc (stable), sign-fix, clamp, rescale."""
    lam, V, _ = jacobi(cov)
    order = np.argsort(-lam, kind="stable")
    lam, V = lam[order], V[:, order]
    d = lam.shape[0]
    piv = np.argmax(np.abs(V), axis=0)
    sg = np.sign(V[piv, np.arange(d)])
    sg[sg == 0] = 1.0
    V = V * sg
    raw = np.maximum(lam, 0.0)
    top = float(raw[0]) if raw.size else 0.0
    if top <= 0.0:
        scaled = np.ones_like(raw)
    else:
        fl = np.maximum(raw, ZERO_EIG_REL * top)
        scaled = fl / float(fl.min())
    return scaled, V, raw


def allocate(scaled, n_sub, s):
    """spectral.py:234-265 -- greedy min-log-product bucket, ties -> lowest."""
    buckets = [[] for _ in range(n_sub)]
    logp = np.zeros(n_sub)
    for i in range(n_sub * s):
        best = None
        for j in range(n_sub):
            if len(buckets[j]) < s and (best is None or logp[j] < logp[best]):
                best = j
        buckets[best].append(i)
        logp[best] += math.log(scaled[i])
    return buckets, logp


def fit_transform(X, n_sub, s):
    """spectral.py:268-298 -> (mean f32[d], [blocks f32 d x s], warnings)."""
    X = np.asarray(X)
    mu, cov = fit_covariance(X)
    scaled, V, raw = eigensystem(cov)
    buckets, _ = allocate(scaled, n_sub, s)
    warns = []
    top = float(raw[0])
    rank = 0 if top <= 0.0 else int((raw >= ZERO_EIG_REL * top).sum())
    if rank < n_sub * s:
        warns.append(f"covariance rank {rank} is below the {n_sub * s} retained "
                     "directions; floored eigenvalues keep the allocation defined "
                     "but quality may degrade")
    blocks = [np.ascontiguousarray(V[:, b], dtype=np.float32) for b in buckets]
    return mu.astype(np.float32), blocks, warns


def transform(mean32, blocks, P):
    """spectral.py:301-316 -- f32((f64(P) - f64(mu32)) @ f64(B32))."""
    M = np.concatenate(blocks, axis=1).astype(np.float64)
    return ((np.asarray(P).astype(np.float64) - mean32.astype(np.float64)) @ M).astype(np.float32)


# ------------------------------------------------------------------ k-means
def _sqd(X64, xsq, C):
    """clustering.py:34-38 -- max((xsq - 2 X.C) + csq, 0)."""
    csq = np.einsum("ij,ij->i", C, C)
    out = xsq[:, None] - 2.0 * (X64 @ C.T) + csq[None, :]
    np.maximum(out, 0.0, out=out)
    return out


@dataclass
class KMeansResult:
    centroids: np.ndarray          # f32 (k, m)
    labels: np.ndarray             # i32 (n,)
    history: list
    seeds: list                    # k-means++ chosen point indices


def kmeans(X, k, iters, seed):
    """clustering.py:41-115.  k-means++ via the cumsum/searchsorted form of
    ``Generator.choice(n, p)`` (one ``random()`` per draw), then Lloyd."""
    X = np.asarray(X, dtype=np.float32)
    n, m = X.shape
    if n < k:
        raise OracleError("InsufficientDataError", f"{n} points cannot fill {k} clusters")
    X64 = X.astype(np.float64)
    xsq = np.einsum("ij,ij->i", X64, X64)
    rng = np.random.default_rng(seed)
    C = np.empty((k, m))
    first = int(rng.integers(n))
    picks = [first]
    C[0] = X64[first]
    best = _sqd(X64, xsq, C[:1])[:, 0]
    for i in range(1, k):
        tot = float(best.sum())
        if tot > 0.0:
            cdf = (best / tot).cumsum()
            cdf /= cdf[-1]
            idx = int(cdf.searchsorted(rng.random(), side="right"))
        else:
            idx = int(rng.integers(n))
        picks.append(idx)
        C[i] = X64[idx]
        np.minimum(best, _sqd(X64, xsq, C[i:i + 1])[:, 0], out=best)
    labels = None
    hist = []
    for _ in range(iters):
        dd = _sqd(X64, xsq, C)
        lab = np.argmin(dd, axis=1).astype(np.int32)
        pd = dd[np.arange(n), lab]
        hist.append(float(pd.sum()))
        if labels is not None and np.array_equal(lab, labels):
            labels = lab
            break
        labels = lab
        cnt = np.bincount(labels, minlength=k)
        acc = np.zeros((k, m))
        np.add.at(acc, labels, X64)
        full = cnt > 0
        C[full] = acc[full] / cnt[full, None]
        far = None
        for j in np.flatnonzero(~full):
            if far is None:
                far = pd.copy()
            p = int(np.argmax(far))
            C[j] = X64[p]
            labels[p] = np.int32(j)
            far[p] = -1.0
    return KMeansResult(C.astype(np.float32), labels, hist, picks)


# ------------------------------------------------------------------- index
@dataclass
class OracleIndex:
    n: int
    d: int
    n_sub: int
    s: int
    clusters: int
    iters: int
    seed: int
    mean: np.ndarray
    blocks: list
    cb1: list                      # per subspace f32 (K', split)
    cb2: list                      # per subspace f32 (K', s - split)
    cells: list                    # per subspace {(l1, l2): u32 ids ascending}
    labels: list = field(default_factory=list)   # per subspace (l1, l2) i32
    seeds: list = field(default_factory=list)
    warnings: list = field(default_factory=list)

    @property
    def kprime(self):
        return math.isqrt(self.clusters)

    @property
    def split(self):
        return (self.s + 1) // 2

    def sizes(self, j):
        """Dense (K', K') cell-size table of subspace j."""
        kp = self.kprime
        out = np.zeros((kp, kp), dtype=np.int64)
        for (a, b), ids in self.cells[j].items():
            out[a, b] = ids.size
        return out


def cells_from_labels(l1, l2):
    """imi.py:72-81 -- stable (l1, l2) sort, ids ascending in each cell."""
    a = np.asarray(l1).astype(np.int64)
    b = np.asarray(l2).astype(np.int64)
    n = a.size
    order = np.lexsort((np.arange(n), b, a))
    ka, kb = a[order], b[order]
    cut = np.flatnonzero((ka[1:] != ka[:-1]) | (kb[1:] != kb[:-1])) + 1
    lo = np.concatenate(([0], cut))
    hi = np.concatenate((cut, [n]))
    ids = order.astype(np.uint32)
    return {(int(ka[x]), int(kb[x])): ids[x:y].copy() for x, y in zip(lo, hi)}


def _kmeans_half_worker(job):
    """One k-means half in a spawned process (``build_index(workers=...)``):
    the transformed matrix is read from shared memory, BLAS runs one thread."""
    from multiprocessing import shared_memory

    name, shape, col0, col1, kp, iters, seed = job
    shm = shared_memory.SharedMemory(name=name)
    try:
        T = np.ndarray(shape, dtype=np.float32, buffer=shm.buf)
        r = kmeans(np.ascontiguousarray(T[:, col0:col1]), kp, iters, seed)
    finally:
        shm.close()
    return r


def _kmeans_halves(T, n_sub, s, kp, iters, seed, workers):
    """The 2*N_s k-means runs of imi.py:68-69, in order; with workers > 1 they
    run in parallel processes (independent problems: identical results)."""
    split = (s + 1) // 2
    jobs = []
    for j in range(n_sub):
        sj = derive_seed(seed, j)
        jobs.append((j * s, j * s + split, kp, iters, derive_seed(sj, 0)))
        jobs.append((j * s + split, (j + 1) * s, kp, iters, derive_seed(sj, 1)))
    if workers <= 1:
        return [kmeans(T[:, a:b], k, it, sd) for a, b, k, it, sd in jobs]
    import multiprocessing as mp
    import os
    from multiprocessing import shared_memory

    T = np.ascontiguousarray(T, dtype=np.float32)
    shm = shared_memory.SharedMemory(create=True, size=max(T.nbytes, 1))
    saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS")}
    try:
        np.ndarray(T.shape, np.float32, buffer=shm.buf)[:] = T
        os.environ["OPENBLAS_NUM_THREADS"] = "1"   # one BLAS thread per process (inherited at spawn)
        os.environ["OMP_NUM_THREADS"] = "1"
        with mp.get_context("spawn").Pool(min(workers, len(jobs))) as pool:
            return pool.map(_kmeans_half_worker, [(shm.name, T.shape) + jb for jb in jobs], chunksize=1)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        shm.close()
        shm.unlink()


def build_index(X, n_sub, s, clusters, iters=20, seed=0, T=None, model=None, workers=1, timings=None):
    """engine.py:122-174 + imi.py:49-85.  ``model``/``T`` let stage-wise
    parity tests inject a fixed transform; ``workers`` > 1 runs the 2*N_s
    independent k-means halves in parallel processes (the CPU baseline);
    ``timings`` (a dict) receives transform / k-means seconds like
    engine.py:156-166."""
    import time as _time

    t0 = _time.perf_counter()
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, d = X.shape
    kp = math.isqrt(clusters)
    if model is None:
        mean, blocks, warns = fit_transform(X, n_sub, s)
    else:
        mean, blocks = model
        warns = []
    if T is None:
        T = transform(mean, blocks, X)
    t1 = _time.perf_counter()
    split = (s + 1) // 2
    idx = OracleIndex(n, d, n_sub, s, clusters, iters, seed, mean, list(blocks),
                      [], [], [], warnings=warns)
    halves = _kmeans_halves(T, n_sub, s, kp, iters, seed, workers)
    for j in range(n_sub):
        r1, r2 = halves[2 * j], halves[2 * j + 1]
        idx.cb1.append(r1.centroids)
        idx.cb2.append(r2.centroids)
        idx.labels.append((r1.labels, r2.labels))
        idx.seeds.append((r1.seeds, r2.seeds))
        idx.cells.append(cells_from_labels(r1.labels, r2.labels))
    if timings is not None:
        timings["transform_seconds"] = t1 - t0
        timings["kmeans_seconds"] = _time.perf_counter() - t1
        timings["build_seconds"] = _time.perf_counter() - t0
    return idx


# ------------------------------------------------------------------- query
def centroid_order(c1, c2, q_sub, split):
    """imi.py:88-106 -- fp64 direct-form distances, stable argsort."""
    q = np.asarray(q_sub, dtype=np.float64).ravel()
    e1 = c1.astype(np.float64) - q[:split]
    e2 = c2.astype(np.float64) - q[split:]
    d1 = np.einsum("ij,ij->i", e1, e1)
    d2 = np.einsum("ij,ij->i", e2, e2)
    return d1, np.argsort(d1, kind="stable"), d2, np.argsort(d2, kind="stable")


def retrieval_target(alpha, n):
    """imi.py:109-112."""
    return min(n, math.ceil(alpha * n))


def traverse(alpha, n, kprime, d1, i1, d2, i2, size_of):
    """imi.py:130-166 -- min-heap multi-sequence traversal.

    ``size_of(l1, l2)`` returns the cell size (0 for a missing cell).
    Returns (pops [(key, l1, l2)], retrieved)."""
    target = retrieval_target(alpha, n)
    pops = []
    got = 0
    frontier = [(float(d1[i1[0]] + d2[i2[0]]), 0, 0)]
    while frontier:
        key, r, c = heapq.heappop(frontier)
        a, b = int(i1[r]), int(i2[c])
        pops.append((key, a, b))
        got += size_of(a, b)
        if got >= target:
            break
        if c == 0 and r + 1 < kprime:
            heapq.heappush(frontier, (float(d1[i1[r + 1]] + d2[i2[0]]), r + 1, 0))
        if c + 1 < kprime:
            heapq.heappush(frontier, (float(d1[i1[r]] + d2[i2[c + 1]]), r, c + 1))
    return pops, got


def query_scores(index: OracleIndex, q, alpha, trace=None):
    """engine.py:188-220 -- uint8 collision counts over all n points."""
    q = np.asarray(q, dtype=np.float32).ravel()
    sc = np.zeros(index.n, dtype=np.uint8)
    qt = transform(index.mean, index.blocks, q[None, :])[0]
    s, kp, sp = index.s, index.kprime, index.split
    for j in range(index.n_sub):
        cells = index.cells[j]
        d1, i1, d2, i2 = centroid_order(index.cb1[j], index.cb2[j], qt[j * s:(j + 1) * s], sp)
        pops, got = traverse(alpha, index.n, kp, d1, i1, d2, i2,
                             lambda a, b: cells[(a, b)].size if (a, b) in cells else 0)
        if trace is not None:
            trace.append((pops, got))
        hit = [cells[(a, b)] for _, a, b in pops if (a, b) in cells]
        if hit:
            sc[np.concatenate(hit)] += 1
    return sc


def select(scores, beta, n_sub, n=None):
    """engine.py:223-253 -- Alg. 5 threshold scan (break level included)."""
    scores = np.asarray(scores)
    if n is None:
        n = scores.shape[0]
    h = np.bincount(scores, minlength=n_sub + 1)
    budget = beta * n
    level = n_sub
    taken = 0
    for j in range(n_sub, -1, -1):
        taken += int(h[j])
        if h[j] <= budget - taken:
            level -= 1
        else:
            break
    level = max(level, 0)
    ids = np.flatnonzero(scores >= level)
    return ids, taken, level, h


def rerank(X, q, ids, k):
    """engine.py:256-279 -- fp64 exact distances, order by (d2, id)."""
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size == 0:
        return np.empty(0, np.int32), np.empty(0, np.float32), np.empty(0)
    qd = np.asarray(q, dtype=np.float64).ravel()
    e = np.asarray(X)[ids].astype(np.float64) - qd
    d2 = np.einsum("ij,ij->i", e, e)
    np.maximum(d2, 0.0, out=d2)
    o = np.lexsort((ids, d2))[:min(k, ids.size)]
    return ids[o].astype(np.int32), np.sqrt(d2[o]).astype(np.float32), d2[o]


def knn(index, X, q, alpha, beta, k):
    """engine.py:282-287 -> (ids, dists, candidate_num, last_collision)."""
    sc = query_scores(index, q, alpha)
    ids, num, level, _ = select(sc, beta, index.n_sub, index.n)
    rid, rd, _ = rerank(X, q, ids, k)
    return rid, rd, num, level


def knn_batch(index, X, Q, alpha, beta, k, threads=1):
    """Batched driver with the padding of cli.py:155-164; a thread pool per
    query like bench._query_pass (bench.py:120-129)."""
    Q = np.asarray(Q, dtype=np.float32)
    nq = Q.shape[0]
    out_i = np.full((nq, k), -1, np.int32)
    out_d = np.full((nq, k), np.inf, np.float32)
    num = np.zeros(nq, np.int64)
    lvl = np.zeros(nq, np.int32)

    def one(r):
        a, b, c, e = knn(index, X, Q[r], alpha, beta, k)
        out_i[r, :a.size] = a
        out_d[r, :b.size] = b
        num[r] = c
        lvl[r] = e

    if threads <= 1:
        for r in range(nq):
            one(r)
    else:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(one, range(nq)))
    return out_i, out_d, num, lvl


def sc_linear_scores(T, qt, n_sub, s, alpha):
    """engine.py:290-321 -- exact collisions: per subspace, the ceil(alpha n)
    nearest rows by (fp64 einsum d2, id) collide."""
    T = np.asarray(T)
    qt = np.asarray(qt, dtype=np.float64).ravel()
    n = T.shape[0]
    collide = min(n, math.ceil(alpha * n))
    scores = np.zeros(n, np.uint8)
    ids = np.arange(n)
    for j in range(n_sub):
        diff = T[:, j * s:(j + 1) * s].astype(np.float64) - qt[j * s:(j + 1) * s]
        dd = np.einsum("ij,ij->i", diff, diff)
        scores[np.lexsort((ids, dd))[:collide]] += 1
    return scores


def ground_truth(base, queries, k):
    """dataio.py:142-172 -- exact k-NN, fp64 expansion form, ties by id."""
    X = np.asarray(base).astype(np.float64)
    Q = np.asarray(queries).astype(np.float64)
    xsq = np.einsum("ij,ij->i", X, X)
    all_ids = np.arange(X.shape[0])
    ids = np.empty((Q.shape[0], k), np.int32)
    ds = np.empty((Q.shape[0], k), np.float32)
    for a in range(0, Q.shape[0], 256):
        ch = Q[a:a + 256]
        qsq = np.einsum("ij,ij->i", ch, ch)
        dd = xsq[None, :] - 2.0 * (ch @ X.T) + qsq[:, None]
        np.maximum(dd, 0.0, out=dd)
        for r in range(ch.shape[0]):
            o = np.lexsort((all_ids, dd[r]))[:k]
            ids[a + r] = o
            ds[a + r] = np.sqrt(dd[r, o])
    return ids, ds


# ------------------------------------------------------------- persistence
_HDR = struct.Struct("<QIIIIIq")


def serialize(index: OracleIndex) -> bytes:
    """engine.py:345-384 -- index file format v1 with blake2b-64 trailer."""
    buf = bytearray(b"TACO")
    buf += struct.pack("<H", 1)
    buf += _HDR.pack(index.n, index.d, index.n_sub, index.s, index.clusters,
                     index.iters, index.seed)
    buf += index.mean.astype("<f4").tobytes()
    for b in index.blocks:
        buf += b.astype("<f4").tobytes(order="F")
    for j in range(index.n_sub):
        buf += index.cb1[j].astype("<f4").tobytes()
        buf += index.cb2[j].astype("<f4").tobytes()
        keys = sorted(index.cells[j])
        buf += struct.pack("<II", index.kprime, len(keys))
        for a, b in keys:
            ids = index.cells[j][(a, b)]
            buf += struct.pack("<HHI", a, b, ids.size)
            buf += ids.astype("<u4").tobytes()
    return bytes(buf) + hashlib.blake2b(bytes(buf), digest_size=8).digest()


def deserialize(blob: bytes) -> OracleIndex:
    """engine.py:425-494 (checks trimmed to what parity needs)."""
    if blob[:4] != b"TACO":
        raise OracleError("FormatError", "bad magic")
    body, tag = blob[:-8], blob[-8:]
    if hashlib.blake2b(body, digest_size=8).digest() != tag:
        raise OracleError("CorruptionError", "checksum mismatch")
    off = 6
    n, d, ns, s, K, it, seed = _HDR.unpack_from(body, off)
    off += _HDR.size

    def f32(cnt):
        nonlocal off
        a = np.frombuffer(body, "<f4", cnt, off).astype(np.float32)
        off += 4 * cnt
        return a

    mean = f32(d)
    blocks = [f32(d * s).reshape((d, s), order="F").copy() for _ in range(ns)]
    kp = math.isqrt(K)
    sp = (s + 1) // 2
    idx = OracleIndex(n, d, ns, s, K, it, seed, mean, blocks, [], [], [])
    for _ in range(ns):
        idx.cb1.append(f32(kp * sp).reshape(kp, sp))
        idx.cb2.append(f32(kp * (s - sp)).reshape(kp, s - sp))
        _, nc = struct.unpack_from("<II", body, off)
        off += 8
        cells = {}
        for _ in range(nc):
            a, b, sz = struct.unpack_from("<HHI", body, off)
            off += 8
            cells[(a, b)] = np.frombuffer(body, "<u4", sz, off).astype(np.uint32)
            off += 4 * sz
        idx.cells.append(cells)
    return idx
