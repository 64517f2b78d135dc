"""Inverted multi-index (reference imi.py) on the B200 path.

Cells live on the device as a chunk-major CSR (see csrc/index.cuh); the
``cells`` mapping of an index built or loaded here is a lazy view that
materialises the reference's ``{(l1, l2): uint32 ids}`` dict on first use.
"""

from __future__ import annotations

import math
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .clustering import KMeansModel, check_kmeans_args, draw_plan, forced_plan
from .errors import DimensionMismatchError, ParameterError
from .seeding import derive_seed

_EMPTY_IDS = np.empty(0, dtype=np.uint32)


class DeviceCells(Mapping):
    """Read-only ``{(l1, l2): ids}`` view of subspace ``j`` of a device index."""

    def __init__(self, dev, j: int, kprime: int):
        self._dev, self._j, self._kp = dev, j, kprime
        self._d = None

    def _load(self):
        if self._d is None:
            K2 = self._kp * self._kp
            offs = np.empty(K2 + 1, np.int64)
            ids = np.empty(self._dev.n, np.uint32)
            nat.call("taco_get_cells", self._dev.h, self._j, nat.ptr(offs), nat.ptr(ids))
            nz = np.flatnonzero(np.diff(offs))
            self._d = {(int(c // self._kp), int(c % self._kp)): ids[offs[c]:offs[c + 1]]
                       for c in nz}
        return self._d

    def __getitem__(self, key):
        return self._load()[key]

    def __iter__(self):
        return iter(self._load())

    def __len__(self):
        return len(self._load())


@dataclass(frozen=True)
class InvertedMultiIndex:
    codebook1: KMeansModel
    codebook2: KMeansModel
    cells: Mapping                 # (label1, label2) -> ids, ascending
    codebook_size: int             # clusters per codebook (sqrt of K)
    split: int                     # first half covers dims [0, split)

    @property
    def subspace_dim(self) -> int:
        return self.codebook1.dim + self.codebook2.dim

    @property
    def n_points(self) -> int:
        return sum(ids.size for ids in self.cells.values())


@dataclass(frozen=True)
class ActivationResult:
    retrieved_clusters: tuple
    retrieved_num: int
    pop_trace: tuple               # (distance sum, label1, label2)


def build_subspace_index(subspace_data, n_cells: int, kmeans_iters: int = 20,
                         seed: int = 0) -> InvertedMultiIndex:
    """Two GPU k-means runs over the halves + the device CSR (imi.py:49-85)."""
    X = np.ascontiguousarray(np.asarray(subspace_data, dtype=np.float32))
    if X.ndim != 2:
        raise ParameterError(f"expected a 2-D matrix, got shape {X.shape}")
    n, s = X.shape
    if s < 2:
        raise ParameterError(f"subspace dimension {s} cannot be split into two parts")
    kprime = math.isqrt(int(n_cells)) if n_cells >= 1 else 0
    if kprime < 1 or kprime * kprime != n_cells:
        raise ParameterError(f"cluster count {n_cells} is not a perfect square")
    if kprime > 0xFFFF:
        raise ParameterError(f"per-codebook cluster count {kprime} exceeds 65535")
    split = (s + 1) // 2
    check_kmeans_args(X[:, :split], kprime, kmeans_iters)
    dev = nat.DeviceIndex(n, s, 1, s, n_cells, kmeans_iters)
    nat.call("taco_index_set_transformed", dev.h, nat.ptr(X))
    models = run_kmeans_all(dev, n, 1, s, kprime, kmeans_iters, lambda j, h: derive_seed(seed, h))
    nat.call("taco_build_cells", dev.h)
    return InvertedMultiIndex(codebook1=models[0][0], codebook2=models[0][1],
                              cells=DeviceCells(dev, 0, kprime), codebook_size=kprime, split=split)


def run_kmeans_all(dev, n, n_sub, s, kprime, iters, seed_of):
    """All 2*N_s halves on concurrent streams; returns [(cb1, cb2)] per subspace."""
    H = 2 * n_sub
    firsts = np.empty(H, np.int64)
    unis = np.zeros((H, max(kprime - 1, 0)))
    seeds = []
    for hh in range(H):
        sd = seed_of(hh // 2, hh % 2)
        seeds.append(sd)
        firsts[hh], unis[hh] = draw_plan(n, kprime, sd)
    deg = np.zeros(H, np.int32)
    unis = np.ascontiguousarray(unis)
    nat.call("taco_kmeans_all", dev.h, nat.ptr(firsts), nat.ptr(unis), None, nat.ptr(deg))
    if (deg < kprime).any():
        forced = np.full((H, max(kprime - 1, 0)), -1, np.int64)
        for hh in np.flatnonzero(deg < kprime):
            forced[hh] = forced_plan(n, kprime, seeds[hh], int(deg[hh]))
        nat.call("taco_kmeans_all", dev.h, nat.ptr(firsts), nat.ptr(unis), nat.ptr(forced),
                 nat.ptr(deg))
    m1 = (s + 1) // 2
    m2 = s - m1
    cb1 = np.empty((n_sub, kprime, m1), np.float32)
    cb2 = np.empty((n_sub, kprime, m2), np.float32)
    nat.call("taco_get_codebooks", dev.h, nat.ptr(cb1), nat.ptr(cb2))
    labels = {}

    def fetch_labels():   # one device -> host copy of all 2*N_s label vectors, on first use
        if not labels:
            lab1 = np.empty((n_sub, n), np.int32)
            lab2 = np.empty((n_sub, n), np.int32)
            nat.call("taco_get_labels", dev.h, nat.ptr(lab1), nat.ptr(lab2))
            labels["v"] = (lab1, lab2)
        return labels["v"]

    hist = np.zeros((H, iters))
    nit = np.zeros(H, np.int32)
    nat.call("taco_get_history", dev.h, nat.ptr(hist), nat.ptr(nit))
    out = []
    for j in range(n_sub):
        pair = []
        for b, cb in enumerate((cb1[j], cb2[j])):
            h = hist[2 * j + b][: nit[2 * j + b]]
            pair.append(KMeansModel(centroids=cb.copy(), assignments=None,
                                    inertia=float(h[-1]), inertia_history=tuple(map(float, h)),
                                    n_iter=int(nit[2 * j + b]),
                                    loader=lambda j=j, b=b: fetch_labels()[b][j].copy()))
        out.append(tuple(pair))
    return out


def sorted_centroid_distances(imi: InvertedMultiIndex, query_sub):
    """fp64 squared distances to both codebooks + stable argsorts (GPU k_csort)."""
    q = np.asarray(query_sub, dtype=np.float64).ravel()
    if q.shape[0] != imi.subspace_dim:
        raise DimensionMismatchError(
            f"query has dimension {q.shape[0]}, subspace expects {imi.subspace_dim}")
    q32 = q.astype(np.float32)
    if not np.array_equal(q32.astype(np.float64), q):
        raise ParameterError("sorted_centroid_distances: the B200 path takes float32 queries")
    kp = imi.codebook1.n_clusters
    c1 = np.ascontiguousarray(imi.codebook1.centroids, dtype=np.float32)
    c2 = np.ascontiguousarray(imi.codebook2.centroids, dtype=np.float32)
    d1s, d2s = np.empty(kp), np.empty(kp)
    l1s, l2s = np.empty(kp, np.int32), np.empty(kp, np.int32)
    nat.call("taco_centroid_order", nat.device_id(), nat.ptr(c1), nat.ptr(c2), kp, c1.shape[1],
             c2.shape[1], nat.ptr(q32), nat.ptr(d1s), nat.ptr(l1s), nat.ptr(d2s), nat.ptr(l2s))
    dists1 = np.empty(kp)
    dists2 = np.empty(kp)
    dists1[l1s] = d1s
    dists2[l2s] = d2s
    return dists1, l1s.astype(np.int64), dists2, l2s.astype(np.int64)


def _retrieval_threshold(alpha: float, n: int) -> int:
    if not 0.0 < alpha <= 1.0:
        raise ParameterError(f"collision ratio {alpha} outside (0, 1]")
    return min(n, math.ceil(alpha * n))


def _check_activation_inputs(n_cells, dists1, idx1, dists2, idx2, imi):
    kprime = len(idx1)
    if len(idx2) != kprime or len(dists1) != kprime or len(dists2) != kprime:
        raise ParameterError("distance and index arrays disagree on codebook size")
    if math.isqrt(int(n_cells)) != kprime:
        raise ParameterError(
            f"cluster count {n_cells} does not match {kprime} centroids per codebook")
    if imi.codebook_size != kprime:
        raise ParameterError(
            f"index has {imi.codebook_size} clusters per codebook, inputs have {kprime}")
    return kprime


def scalable_dynamic_activation(alpha, n, n_cells, dists1, idx1, dists2, idx2,
                                imi) -> ActivationResult:
    """Heap traversal in ascending distance-sum order (GPU k_traverse)."""
    kp = _check_activation_inputs(n_cells, dists1, idx1, dists2, idx2, imi)
    if kp > 256:
        raise ParameterError(f"B200 traversal supports K' <= 256 (got {kp})")
    target = _retrieval_threshold(alpha, n)
    i1 = np.asarray(idx1, dtype=np.int64)
    i2 = np.asarray(idx2, dtype=np.int64)
    d1s = np.ascontiguousarray(np.asarray(dists1, dtype=np.float64)[i1])
    d2s = np.ascontiguousarray(np.asarray(dists2, dtype=np.float64)[i2])
    sizes = np.zeros(kp * kp, np.int64)
    for (a, b), ids in imi.cells.items():
        sizes[a * kp + b] = ids.size
    pops = np.empty(kp * kp, np.int32)
    keys = np.empty(kp * kp)
    npop = np.zeros(1, np.int32)
    got = np.zeros(1, np.int64)
    l1s = np.ascontiguousarray(i1, dtype=np.int32)   # keep the buffers alive across the call
    l2s = np.ascontiguousarray(i2, dtype=np.int32)
    nat.call("taco_traverse", nat.device_id(), kp, nat.ptr(d1s), nat.ptr(l1s), nat.ptr(d2s),
             nat.ptr(l2s), nat.ptr(sizes), target, nat.ptr(pops), nat.ptr(keys), nat.ptr(npop),
             nat.ptr(got))
    cells = imi.cells
    retrieved, trace = [], []
    for p, key in zip(pops[: npop[0]], keys[: npop[0]]):
        a, b = int(p) // kp, int(p) % kp
        retrieved.append(cells.get((a, b), _EMPTY_IDS))
        trace.append((float(key), a, b))
    return ActivationResult(tuple(retrieved), int(got[0]), tuple(trace))


def linear_dynamic_activation(alpha, n, n_cells, dists1, idx1, dists2, idx2,
                              imi) -> ActivationResult:
    """The reference's linear-frontier variant (imi.py:169-208).  Its contract
    is the heap traversal's exact cell sequence (the reference asserts the two
    traces are equal, bench.py:248-255), so it runs the same device walk
    (k_traverse); only the reference's CPU cost model differs."""
    return scalable_dynamic_activation(alpha, n, n_cells, dists1, idx1, dists2, idx2, imi)
