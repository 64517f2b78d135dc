"""k-means (reference clustering.py) with the arithmetic on the GPU.

The host keeps only the random stream: ``default_rng(seed)`` draws the
first centroid with ``integers(n)`` and one ``random()`` per k-means++
draw, exactly the calls ``Generator.choice(n, p=...)`` makes in the
reference (clustering.py:44-51).  The device does the D^2 updates, the
certified CDF search (k_pp_search), the Lloyd assignments and the
sequential per-cluster sums (build.cu).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .errors import DimensionMismatchError, InsufficientDataError, ParameterError

MAX_HALF_DIM = 32
MAX_CLUSTERS = 256


class KMeansModel:
    """Fitted codebook (reference clustering.py:17-31).

    ``assignments`` may be supplied lazily through ``loader`` (a callable
    returning the int32 labels): a device-built index keeps its labels in HBM
    and copies them to the host only when a caller first reads them."""

    __slots__ = ("centroids", "_assignments", "_loader", "inertia", "inertia_history", "n_iter")

    def __init__(self, centroids, assignments=None, inertia: float = float("nan"),
                 inertia_history: tuple = (), n_iter: int = 0, *, loader=None):
        self.centroids = centroids
        self._assignments = assignments
        self._loader = loader
        self.inertia = inertia
        self.inertia_history = inertia_history
        self.n_iter = n_iter

    @property
    def assignments(self):
        if self._assignments is None and self._loader is not None:
            self._assignments = self._loader()
            self._loader = None
        return self._assignments

    @property
    def n_clusters(self) -> int:
        return self.centroids.shape[0]

    @property
    def dim(self) -> int:
        return self.centroids.shape[1]

    def __repr__(self):
        return (f"KMeansModel(n_clusters={self.n_clusters}, dim={self.dim}, inertia={self.inertia!r}, "
                f"n_iter={self.n_iter})")


def draw_plan(n: int, k: int, seed: int):
    """(first, uniforms[k-1]) of the reference's k-means++ stream."""
    rng = np.random.default_rng(seed)
    first = int(rng.integers(n))
    uni = np.array([rng.random() for _ in range(k - 1)], dtype=np.float64)
    return first, uni


def forced_plan(n: int, k: int, seed: int, degenerate_at: int):
    """Replay when the D^2 total hit 0 at draw ``degenerate_at``: from there on
    every draw is ``rng.integers(n)`` (clustering.py:50-51)."""
    rng = np.random.default_rng(seed)
    rng.integers(n)
    forced = np.full(max(k - 1, 0), -1, np.int64)
    for i in range(1, k):
        if i < degenerate_at:
            rng.random()
        else:
            forced[i - 1] = int(rng.integers(n))
    return forced


def check_kmeans_args(X, n_clusters, max_iter):
    if X.ndim != 2:
        raise ParameterError(f"k-means expects a 2-D matrix, got shape {X.shape}")
    n, m = X.shape
    if n_clusters < 1:
        raise ParameterError(f"cluster count must be positive, got {n_clusters}")
    if m < 1:
        raise ParameterError("points need at least one dimension")
    if max_iter < 1:
        raise ParameterError(f"iteration cap must be positive, got {max_iter}")
    if n < n_clusters:
        raise InsufficientDataError(f"{n} points cannot fill {n_clusters} clusters")
    if m > MAX_HALF_DIM or n_clusters > MAX_CLUSTERS:
        raise ParameterError(f"B200 k-means supports m <= {MAX_HALF_DIM} and k <= {MAX_CLUSTERS} "
                             f"(got m={m}, k={n_clusters})")


def kmeans(data, n_clusters: int, max_iter: int = 20, seed: int = 0) -> KMeansModel:
    """Seeded k-means++ then at most max_iter Lloyd iterations (GPU)."""
    X = np.ascontiguousarray(np.asarray(data, dtype=np.float32))
    check_kmeans_args(X, n_clusters, max_iter)
    n, m = X.shape
    k = int(n_clusters)
    first, uni = draw_plan(n, k, seed)
    cent = np.empty((k, m), np.float32)
    lab = np.empty(n, np.int32)
    hist = np.zeros(max_iter)
    nit = np.zeros(1, np.int32)
    deg = np.zeros(1, np.int32)

    def run(forced):
        nat.call("taco_kmeans", nat.device_id(), nat.ptr(X), n, m, k, int(max_iter), first,
                 nat.ptr(uni), nat.ptr(forced), nat.ptr(cent), nat.ptr(lab), nat.ptr(hist),
                 nat.ptr(nit), nat.ptr(deg))

    run(None)
    if deg[0] < k:
        run(forced_plan(n, k, seed, int(deg[0])))
    history = tuple(float(v) for v in hist[: int(nit[0])])
    return KMeansModel(centroids=cent, assignments=lab, inertia=history[-1],
                       inertia_history=history, n_iter=len(history))


def assign(model: KMeansModel, point) -> int:
    """Index of the nearest centroid, ties to the lowest index
    (clustering.py:118-127).  The device computes the reference's fp64
    direct-form einsum distances and their stable rank (k_csort); the first
    entry of a stable ascending argsort is numpy's first argmin."""
    p = np.asarray(point, dtype=np.float64).ravel()
    if p.shape[0] != model.dim:
        raise DimensionMismatchError(
            f"point has dimension {p.shape[0]}, centroids have {model.dim}")
    p32 = p.astype(np.float32)
    if not np.array_equal(p32.astype(np.float64), p):
        raise ParameterError("assign: the B200 path takes float32-representable points")
    C = np.ascontiguousarray(model.centroids, dtype=np.float32)
    k, m = C.shape
    q = np.ascontiguousarray(np.concatenate([p32, p32]))
    d1s, d2s = np.empty(k), np.empty(k)
    l1s, l2s = np.empty(k, np.int32), np.empty(k, np.int32)
    nat.call("taco_centroid_order", nat.device_id(), nat.ptr(C), nat.ptr(C), k, m, m, nat.ptr(q),
             nat.ptr(d1s), nat.ptr(l1s), nat.ptr(d2s), nat.ptr(l2s))
    return int(l1s[0])


__all__ = ["KMeansModel", "assign", "kmeans", "draw_plan", "forced_plan", "DimensionMismatchError"]
