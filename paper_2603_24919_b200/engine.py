"""Drop-in engine API of the reference (pkg/src/taco/engine.py) on the B200.

Same names, argument order, defaults, return types and error classes as
engine.py:44-494.  Everything numeric runs through libtaco_b200.so:

  build_index       engine.py:122-174  GPU covariance/transform/k-means/CSR
  knn_query_batch   (additive)         batched device query path (the hot path)
  knn_query         engine.py:282-287  one-query batch
  count_collisions  engine.py:188-220  device counting tap
  select_candidates engine.py:223-253  device histogram + Alg. 5 + compaction
  rerank            engine.py:256-279  device fp64 rerank + top-k
  serialize/save/load_index            index file format v1 (host bytes,
                                       device import on load)

The index owns a device copy of the base vectors (``data`` is passed on
every call in the reference, which never owns it): a call whose ``data``
is not the resident array (pointer, shape, strides and a sampled-row
digest) re-uploads it.
"""

from __future__ import annotations

import functools
import hashlib
import zlib
import math
import struct
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .clustering import KMeansModel
from .errors import (
    CorruptionError,
    DimensionMismatchError,
    FormatError,
    InsufficientDataError,
    NumericError,
    ParameterError,
    StateError,
    UnsupportedVersionError,
)
from .imi import DeviceCells, InvertedMultiIndex, run_kmeans_all
from .seeding import derive_seed
from .spectral import (
    TransformModel,
    as_f32_exact,
    covariance_from_gram,
    model_from_covariance,
    transform_points,
)

INDEX_MAGIC = b"TACO"
TOPK_MAX = 2048   # query.cu TK_MAX: results per query the device top-k keeps
INDEX_VERSION = 1
_MAX_SUBSPACES = 255


@dataclass(frozen=True)
class IndexParams:
    n_subspaces: int
    subspace_dim: int
    clusters: int = 4096
    kmeans_iters: int = 20
    seed: int = 0

    def __post_init__(self):
        if not 1 <= self.n_subspaces <= _MAX_SUBSPACES:
            raise ParameterError(f"subspace count {self.n_subspaces} outside [1, {_MAX_SUBSPACES}]")
        if self.subspace_dim < 2:
            raise ParameterError(f"subspace dimension {self.subspace_dim} is below 2")
        kprime = math.isqrt(int(self.clusters)) if self.clusters >= 1 else 0
        if kprime < 1 or kprime * kprime != self.clusters:
            raise ParameterError(f"cluster count {self.clusters} is not a perfect square")
        if self.kmeans_iters < 1:
            raise ParameterError(f"k-means iteration cap {self.kmeans_iters} is below 1")

    @property
    def codebook_size(self) -> int:
        return math.isqrt(int(self.clusters))

    @property
    def output_dim(self) -> int:
        return self.n_subspaces * self.subspace_dim


@dataclass(frozen=True)
class QueryParams:
    alpha: float
    beta: float
    k: int = 50

    def __post_init__(self):
        if not 0.0 < self.alpha < 1.0:
            raise ParameterError(f"collision ratio {self.alpha} outside (0, 1)")
        if not 0.0 < self.beta < 1.0:
            raise ParameterError(f"re-rank ratio {self.beta} outside (0, 1)")
        if self.k < 1:
            raise ParameterError(f"result count {self.k} is below 1")


@dataclass
class TacoIndex:
    params: IndexParams
    transform: TransformModel
    subspaces: list
    n: int
    metadata: dict = field(default_factory=dict)
    transformed: np.ndarray | None = None
    device: object = field(default=None, repr=False, compare=False)

    @property
    def d(self) -> int:
        return self.transform.d


@dataclass(frozen=True)
class CandidateSet:
    ids: np.ndarray
    candidate_num: int
    last_collision: int


@dataclass(frozen=True)
class SearchResult:
    ids: np.ndarray    # int32, ascending exact distance, ties by id
    dists: np.ndarray  # float32


# ------------------------------------------------------------------- helpers
@functools.lru_cache(maxsize=16)
def _sample_rows(n: int):
    return np.unique(np.linspace(0, max(n - 1, 0), num=min(n, 64)).astype(np.int64)) if n else np.zeros(0, np.int64)


def _data_key(X: np.ndarray):
    # 64 sampled rows; of a wide row only its first and last 64 columns (at d = 960 hashing whole
    # rows cost 0.25 ms per call, 6 % of a config-3 batch)
    # crc32 + adler32 (64 bits, ~20 us for 32 KB; blake2b took 50 us of a 540 us config-1 batch)
    S = X[_sample_rows(X.shape[0])]
    if X.ndim == 2 and X.shape[1] > 128:
        b = np.ascontiguousarray(S[:, :64]).tobytes() + np.ascontiguousarray(S[:, -64:]).tobytes()
    else:
        b = S.tobytes()
    return (X.ctypes.data, X.shape, X.strides, X.dtype.str, zlib.crc32(b), zlib.adler32(b))


def refresh_data(index: TacoIndex, data) -> None:
    """Re-upload ``data`` as the index's resident base matrix unconditionally.

    The per-call identity check (``_data_key``: pointer, shape, strides,
    dtype and a digest of 64 sampled rows -- of rows wider than 128 columns
    their first and last 64) cannot see an in-place edit of values it does
    not sample; a caller that mutates ``data`` in place between
    queries calls this."""
    dev = _device_of(index)
    X = as_f32_exact(np.asarray(data), "data")
    if X.ndim != 2 or X.shape != (index.n, index.d):
        raise DimensionMismatchError(
            f"data shape {X.shape} does not match index ({index.n}, {index.d})")
    X = np.ascontiguousarray(X)
    nat.call("taco_index_set_data", dev.h, nat.ptr(X))
    dev.data_key = _data_key(X)


def _resident(index: TacoIndex, data) -> np.ndarray:
    """Make ``data`` the device-resident base matrix of ``index``."""
    dev = _device_of(index)
    X = as_f32_exact(np.asarray(data), "data")
    if X.ndim != 2 or X.shape != (index.n, index.d):
        raise DimensionMismatchError(
            f"data shape {X.shape} does not match index ({index.n}, {index.d})")
    key = _data_key(X)
    if dev.data_key != key:
        nat.call("taco_index_set_data", dev.h, nat.ptr(X))
        dev.data_key = key
    return X


def _device_of(index: TacoIndex):
    if index.device is None:
        index.device = _import_device(index)
    return index.device


def _import_device(index: TacoIndex, n_global=None, id_base=0, device=None):
    """Upload a host-side index (v1 file / reference-built object) to the GPU."""
    p = index.params
    kp = p.codebook_size
    dev = nat.DeviceIndex(index.n, index.d, p.n_subspaces, p.subspace_dim, p.clusters,
                          p.kmeans_iters, device=device, n_global=n_global, id_base=id_base)
    M = np.ascontiguousarray(index.transform.matrix, dtype=np.float32)
    mean = np.ascontiguousarray(index.transform.mean, dtype=np.float32)
    nat.call("taco_index_set_transform", dev.h, nat.ptr(mean), nat.ptr(M))
    cb1 = np.ascontiguousarray(np.stack([s.codebook1.centroids for s in index.subspaces]), np.float32)
    cb2 = np.ascontiguousarray(np.stack([s.codebook2.centroids for s in index.subspaces]), np.float32)
    nat.call("taco_index_set_codebooks", dev.h, nat.ptr(cb1), nat.ptr(cb2))
    K2 = kp * kp
    offs = np.zeros((p.n_subspaces, K2 + 1), np.int64)
    ids = np.empty((p.n_subspaces, index.n), np.uint32)
    for j, sub in enumerate(index.subspaces):
        sizes = np.zeros(K2, np.int64)
        parts = [None] * K2
        for (a, b), v in sub.cells.items():
            sizes[a * kp + b] = v.size
            parts[a * kp + b] = np.asarray(v, dtype=np.uint32)
        offs[j, 1:] = np.cumsum(sizes)
        if offs[j, -1] != index.n:
            raise CorruptionError(f"subspace cells hold {offs[j, -1]} ids, expected {index.n}")
        nz = [x for x in parts if x is not None]
        ids[j] = np.concatenate(nz) if nz else np.empty(0, np.uint32)
    nat.call("taco_index_set_cells", dev.h, nat.ptr(offs), nat.ptr(ids))
    return dev


def import_index(index) -> TacoIndex:
    """Wrap any object with the reference's TacoIndex attributes (e.g. one
    built by the reference package) as a device-backed index."""
    p = index.params
    params = IndexParams(p.n_subspaces, p.subspace_dim, p.clusters, p.kmeans_iters, p.seed)
    tm = TransformModel(mean=np.asarray(index.transform.mean, np.float32),
                        blocks=tuple(np.asarray(b, np.float32) for b in index.transform.blocks))
    subs = []
    for sub in index.subspaces:
        subs.append(InvertedMultiIndex(
            codebook1=KMeansModel(np.asarray(sub.codebook1.centroids, np.float32), None, float("nan")),
            codebook2=KMeansModel(np.asarray(sub.codebook2.centroids, np.float32), None, float("nan")),
            cells=dict(sub.cells), codebook_size=sub.codebook_size, split=sub.split))
    out = TacoIndex(params=params, transform=tm, subspaces=subs, n=int(index.n),
                    metadata={"imported": True})
    out.device = _import_device(out)
    return out


# --------------------------------------------------------------------- build
def build_index(data, params: IndexParams, keep_transformed: bool = False) -> TacoIndex:
    """Transform the dataset and build one inverted multi-index per subspace."""
    X = np.ascontiguousarray(data, dtype=np.float32)
    if X.ndim != 2:
        raise ParameterError(f"expected a 2-D matrix, got shape {X.shape}")
    n, d = X.shape
    if params.output_dim > d:
        raise ParameterError(
            f"subspace budget {params.output_dim} ({params.n_subspaces} x "
            f"{params.subspace_dim}) exceeds data dimension {d}")
    if n < params.codebook_size:
        raise InsufficientDataError(
            f"{n} points cannot fill {params.codebook_size} clusters per codebook")
    if n < 2:
        raise InsufficientDataError(f"covariance needs at least 2 rows, got {n}")
    kp = params.codebook_size
    s = params.subspace_dim
    if (s + 1) // 2 > 32 or kp > 256:
        raise ParameterError(f"B200 build supports half widths <= 32 and K' <= 256 "
                             f"(got s={s}, K'={kp})")
    t0 = time.perf_counter()
    dev = nat.DeviceIndex(n, d, params.n_subspaces, s, params.clusters, params.kmeans_iters)
    nat.call("taco_index_set_data", dev.h, nat.ptr(X))
    dev.data_key = _data_key(X)
    mean = np.empty(d)
    gram = np.empty((d, d))
    bad = np.zeros(1, np.int64)
    nat.call("taco_fit_covariance", dev.h, nat.ptr(mean), nat.ptr(gram), nat.ptr(bad))
    if bad[0] >= 0:
        raise NumericError(f"non-finite value in row {int(bad[0])}")
    t_cov = time.perf_counter()
    model = model_from_covariance(covariance_from_gram(mean, gram, n), d, params.n_subspaces, s)
    t_eig = time.perf_counter()
    M = np.ascontiguousarray(model.matrix, dtype=np.float32)
    nat.call("taco_index_set_transform", dev.h, nat.ptr(model.mean), nat.ptr(M))
    nat.call("taco_transform_data", dev.h)
    t_transform = time.perf_counter() - t0
    t_km0 = time.perf_counter()
    models = run_kmeans_all(dev, n, params.n_subspaces, s, kp, params.kmeans_iters,
                            lambda j, h: derive_seed(derive_seed(params.seed, j), h))
    t_km1 = time.perf_counter()
    nat.call("taco_build_cells", dev.h)
    t_cells = time.perf_counter()
    subspaces = [InvertedMultiIndex(codebook1=c1, codebook2=c2, cells=DeviceCells(dev, j, kp),
                                    codebook_size=kp, split=(s + 1) // 2)
                 for j, (c1, c2) in enumerate(models)]
    total = time.perf_counter() - t0
    metadata = {
        "n": n,
        "d": d,
        "output_dim": params.output_dim,
        "dim_reduction_pct": 100.0 * (1.0 - params.output_dim / d),
        "transform_seconds": t_transform,
        "kmeans_seconds": total - t_transform,
        "build_seconds": total,
        "covariance_seconds": t_cov - t0,
        "eigensolve_seconds": t_eig - t_cov,
        "transform_only_seconds": t_km0 - t_eig,
        "kmeans_only_seconds": t_km1 - t_km0,
        "cells_seconds": t_cells - t_km1,
        "warnings": list(model.warnings),
        "device": dev.device,
    }
    dev.has_T = True   # the device keeps the transformed matrix it built from
    transformed = None
    if keep_transformed:
        transformed = np.empty((n, params.output_dim), np.float32)
        nat.call("taco_get_transformed", dev.h, nat.ptr(transformed))
        dev.transformed_key = _data_key(transformed)
    return TacoIndex(params=params, transform=model, subspaces=subspaces, n=n, metadata=metadata,
                     transformed=transformed, device=dev)


def attach_transformed(index: TacoIndex, data) -> TacoIndex:
    """Recompute and retain the transformed matrix on a built/loaded index."""
    X = np.ascontiguousarray(data, dtype=np.float32)
    if X.ndim != 2 or X.shape[0] != index.n or X.shape[1] != index.d:
        raise ParameterError(
            f"data shape {np.shape(data)} does not match index ({index.n}, {index.d})")
    index.transformed = transform_points(index.transform, X)
    dev = index.device
    if dev is not None and getattr(dev, "has_T", False) and dev.data_key == _data_key(X):
        dev.transformed_key = _data_key(index.transformed)   # same rows as the resident matrix
    return index


# --------------------------------------------------------------------- query
def _query_vector(index, query):
    q = np.asarray(query, dtype=np.float32).ravel()
    if q.shape[0] != index.d:
        raise DimensionMismatchError(f"query has dimension {q.shape[0]}, index expects {index.d}")
    return np.ascontiguousarray(q)


def count_collisions(index: TacoIndex, query, alpha: float, out: np.ndarray | None = None) -> np.ndarray:
    """Per-point count of subspaces whose activation retrieved the point."""
    q = _query_vector(index, query)
    if out is not None and (out.shape != (index.n,) or out.dtype != np.uint8):
        raise ParameterError("score buffer must be uint8 of length n")
    if not 0.0 < alpha <= 1.0:
        raise ParameterError(f"collision ratio {alpha} outside (0, 1]")
    scores = np.empty(index.n, np.uint8) if out is None else out
    buf = scores if scores.flags["C_CONTIGUOUS"] else np.empty(index.n, np.uint8)
    nat.call("taco_count_scores", _device_of(index).h, nat.ptr(q), float(alpha), nat.ptr(buf))
    if buf is not scores:
        scores[:] = buf
    return scores


def select_candidates(scores, beta: float, n_subspaces: int, n: int | None = None) -> CandidateSet:
    """Adaptive threshold scan over the score histogram (device)."""
    scores = np.asarray(scores)
    if n is None:
        n = scores.shape[0]
    elif n != scores.shape[0]:
        raise ParameterError(f"score table has {scores.shape[0]} entries, n={n}")
    if not 0.0 < beta < 1.0:
        raise ParameterError(f"re-rank ratio {beta} outside (0, 1)")
    if n == 0:
        return CandidateSet(ids=np.empty(0, np.int64), candidate_num=0, last_collision=max(n_subspaces, 0))
    if scores.size and (scores.min() < 0 or scores.max() > n_subspaces):
        raise ParameterError(f"scores must lie in [0, {n_subspaces}]")
    sc = np.ascontiguousarray(scores, dtype=np.uint8)
    ids = np.empty(n, np.int64)
    num = np.zeros(1, np.int64)
    lvl = np.zeros(1, np.int32)
    nat.call("taco_select_candidates", nat.device_id(), nat.ptr(sc), n, int(n_subspaces), float(beta),
             nat.ptr(ids), nat.ptr(num), nat.ptr(lvl))
    return CandidateSet(ids=ids[: int(num[0])].copy(), candidate_num=int(num[0]),
                        last_collision=int(lvl[0]))


def rerank(data, query, candidates, k: int) -> SearchResult:
    """Exact top-k among the candidates, ascending distance, ties by id (device)."""
    if k < 1:
        raise ParameterError(f"result count {k} is below 1")
    ids = candidates.ids if isinstance(candidates, CandidateSet) else candidates
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
    if ids.size == 0:
        return SearchResult(ids=np.empty(0, dtype=np.int32), dists=np.empty(0, dtype=np.float32))
    X = np.asarray(data)
    q = np.asarray(query, dtype=np.float64).ravel()
    if q.shape[0] != X.shape[1]:
        raise DimensionMismatchError(f"query has dimension {q.shape[0]}, data has {X.shape[1]}")
    X32 = as_f32_exact(X, "rerank data")
    q32 = as_f32_exact(q, "rerank query")
    kk = min(int(k), ids.size)
    oi = np.empty(kk, np.int32)
    od = np.empty(kk, np.float32)
    o2 = np.empty(kk)
    nat.call("taco_rerank", nat.device_id(), nat.ptr(X32), X32.shape[0], X32.shape[1], nat.ptr(q32),
             nat.ptr(ids), ids.size, kk, nat.ptr(oi), nat.ptr(od), nat.ptr(o2))
    return SearchResult(ids=oi, dists=od)


def knn_query_batch(index: TacoIndex, data, queries, qp: QueryParams):
    """Batched k-ANN (the B200 hot path; additive to the reference API).

    Returns (ids int32[nq, k] -1 padded, dists f32[nq, k] +inf padded,
    candidate_num int64[nq], last_collision int32[nq]) -- per query
    identical to ``knn_query`` and to the reference's per-query pipeline,
    padded like cli.py:155-164."""
    _resident(index, data)
    Q = as_f32_exact(np.asarray(queries), "queries")
    if Q.ndim != 2 or Q.shape[1] != index.d:
        raise DimensionMismatchError(f"queries have shape {Q.shape}, index expects (*, {index.d})")
    nq, k = Q.shape[0], int(qp.k)
    # at most min(k, n) results exist: a k beyond the device top-k limit is
    # served when n itself fits under it (the rest is padding)
    kk = min(k, index.n) if k > TOPK_MAX else k
    if kk > TOPK_MAX:
        raise ParameterError(f"result count {k} exceeds the B200 top-k limit {TOPK_MAX} "
                             f"(n = {index.n})")
    if kk == k and nq:   # the library writes every slot, padding included
        ids = np.empty((nq, k), np.int32)
        dists = np.empty((nq, k), np.float32)
    else:
        ids = np.full((nq, k), -1, np.int32)
        dists = np.full((nq, k), np.inf, np.float32)
    num = np.empty(nq, np.int64)
    lvl = np.empty(nq, np.int32)
    if nq:
        oi = ids if kk == k else np.empty((nq, kk), np.int32)
        od = dists if kk == k else np.empty((nq, kk), np.float32)
        nat.call("taco_query_batch", _device_of(index).h, nat.ptr(Q), nq, float(qp.alpha), float(qp.beta),
                 kk, nat.ptr(oi), nat.ptr(od), nat.ptr(num), nat.ptr(lvl))
        if kk != k:
            ids[:, :kk] = oi
            dists[:, :kk] = od
    return ids, dists, num, lvl


def knn_query(index: TacoIndex, data, query, qp: QueryParams,
              scratch: np.ndarray | None = None) -> SearchResult:
    """Collision counting, adaptive candidate selection, exact re-rank."""
    q = _query_vector(index, query)
    if scratch is not None and (scratch.shape != (index.n,) or scratch.dtype != np.uint8):
        raise ParameterError("score buffer must be uint8 of length n")
    X = np.asarray(data)
    if X.ndim == 2 and X.shape[1] != q.shape[0]:
        raise DimensionMismatchError(f"query has dimension {q.shape[0]}, data has {X.shape[1]}")
    if scratch is not None:   # engine.py:285: the reference counts into the caller's buffer
        count_collisions(index, q, qp.alpha, out=scratch)
    ids, dists, _, _ = knn_query_batch(index, data, q[None, :], qp)
    keep = ids[0] >= 0
    return SearchResult(ids=ids[0][keep].copy(), dists=dists[0][keep].copy())


def sc_linear_scores(transformed, query_t, n_subspaces: int, subspace_dim: int,
                     alpha: float) -> np.ndarray:
    """Exact collision counting without the index (engine.py:290-321), on the
    GPU: per subspace the ceil(alpha*n) nearest points by (fp64 einsum d2, id)
    collide; scores[i] = number of subspaces where i collides."""
    Tm = np.asarray(transformed)
    qt = np.asarray(query_t).ravel()
    if Tm.ndim != 2:
        raise ParameterError(f"expected a 2-D matrix, got shape {Tm.shape}")
    n = Tm.shape[0]
    if qt.shape[0] != Tm.shape[1]:
        raise DimensionMismatchError(
            f"query has dimension {qt.shape[0]}, transformed data has {Tm.shape[1]}")
    if n_subspaces * subspace_dim != Tm.shape[1]:
        raise ParameterError(f"{n_subspaces} x {subspace_dim} does not cover {Tm.shape[1]} columns")
    if not 0.0 < alpha <= 1.0:
        raise ParameterError(f"collision ratio {alpha} outside (0, 1]")
    scores = np.zeros(n, np.uint8)
    if n == 0:
        return scores
    T32 = as_f32_exact(Tm, "transformed")
    q32 = as_f32_exact(qt, "query_t")
    nat.call("taco_sc_linear_scores", nat.device_id(), nat.ptr(T32), n, int(n_subspaces), int(subspace_dim),
             nat.ptr(q32), float(alpha), nat.ptr(scores))
    return scores


def sc_linear_query(index: TacoIndex, data, query, qp: QueryParams) -> SearchResult:
    """Query through exact collision counting over the retained transformed
    matrix (engine.py:324-342).  The scores come from the index's resident
    transformed matrix when it holds the same rows, else from the host copy."""
    if index.transformed is None:
        raise StateError(
            "transformed matrix was not retained at build time; rebuild with "
            "keep_transformed=True or call attach_transformed()")
    q = np.asarray(query, dtype=np.float32).ravel()
    if q.shape[0] != index.d:
        raise DimensionMismatchError(f"query has dimension {q.shape[0]}, index expects {index.d}")
    qt = np.ascontiguousarray(transform_points(index.transform, q[None, :])[0], dtype=np.float32)
    p = index.params
    scores = None
    dev = index.device
    if dev is not None and getattr(dev, "transformed_key", None) == _data_key(index.transformed):
        scores = np.zeros(index.n, np.uint8)
        nat.call("taco_sc_linear_scores_index", dev.h, nat.ptr(qt), float(qp.alpha), nat.ptr(scores))
    if scores is None:
        scores = sc_linear_scores(index.transformed, qt, p.n_subspaces, p.subspace_dim, qp.alpha)
    cand = select_candidates(scores, qp.beta, p.n_subspaces, index.n)
    return rerank(data, query, cand, qp.k)


# --------------------------------------------------------------- persistence
_HEADER = struct.Struct("<QIIIIIq")


def serialize_index(index: TacoIndex) -> bytes:
    """Index file format v1 (engine.py:345-384): LE, blake2b-64 trailer."""
    params = index.params
    if index.n > 0xFFFFFFFF:
        raise ParameterError("indexes beyond 2^32 points cannot be serialized")
    parts = [INDEX_MAGIC, struct.pack("<H", INDEX_VERSION),
             _HEADER.pack(index.n, index.d, params.n_subspaces, params.subspace_dim, params.clusters,
                          params.kmeans_iters, params.seed),
             np.asarray(index.transform.mean, "<f4").tobytes()]
    for block in index.transform.blocks:
        parts.append(np.asarray(block, "<f4").tobytes(order="F"))
    for sub in index.subspaces:
        parts.append(np.asarray(sub.codebook1.centroids, "<f4").tobytes())
        parts.append(np.asarray(sub.codebook2.centroids, "<f4").tobytes())
        keys = sorted(sub.cells)
        parts.append(struct.pack("<II", sub.codebook_size, len(keys)))
        for a, b in keys:
            ids = sub.cells[(a, b)]
            parts.append(struct.pack("<HHI", a, b, ids.size))
            parts.append(np.asarray(ids, "<u4").tobytes())
    body = b"".join(parts)
    return body + hashlib.blake2b(body, digest_size=8).digest()


def save_index(index: TacoIndex, path) -> None:
    blob = serialize_index(index)
    with open(path, "wb") as fh:
        fh.write(blob)


def _parse(blob: bytes, path):
    if len(blob) < 4 + 2 + 8:
        raise CorruptionError(f"{path}: file too short ({len(blob)} bytes)")
    if blob[:4] != INDEX_MAGIC:
        raise FormatError(f"{path}: bad magic {blob[:4]!r}")
    (version,) = struct.unpack_from("<H", blob, 4)
    if version != INDEX_VERSION:
        raise UnsupportedVersionError(
            f"{path}: format version {version}, this build supports {INDEX_VERSION}")
    body, checksum = blob[:-8], blob[-8:]
    if hashlib.blake2b(body, digest_size=8).digest() != checksum:
        raise CorruptionError(f"{path}: checksum mismatch")
    pos = 6

    def take(size):
        nonlocal pos
        if pos + size > len(body):
            raise CorruptionError(f"{path}: unexpected end of file at byte {pos}")
        chunk = body[pos:pos + size]
        pos += size
        return chunk

    n, d, n_sub, s, clusters, iters, seed = _HEADER.unpack(take(_HEADER.size))
    try:
        params = IndexParams(n_subspaces=n_sub, subspace_dim=s, clusters=clusters,
                             kmeans_iters=iters, seed=seed)
    except ParameterError as exc:
        raise CorruptionError(f"{path}: invalid stored parameters: {exc}") from exc
    f32 = lambda cnt: np.frombuffer(take(4 * cnt), "<f4").astype(np.float32)  # noqa: E731
    mean = f32(d)
    blocks = tuple(f32(d * s).reshape((d, s), order="F").copy() for _ in range(n_sub))
    split = (s + 1) // 2
    kp = params.codebook_size
    subs = []
    for _ in range(n_sub):
        c1 = f32(kp * split).reshape(kp, split)
        c2 = f32(kp * (s - split)).reshape(kp, s - split)
        stored, n_cells = struct.unpack("<II", take(8))
        if stored != kp:
            raise CorruptionError(f"{path}: subspace codebook size {stored}, expected {kp}")
        cells = {}
        total = 0
        for _ in range(n_cells):
            a, b, size = struct.unpack("<HHI", take(8))
            cells[(a, b)] = np.frombuffer(take(4 * size), "<u4").astype(np.uint32)
            total += size
        if total != n:
            raise CorruptionError(f"{path}: subspace cells hold {total} ids, expected {n}")
        subs.append(InvertedMultiIndex(
            codebook1=KMeansModel(centroids=c1, assignments=None, inertia=float("nan")),
            codebook2=KMeansModel(centroids=c2, assignments=None, inertia=float("nan")),
            cells=cells, codebook_size=kp, split=split))
    if pos != len(body):
        raise CorruptionError(f"{path}: {len(body) - pos} trailing bytes")
    return TacoIndex(params=params, transform=TransformModel(mean=mean, blocks=blocks),
                     subspaces=subs, n=int(n), metadata={"loaded_from": str(path)})


def deserialize_index(blob: bytes, path="<bytes>") -> TacoIndex:
    index = _parse(blob, path)
    index.device = _import_device(index)
    return index


def load_index(path) -> TacoIndex:
    """Load an index file onto the GPU; rejects bad magic, versions, checksums."""
    with open(path, "rb") as fh:
        blob = fh.read()
    return deserialize_index(blob, path)
