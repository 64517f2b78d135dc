"""Spectral transform (reference spectral.py) on the B200 path.

* ``fit_covariance``   fp64 mean + centred Gram on the GPU (k_colmean_seq,
                       k_gram), normalised/symmetrised here exactly as
                       spectral.py:109-110 does.
* ``jacobi_eigh``      validation/tolerance in numpy as spectral.py:148-158,
                       sweeps in the native host restatement (jacobi.cpp) --
                       bit-identical to the reference's numpy sweeps.
* ``eigendecompose`` / ``allocate_eigensystem``: O(d^2) host bookkeeping
                       identical to spectral.py:198-265.
* ``transform_points`` GPU fp64 GEMM (k_transform).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import (
    ConvergenceError,
    DimensionMismatchError,
    InsufficientDataError,
    NumericError,
    ParameterError,
)

ZERO_EIGENVALUE_REL = 1e-12
JACOBI_TOL_REL = 1e-9
JACOBI_MAX_SWEEPS = 100


@dataclass(frozen=True)
class CovarianceModel:
    mean: np.ndarray  # (d,) float64
    cov: np.ndarray   # (d, d) float64, symmetric


@dataclass(frozen=True)
class EigenSystem:
    eigenvalues: np.ndarray      # (d,) float64, scaled, descending
    eigenvectors: np.ndarray     # (d, d) float64, column i pairs with eigenvalues[i]
    scale_factor: float
    raw_eigenvalues: np.ndarray  # (d,) float64, clamped at 0

    @property
    def dim(self) -> int:
        return self.eigenvalues.shape[0]


@dataclass(frozen=True)
class SubspaceAllocation:
    buckets: tuple
    log_products: np.ndarray

    @property
    def products(self) -> np.ndarray:
        return np.exp(self.log_products)


@dataclass(frozen=True)
class TransformModel:
    mean: np.ndarray                 # (d,) float32
    blocks: tuple                    # N_s arrays (d, s) float32
    warnings: tuple = ()

    @property
    def d(self) -> int:
        return self.mean.shape[0]

    @property
    def n_subspaces(self) -> int:
        return len(self.blocks)

    @property
    def subspace_dim(self) -> int:
        return self.blocks[0].shape[1]

    @property
    def output_dim(self) -> int:
        return self.n_subspaces * self.subspace_dim

    @property
    def matrix(self) -> np.ndarray:
        return np.concatenate(self.blocks, axis=1)


def as_f32_exact(X, what: str) -> np.ndarray:
    """The device path reads float32; other dtypes are accepted only when
    every value is exactly a float32 (so the fp64 math is unchanged)."""
    A = np.asarray(X)
    if A.dtype == np.float32:
        return np.ascontiguousarray(A)
    A32 = np.ascontiguousarray(A, dtype=np.float32)
    with np.errstate(invalid="ignore"):
        same = np.array_equal(A32.astype(A.dtype), A, equal_nan=True) if A.size else True
    if not same:
        raise ParameterError(f"{what}: the B200 path takes float32 values (got {A.dtype} "
                             "values not representable in float32)")
    return A32


def covariance_from_gram(mean, gram, n):
    cov = gram / (n - 1)                      # spectral.py:109
    return CovarianceModel(mean=mean, cov=(cov + cov.T) / 2.0)   # spectral.py:110


def fit_covariance(data) -> CovarianceModel:
    """Row mean and unbiased sample covariance, symmetrized on return."""
    X = np.asarray(data)
    if X.ndim != 2:
        raise ParameterError(f"expected a 2-D matrix, got shape {X.shape}")
    n, d = X.shape
    if n < 2:
        raise InsufficientDataError(f"covariance needs at least 2 rows, got {n}")
    X32 = as_f32_exact(X, "fit_covariance")
    mean = np.empty(d)
    gram = np.empty((d, d))
    bad = np.zeros(1, np.int64)
    nat.call("taco_covariance", nat.device_id(), nat.ptr(X32), n, d, nat.ptr(mean), nat.ptr(gram),
             nat.ptr(bad))
    if bad[0] >= 0:
        raise NumericError(f"non-finite value in row {int(bad[0])}")
    return covariance_from_gram(mean, gram, n)


def _eig_on_device() -> bool:
    """The sweeps run on the GPU (eigen.cu) unless TACO_EIG=host selects the
    bit-identical host restatement (jacobi.cpp), e.g. on a machine without a GPU."""
    if os.environ.get("TACO_EIG", "") == "host":
        return False
    return nat.gpu_available()


def jacobi_eigh(matrix, tol_rel: float = JACOBI_TOL_REL, max_sweeps: int = JACOBI_MAX_SWEEPS):
    """Eigensystem via cyclic Jacobi rotations (spectral.py:139-195)."""
    A = np.array(matrix, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ParameterError(f"expected a square matrix, got shape {A.shape}")
    d = A.shape[0]
    scale = max(1.0, float(np.abs(A).max()) if A.size else 1.0)
    if float(np.abs(A - A.T).max() if A.size else 0.0) > 1e-6 * scale:
        raise ParameterError("matrix is not symmetric")
    A = np.ascontiguousarray((A + A.T) / 2.0)
    if d <= 1:
        return np.diag(A).copy(), np.eye(d)
    # ||A||_F without BLAS: np.linalg.norm routes through a threaded OpenBLAS
    # ddot (n > 10^4), whose worker threads then spin for ~0.1 s and starve
    # the staged upload of the next build of host cores (30 ms instead of 9).
    # The threshold differs from it at most in the last bits, as the threaded
    # ddot's own value does between machines with different core counts.
    tol = tol_rel * math.sqrt(float(np.sum(A * A)))
    V = np.empty((d, d))
    sweeps = np.zeros(1, np.int32)
    resid = np.zeros(1)
    if _eig_on_device():
        rc = nat.lib().taco_jacobi_sweeps_device(nat.device_id(), nat.ptr(A), nat.ptr(V), d, tol,
                                                 int(max_sweeps), nat.ptr(sweeps), nat.ptr(resid))
    else:
        rc = nat.lib().taco_jacobi_sweeps(nat.ptr(A), nat.ptr(V), d, tol, int(max_sweeps),
                                          nat.ptr(sweeps), nat.ptr(resid))
    if rc == 5:
        raise ConvergenceError(nat.lib().taco_last_error().decode())
    nat.check(rc)
    return np.diag(A).copy(), V


def _scale_spectrum(raw):
    lam_max = float(raw[0]) if raw.size else 0.0
    if lam_max <= 0.0:
        return np.ones_like(raw), 1.0
    floored = np.maximum(raw, ZERO_EIGENVALUE_REL * lam_max)
    smallest = float(floored.min())
    return floored / smallest, 1.0 / smallest


def eigendecompose(cov: CovarianceModel) -> EigenSystem:
    """Sorted, sign-fixed, clamped and rescaled spectrum (spectral.py:207-231)."""
    vals, vecs = jacobi_eigh(cov.cov)
    order = np.argsort(-vals, kind="stable")
    vals, vecs = vals[order], vecs[:, order]
    d = vals.shape[0]
    pivot = np.argmax(np.abs(vecs), axis=0)
    signs = np.sign(vecs[pivot, np.arange(d)])
    signs[signs == 0] = 1.0
    vecs = vecs * signs
    raw = np.maximum(vals, 0.0)
    scaled, factor = _scale_spectrum(raw)
    return EigenSystem(eigenvalues=scaled, eigenvectors=vecs, scale_factor=factor,
                       raw_eigenvalues=raw)


def allocate_eigensystem(eig: EigenSystem, d: int, n_subspaces: int,
                         subspace_dim: int) -> SubspaceAllocation:
    """Greedy min-log-product bucket assignment (spectral.py:234-265)."""
    if n_subspaces < 1 or subspace_dim < 1:
        raise ParameterError(f"need positive bucket counts, got {n_subspaces} x {subspace_dim}")
    if eig.dim != d:
        raise ParameterError(f"eigensystem has dimension {eig.dim}, expected {d}")
    retained = n_subspaces * subspace_dim
    if retained > d:
        raise ParameterError(
            f"capacity exceeded: {n_subspaces} subspaces of dimension {subspace_dim} "
            f"need {retained} eigenvectors, only {d} available")
    buckets = [[] for _ in range(n_subspaces)]
    logp = np.zeros(n_subspaces)
    for i in range(retained):
        target = -1
        for j in range(n_subspaces):
            if len(buckets[j]) < subspace_dim and (target < 0 or logp[j] < logp[target]):
                target = j
        buckets[target].append(i)
        logp[target] += math.log(eig.eigenvalues[i])
    return SubspaceAllocation(buckets=tuple(tuple(b) for b in buckets), log_products=logp)


def model_from_covariance(cov: CovarianceModel, d: int, n_subspaces: int,
                          subspace_dim: int) -> TransformModel:
    eig = eigendecompose(cov)
    alloc = allocate_eigensystem(eig, d, n_subspaces, subspace_dim)
    warnings = []
    retained = n_subspaces * subspace_dim
    lam_max = float(eig.raw_eigenvalues[0])
    rank = 0 if lam_max <= 0.0 else int((eig.raw_eigenvalues >= ZERO_EIGENVALUE_REL * lam_max).sum())
    if rank < retained:
        warnings.append(f"covariance rank {rank} is below the {retained} retained "
                        "directions; floored eigenvalues keep the allocation defined "
                        "but quality may degrade")
    blocks = tuple(np.ascontiguousarray(eig.eigenvectors[:, b], dtype=np.float32)
                   for b in alloc.buckets)
    return TransformModel(mean=cov.mean.astype(np.float32), blocks=blocks, warnings=tuple(warnings))


def fit_transform_model(data, n_subspaces: int, subspace_dim: int) -> TransformModel:
    """Fit covariance (GPU), eigendecompose, allocate, assemble the blocks."""
    X = np.asarray(data)
    if X.ndim != 2:
        raise ParameterError(f"expected a 2-D matrix, got shape {X.shape}")
    return model_from_covariance(fit_covariance(X), X.shape[1], n_subspaces, subspace_dim)


def transform_points(model: TransformModel, points) -> np.ndarray:
    """f32((f64 P - f64 mean) @ f64 M) on the GPU (spectral.py:301-316)."""
    P = np.asarray(points)
    if P.ndim != 2:
        raise ParameterError(f"expected a 2-D matrix, got shape {P.shape}")
    if P.shape[1] != model.d:
        raise DimensionMismatchError(
            f"points have dimension {P.shape[1]}, model expects {model.d}")
    P32 = as_f32_exact(P, "transform_points")
    M = np.ascontiguousarray(model.matrix, dtype=np.float32)
    mean = np.ascontiguousarray(model.mean, dtype=np.float32)
    out = np.empty((P.shape[0], M.shape[1]), np.float32)
    if P.shape[0]:
        nat.call("taco_transform_points", nat.device_id(), nat.ptr(mean), nat.ptr(M), model.d,
                 M.shape[1], nat.ptr(P32), P.shape[0], nat.ptr(out))
    return out
