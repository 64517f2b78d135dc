"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/taco_b200.h declares, the native Jacobi sweeps (host code) are
bit-exact against the reference's golden eigensystems, parameter validation and
the v1 index-file parser behave like the reference."""

import hashlib
import re
import struct

import numpy as np
import pytest

from oracle import taco_oracle as O
from paper_2603_24919_b200 import _native as nat
from paper_2603_24919_b200 import engine as E
from paper_2603_24919_b200 import spectral as S
from paper_2603_24919_b200.errors import (ConvergenceError, CorruptionError, FormatError,
                                          ParameterError, UnsupportedVersionError)

HEADER = "include/taco_b200.h"


def test_library_exports_every_declared_symbol():
    decl = set(re.findall(r"^(?:int|int32_t|int64_t|const char\*|void\*)\s+(taco_\w+)\(",
                          open(HEADER).read(), flags=re.M))
    assert len(decl) >= 30
    lib = nat.lib()
    for name in decl:
        assert hasattr(lib, name), name
    assert set(nat.exported_symbols()) <= decl
    assert lib.taco_version() == 1


def test_native_jacobi_bit_exact(golden):
    u = golden("units")
    for c in range(6):
        w, V = S.jacobi_eigh(u[f"jac{c}_A"])
        np.testing.assert_array_equal(w, u[f"jac{c}_w"])
        np.testing.assert_array_equal(V, u[f"jac{c}_V"])


def test_native_jacobi_matches_oracle_on_covariances():
    rng = np.random.default_rng(3)
    for d in (4, 17, 64):
        X = rng.normal(size=(400, d)) @ rng.normal(size=(d, d))
        _, cov = O.fit_covariance(X.astype(np.float32))
        w, V = S.jacobi_eigh(cov)
        w0, V0, _ = O.jacobi(cov)
        np.testing.assert_array_equal(w, w0)
        np.testing.assert_array_equal(V, V0)


def test_jacobi_errors():
    with pytest.raises(ParameterError):
        S.jacobi_eigh(np.ones((2, 3)))
    with pytest.raises(ParameterError):
        S.jacobi_eigh(np.array([[1.0, 2.0], [0.0, 1.0]]))
    rng = np.random.default_rng(0)
    A = rng.normal(size=(12, 12))
    with pytest.raises(ConvergenceError):
        S.jacobi_eigh(A + A.T, max_sweeps=1)


def test_eigensystem_postprocessing_matches_oracle():
    rng = np.random.default_rng(5)
    X = (rng.normal(size=(500, 24)) @ rng.normal(size=(24, 24))).astype(np.float32)
    mu, cov = O.fit_covariance(X)
    eig = S.eigendecompose(S.CovarianceModel(mean=mu, cov=cov))
    scaled, V, raw = O.eigensystem(cov)
    np.testing.assert_array_equal(eig.eigenvalues, scaled)
    np.testing.assert_array_equal(eig.eigenvectors, V)
    alloc = S.allocate_eigensystem(eig, 24, 4, 5)
    buckets, logp = O.allocate(scaled, 4, 5)
    assert [list(b) for b in alloc.buckets] == buckets
    np.testing.assert_array_equal(alloc.log_products, logp)


def test_params_validation():
    with pytest.raises(ParameterError):
        E.IndexParams(n_subspaces=0, subspace_dim=4)
    with pytest.raises(ParameterError):
        E.IndexParams(n_subspaces=300, subspace_dim=4)
    with pytest.raises(ParameterError):
        E.IndexParams(n_subspaces=2, subspace_dim=4, clusters=10)
    with pytest.raises(ParameterError):
        E.QueryParams(alpha=0.0, beta=0.5)
    with pytest.raises(ParameterError):
        E.QueryParams(alpha=0.5, beta=1.0)
    with pytest.raises(ParameterError):
        E.QueryParams(alpha=0.5, beta=0.5, k=0)


def test_v1_parser_matches_reference_bytes(golden):
    blob = golden("rig1")["blob"].tobytes()
    idx = E._parse(blob, "rig1")
    assert E.serialize_index(idx) == blob
    ref = O.deserialize(blob)
    for j in range(idx.params.n_subspaces):
        assert sorted(idx.subspaces[j].cells) == sorted(ref.cells[j])


@pytest.mark.parametrize("mutate,exc", [
    (lambda b: b[: len(b) // 2], CorruptionError),
    (lambda b: b[:100] + bytes([b[100] ^ 0xFF]) + b[101:], CorruptionError),
    (lambda b: b[:4] + struct.pack("<H", 99) + b[6:], UnsupportedVersionError),
    (lambda b: b"OOPS" + b[4:], FormatError),
    (lambda b: b[:8], CorruptionError),
])
def test_v1_parser_rejects(golden, mutate, exc):
    blob = golden("rig1")["blob"].tobytes()
    with pytest.raises(exc):
        E._parse(mutate(blob), "bad")


def test_v1_parser_trailing_bytes(golden):
    blob = golden("rig1")["blob"].tobytes()
    body = blob[:-8] + b"\0\0\0\0"
    bad = body + hashlib.blake2b(body, digest_size=8).digest()
    with pytest.raises(CorruptionError):
        E._parse(bad, "trailing")
