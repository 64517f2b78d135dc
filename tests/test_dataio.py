"""fvecs/ivecs ingest (CPU) and the GPU exact ground truth vs the oracle
(dataio.py:36-187)."""

import struct

import numpy as np
import pytest

import paper_2603_24919_b200 as T
from oracle import taco_oracle as O
from paper_2603_24919_b200.errors import DimensionMismatchError, EmptyInputError, FormatError, ParameterError


@pytest.mark.parametrize("kind,dtype", [("float32", np.float32), ("int32", np.int32)])
def test_round_trip_bit_exact(tmp_path, kind, dtype):
    rng = np.random.default_rng(3)
    m = rng.normal(size=(23, 7)).astype(dtype) if kind == "float32" else rng.integers(-9, 9, (23, 7)).astype(dtype)
    p = tmp_path / "m.vecs"
    T.write_vectors(m, p, kind)
    back = T.read_vectors(p, kind)
    assert back.dtype == dtype and back.shape == m.shape
    assert back.tobytes() == m.tobytes()
    # layout: int32 dim then the elements
    raw = p.read_bytes()
    assert struct.unpack_from("<i", raw, 0)[0] == 7 and len(raw) == 23 * 32


def test_read_errors(tmp_path):
    p = tmp_path / "x.fvecs"
    p.write_bytes(b"")
    with pytest.raises(EmptyInputError):
        T.read_vectors(p)
    p.write_bytes(b"\x01\x00")
    with pytest.raises(FormatError, match="byte offset 0"):
        T.read_vectors(p)
    good = struct.pack("<i", 2) + struct.pack("<2f", 1.0, 2.0)
    p.write_bytes(good + good[:6])
    with pytest.raises(FormatError, match="truncated record at byte offset 12"):
        T.read_vectors(p)
    p.write_bytes(good + struct.pack("<i", 3) + struct.pack("<2f", 1.0, 2.0))
    with pytest.raises(FormatError, match="record 1 .byte offset 12. declares dimension 3"):
        T.read_vectors(p)
    p.write_bytes(struct.pack("<i", 0))
    with pytest.raises(FormatError, match="invalid dimension 0"):
        T.read_vectors(p)
    with pytest.raises(ParameterError):
        T.read_vectors(p, "float64")


def test_sampling_and_split():
    m = np.arange(40, dtype=np.float32).reshape(20, 2)
    rows, ids = T.sample_subset(m, 5, 7)
    np.testing.assert_array_equal(rows, m[ids])
    assert len(set(ids.tolist())) == 5
    base, q, qid = T.split_queries(m, 4, 9)
    assert base.shape == (16, 2) and q.shape == (4, 2)
    np.testing.assert_array_equal(q, m[qid])
    with pytest.raises(ParameterError):
        T.split_queries(m, 20, 1)
    with pytest.raises(ParameterError):
        T.sample_subset(m, 0, 1)


def test_ground_truth_validation():
    X = np.zeros((5, 3), np.float32)
    with pytest.raises(DimensionMismatchError):
        T.compute_ground_truth(X, np.zeros((2, 4), np.float32), 1)
    with pytest.raises(ParameterError):
        T.compute_ground_truth(X, np.zeros((2, 3), np.float32), 6)


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,nq,k,ints", [(5000, 32, 40, 10, False), (3000, 128, 33, 100, True),
                                           (2000, 37, 20, 7, False), (1500, 960, 5, 10, False)])
def test_gpu_ground_truth_matches_oracle(n, d, nq, k, ints):
    rng = np.random.default_rng(n + d)
    if ints:   # integer data: many exact distance ties -> id order decides
        X = rng.integers(0, 4, (n, d)).astype(np.float32)
        Q = rng.integers(0, 4, (nq, d)).astype(np.float32)
    else:
        X = rng.standard_normal((n, d)).astype(np.float32)
        Q = rng.standard_normal((nq, d)).astype(np.float32)
    gt = T.compute_ground_truth(X, Q, k)
    oi, od = O.ground_truth(X, Q, k)
    np.testing.assert_array_equal(gt.ids, oi)
    np.testing.assert_array_equal(gt.dists, od)


@pytest.mark.gpu
def test_gpu_ground_truth_resident_index():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((4000, 16)).astype(np.float32)
    Q = rng.standard_normal((10, 16)).astype(np.float32)
    idx = T.build_index(X, T.IndexParams(2, 8, 16, 5, 0))
    a = T.compute_ground_truth(X, Q, 10, index=idx)
    b = T.compute_ground_truth(X, Q, 10)
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dists, b.dists)


@pytest.mark.gpu
def test_gpu_ground_truth_matches_reference_golden(golden):
    """The GPU exact k-NN against dataio.compute_ground_truth's own outputs
    (tests/golden/groundtruth.npz, made by running the reference)."""
    g = golden("groundtruth")
    for ci, (n, d, nq, k, ints) in enumerate(g["cases"].tolist()):
        rng = np.random.default_rng(n + d)
        if ints:
            X = rng.integers(0, 4, (n, d)).astype(np.float32)
            Q = rng.integers(0, 4, (nq, d)).astype(np.float32)
        else:
            X = rng.standard_normal((n, d)).astype(np.float32)
            Q = rng.standard_normal((nq, d)).astype(np.float32)
        gt = T.compute_ground_truth(X, Q, k)
        np.testing.assert_array_equal(gt.ids, g[f"ids_{ci}"])
        np.testing.assert_array_equal(gt.dists, g[f"dists_{ci}"])
