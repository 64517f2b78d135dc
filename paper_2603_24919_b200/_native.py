"""ctypes binding of libtaco_b200.so (the C ABI in include/taco_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA
device is usable, every entry point raises.  ``build()`` in
``__graft_entry__`` (or ``make -C paper_2603_24919_b200/csrc``) produces the
library next to this file.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtaco_b200.so")
# experiments only: a variant build of the same library (tools/variants.sh)
if os.environ.get("TACO_LIB_VARIANT"):
    LIB_PATH = os.path.abspath(os.environ["TACO_LIB_VARIANT"])

_c_int, _c_i32, _c_i64, _c_dbl, _vp = ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "taco_last_error": [],
    "taco_version": [],
    "taco_launch_count": [],
    "taco_index_create": [_c_int, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i64, _c_i64,
                          ctypes.POINTER(_vp)],
    "taco_index_destroy": [_vp],
    "taco_index_set_data": [_vp, _vp],
    "taco_index_set_data_device": [_vp, _vp],
    "taco_index_row_format": [_vp],
    "taco_index_layout": [_vp, _vp, _vp, _vp],
    "taco_fit_covariance": [_vp, _vp, _vp, _vp],
    "taco_covariance": [_c_int, _vp, _c_i64, _c_i32, _vp, _vp, _vp],
    "taco_jacobi_sweeps": [_vp, _vp, _c_i32, _c_dbl, _c_i32, _vp, _vp],
    "taco_device_count": [],
    "taco_jacobi_sweeps_device": [_c_int, _vp, _vp, _c_i32, _c_dbl, _c_i32, _vp, _vp],
    "taco_index_set_transform": [_vp, _vp, _vp],
    "taco_transform_data": [_vp],
    "taco_index_set_transformed": [_vp, _vp],
    "taco_kmeans_all": [_vp, _vp, _vp, _vp, _vp],
    "taco_build_cells": [_vp],
    "taco_index_set_codebooks": [_vp, _vp, _vp],
    "taco_index_set_labels": [_vp, _vp, _vp],
    "taco_index_set_cells": [_vp, _vp, _vp],
    "taco_index_set_global_sizes": [_vp, _vp],
    "taco_get_codebooks": [_vp, _vp, _vp],
    "taco_get_labels": [_vp, _vp, _vp],
    "taco_get_history": [_vp, _vp, _vp],
    "taco_get_cells": [_vp, _c_i32, _vp, _vp],
    "taco_get_transformed": [_vp, _vp],
    "taco_get_global_sizes": [_vp, _vp],
    "taco_get_local_sizes": [_vp, _vp],
    "taco_query_batch": [_vp, _vp, _c_i64, _c_dbl, _c_dbl, _c_i32, _vp, _vp, _vp, _vp],
    "taco_query_batch_device": [_vp, _vp, _c_i64, _c_dbl, _c_dbl, _c_i32, _vp, _vp, _vp, _vp, _vp],
    "taco_query_count_device": [_vp, _vp, _c_i64, _c_dbl, _vp, _vp],
    "taco_query_front_device": [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_dbl, _c_i32, _vp, _vp],
    "taco_query_front_async": [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_dbl, _c_i32, _vp, _vp],
    "taco_query_pop_buffers": [_vp, _vp, _vp, _vp, _vp],
    "taco_query_count_popped_device": [_vp, _c_i64, _vp, _vp],
    "taco_query_finish_device": [_vp, _c_i64, _vp, _c_dbl, _c_i32, _vp, _vp, _vp, _vp, _vp],
    "taco_query_tile_size": [_vp],
    "taco_topk_merge_device": [_c_i32, _c_i64, _c_i32, _vp, _vp, _vp, _vp, _vp],
    "taco_ground_truth": [_c_int, _vp, _c_i64, _c_i32, _vp, _c_i64, _c_i32, _vp, _vp],
    "taco_ground_truth_index": [_vp, _vp, _c_i64, _c_i32, _vp, _vp],
    "taco_sc_linear_scores": [_c_int, _vp, _c_i64, _c_i32, _c_i32, _vp, _c_dbl, _vp],
    "taco_sc_linear_scores_index": [_vp, _vp, _c_dbl, _vp],
    "taco_count_scores": [_vp, _vp, _c_dbl, _vp],
    "taco_activation_trace": [_vp, _vp, _c_i32, _c_dbl, _c_i32, _vp, _vp, _vp, _vp],
    "taco_select_candidates": [_c_int, _vp, _c_i64, _c_i32, _c_dbl, _vp, _vp, _vp],
    "taco_rerank": [_c_int, _vp, _c_i64, _c_i32, _vp, _vp, _c_i64, _c_i32, _vp, _vp, _vp],
    "taco_centroid_order": [_c_int, _vp, _vp, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp],
    "taco_traverse": [_c_int, _c_i32, _vp, _vp, _vp, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp],
    "taco_transform_points": [_c_int, _vp, _vp, _c_i32, _c_i32, _vp, _c_i64, _vp],
    "taco_debug_force_replay": [_c_int],
    "taco_profile_enable": [_c_int],
    "taco_profile_read": [_vp, _vp, _vp, _c_int],
    "taco_profile_name": [_c_int],
    "taco_profile_kernels": [],
    "taco_index_stream": [_vp],
    "taco_shard_colsum": [_vp, _vp, _vp, _vp],
    "taco_shard_gram": [_vp, _vp, _c_i64, _vp, _vp],
    "taco_gram_block_rows": [],
    "taco_index_set_transformed_device": [_vp, _vp],
    "taco_get_transformed_device": [_vp, _vp],
    "taco_get_labels_device": [_vp, _vp],
    "taco_index_set_labels_device": [_vp, _vp],
    "taco_kmeans": [_c_int, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_i64, _vp, _vp, _vp, _vp, _vp,
                    _vp, _vp],
}
_RESTYPES = {"taco_last_error": ctypes.c_char_p, "taco_launch_count": _c_i64,
             "taco_profile_name": ctypes.c_char_p, "taco_index_stream": _vp}

_CODES = {
    1: errors.ParameterError,
    2: errors.DimensionMismatchError,
    3: errors.InsufficientDataError,
    4: errors.NumericError,
    5: errors.ConvergenceError,
    6: errors.StateError,
    7: errors.DeviceError,
    8: errors.FormatError,
}

_lib = None


def lib():
    """Load (once) and return the native library; raise if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the CUDA path has no CPU fallback)")
        h = ctypes.CDLL(LIB_PATH)
        for name, argt in _SIGS.items():
            fn = getattr(h, name)
            fn.argtypes = argt
            fn.restype = _RESTYPES.get(name, _c_int)
        _lib = h
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def check(rc: int):
    if rc != 0:
        msg = lib().taco_last_error().decode(errors="replace")
        raise _CODES.get(rc, errors.TacoError)(msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("native call needs a C-contiguous array")
    return a.ctypes.data


def gpu_available() -> bool:
    """True when the library sees at least one CUDA device."""
    return int(lib().taco_device_count()) > 0


def device_id() -> int:
    """CUDA device for new indexes: $TACO_DEVICE, else $LOCAL_RANK, else 0."""
    for key in ("TACO_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(key)
        if v not in (None, ""):
            return int(v)
    return 0


def index_layout(h):
    """(ids per chunk, chunks, cluster mode) of a device index (taco_index_layout)."""
    chunk, nch, cm = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int32(0)
    call("taco_index_layout", h, ctypes.byref(chunk), ctypes.byref(nch), ctypes.byref(cm))
    return int(chunk.value), int(nch.value), bool(cm.value)


def launch_count() -> int:
    return int(lib().taco_launch_count())


class DeviceIndex:
    """Owner of one ``taco_index*`` (a point shard resident on one GPU)."""

    def __init__(self, n, d, n_sub, s, clusters, iters, device=None, n_global=None, id_base=0):
        self.device = device_id() if device is None else int(device)
        out = ctypes.c_void_p()
        call("taco_index_create", self.device, int(n), int(d), int(n_sub), int(s), int(clusters),
             int(iters), int(n if n_global is None else n_global), int(id_base), ctypes.byref(out))
        self.h = out
        self.n, self.d, self.n_sub, self.s, self.clusters = int(n), int(d), int(n_sub), int(s), int(clusters)
        self.kprime = int(round(clusters ** 0.5))
        self.data_key = None

    def close(self):
        if getattr(self, "h", None):
            lib().taco_index_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def profile_enable(on: bool):
    check(lib().taco_profile_enable(1 if on else 0))


def profile_read(reset=True):
    """{kernel: (total_ms, launches)}, stats dict."""
    nk = lib().taco_profile_kernels()
    ms = np.zeros(nk)
    cnt = np.zeros(nk, np.int64)
    st = np.zeros(7, np.int64)
    check(lib().taco_profile_read(ptr(ms), ptr(cnt), ptr(st), 1 if reset else 0))
    names = [lib().taco_profile_name(i).decode() for i in range(nk)]
    keys = ("sum_retrieved", "sum_candidates", "sum_pops", "queries", "tiles", "score_bytes", "max_pops")
    return {n: (float(m), int(c)) for n, m, c in zip(names, ms, cnt)}, dict(zip(keys, map(int, st)))


CUDA_STREAM_LEGACY = 0x1   # cudaStreamLegacy


def torch_stream(torch, device=None) -> int:
    """Handle of torch's current stream for the C ABI.  torch reports the legacy
    default stream as 0, which the C ABI reads as "the index's own stream";
    map it to cudaStreamLegacy so library work is ordered with torch's."""
    h = torch.cuda.current_stream(device).cuda_stream
    return h if h else CUDA_STREAM_LEGACY
