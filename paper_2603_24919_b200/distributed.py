"""Point-sharded multi-GPU query path.

One process per GPU (torchrun), NCCL over NVLink/NVSwitch for the two
exchange steps of a query batch:

  1. every rank derives the SAME popped cells (replicated transform,
     codebooks and the GLOBAL cell-size table; global T = min(n, ceil(alpha n)))
     and counts only its own id range  -> per-query level histograms
  2. all_reduce(SUM) of the [nq, N_s+1] int64 histograms
  3. every rank runs the identical Alg. 5 (budget = beta * n_global) and
     reranks its local candidates -> local top-k (fp64 d2, global id)
  4. all_gather of the [nq, k] lists, merge on (d2, id) (lower id wins)

The per-rank compute is a ``ShardBackend``: ``CudaShardBackend`` drives
libtaco_b200.so (taco_query_count_device / taco_query_finish_device /
taco_topk_merge_device); tests substitute a CPU backend to exercise this
orchestration with gloo.  Results are bit-identical to the single-GPU path.

The build is replicated (every rank builds the full, deterministic index
and keeps its shard); a collective build is future work.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .engine import TacoIndex


def shard_range(n: int, rank: int, world: int):
    """GPU g owns [g*ceil(n/G), min(n, (g+1)*ceil(n/G)))."""
    per = math.ceil(n / world)
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


class _DeviceBytes:
    """Zero-copy handle on library-owned device memory (CUDA array interface)."""

    def __init__(self, ptr: int, rows: int, row_bytes: int):
        self.__cuda_array_interface__ = {"shape": (rows, row_bytes), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def _staged(t):
    """gloo cannot move CUDA tensors: stage them through host memory."""
    import torch.distributed as dist

    return t.is_cuda and dist.get_backend() == "gloo"


def _all_reduce(t, op, group=None):
    import torch.distributed as dist

    if _staged(t):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def _all_gather_into(out, inp, group=None):
    import torch.distributed as dist

    if _staged(out):
        h = out.cpu()
        dist.all_gather_into_tensor(h, inp.cpu().clone(), group=group)
        out.copy_(h)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


class CudaShardBackend:
    """One rank's shard on its GPU."""

    @classmethod
    def from_shard(cls, shard):
        """Wrap the device shard a collective build produced
        (distributed_build.sharded_build): its CSR, X, codebooks, transform and
        global cell sizes are already resident."""
        import torch

        self = cls.__new__(cls)
        self.torch = torch
        self.device = shard.backend.device
        self.k_sub = shard.params.n_subspaces
        self.dev = shard.backend.dev
        self.tile = int(nat.lib().taco_query_tile_size(self.dev.h))
        self.k2 = shard.params.clusters
        self.pop_cap = min(self.k2, 256)
        return self

    def __init__(self, index: TacoIndex, X_shard: np.ndarray, id_base: int, n_global: int, device: int):
        import torch

        self.torch = torch
        self.device = device
        p = index.params
        self.k_sub = p.n_subspaces
        n_local = X_shard.shape[0]
        self.dev = nat.DeviceIndex(n_local, index.d, p.n_subspaces, p.subspace_dim, p.clusters,
                                   p.kmeans_iters, device=device, n_global=n_global, id_base=id_base)
        M = np.ascontiguousarray(index.transform.matrix, dtype=np.float32)
        mean = np.ascontiguousarray(index.transform.mean, dtype=np.float32)
        nat.call("taco_index_set_transform", self.dev.h, nat.ptr(mean), nat.ptr(M))
        cb1 = np.ascontiguousarray(np.stack([s.codebook1.centroids for s in index.subspaces]), np.float32)
        cb2 = np.ascontiguousarray(np.stack([s.codebook2.centroids for s in index.subspaces]), np.float32)
        nat.call("taco_index_set_codebooks", self.dev.h, nat.ptr(cb1), nat.ptr(cb2))
        kp = p.codebook_size
        K2 = kp * kp
        gsizes = np.zeros((p.n_subspaces, K2), np.int64)
        offs = np.zeros((p.n_subspaces, K2 + 1), np.int64)
        ids = np.empty((p.n_subspaces, n_local), np.uint32)
        hi = id_base + n_local
        for j, sub in enumerate(index.subspaces):
            sizes = np.zeros(K2, np.int64)
            parts = []
            for key in sorted(sub.cells):
                v = np.asarray(sub.cells[key])
                c = key[0] * kp + key[1]
                gsizes[j, c] = v.size
                a, b = np.searchsorted(v, [id_base, hi])   # ids ascending inside a cell
                if b > a:
                    sizes[c] = b - a
                    parts.append((v[a:b] - id_base).astype(np.uint32))
            offs[j, 1:] = np.cumsum(sizes)
            ids[j] = np.concatenate(parts) if parts else np.empty(0, np.uint32)
        nat.call("taco_index_set_global_sizes", self.dev.h, nat.ptr(gsizes))
        nat.call("taco_index_set_cells", self.dev.h, nat.ptr(offs), nat.ptr(ids))
        Xs = np.ascontiguousarray(X_shard, dtype=np.float32)
        nat.call("taco_index_set_data", self.dev.h, nat.ptr(Xs))
        self.tile = int(nat.lib().taco_query_tile_size(self.dev.h))
        self.k2 = K2
        # popped cells per (query, subspace) slot: the all-gathered rows are
        # nq * N_s * pop_cap * 2 bytes, so start small (config 2 pops <= ~310)
        # and grow to the measured need (kept for later batches)
        self.pop_cap = min(K2, 256)

    def tile_size(self) -> int:
        return self.tile

    # ---- split traversal: each rank walks a slice of the tile's queries
    def front(self, Qt, alpha: float, lo: int, hi: int, rows: int) -> int:
        """Traverse queries [lo, hi) of the tile Qt into rows [lo, hi) of the
        pop buffers; returns the longest traversal if it exceeded the cap."""
        import ctypes
        need = ctypes.c_int64(0)
        nat.call("taco_query_front_device", self.dev.h, Qt.data_ptr(), Qt.shape[0], lo, hi, rows, float(alpha),
                 self.pop_cap, ctypes.byref(need), self._stream())
        return int(need.value)

    def front_async(self, Qt, alpha: float, lo: int, hi: int, rows: int):
        """As ``front`` without a host sync: returns a device int64[1] holding
        the slice's longest walk (checked once per batch by the caller)."""
        need = self.torch.zeros(1, dtype=self.torch.int64, device=f"cuda:{self.device}")
        nat.call("taco_query_front_async", self.dev.h, Qt.data_ptr(), Qt.shape[0], lo, hi, rows, float(alpha),
                 self.pop_cap, need.data_ptr(), self._stream())
        return need

    def raise_pop_cap(self, need: int) -> None:
        """Every rank gets the same all-reduced `need`, so caps stay equal."""
        self.pop_cap = min(self.k2, -(-(need + need // 4) // 64) * 64)

    def pop_views(self, rows: int):
        """uint8 views [rows, bytes per query] of the popped cells, their
        counts and retrieved sizes (rows are contiguous per query)."""
        import ctypes
        pp, pn, pr = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        cap = ctypes.c_int32(0)
        nat.call("taco_query_pop_buffers", self.dev.h, ctypes.byref(pp), ctypes.byref(pn), ctypes.byref(pr),
                 ctypes.byref(cap))
        dev = f"cuda:{self.device}"
        per_row = (2 * self.k_sub * cap.value, 4 * self.k_sub, 8 * self.k_sub)
        return [self.torch.as_tensor(_DeviceBytes(p.value, rows, b), device=dev)
                for p, b in zip((pp, pn, pr), per_row)]

    def count_popped(self, nq: int):
        hist = self.torch.empty((nq, self.k_sub + 1), dtype=self.torch.int64, device=f"cuda:{self.device}")
        nat.call("taco_query_count_popped_device", self.dev.h, nq, hist.data_ptr(), self._stream())
        return hist

    def _stream(self):
        return nat.torch_stream(self.torch, self.device)

    def count(self, Qt, alpha: float):
        torch = self.torch
        nq = Qt.shape[0]
        hist = torch.empty((nq, self.k_sub + 1), dtype=torch.int64, device=Qt.device)
        nat.call("taco_query_count_device", self.dev.h, Qt.data_ptr(), nq, float(alpha), hist.data_ptr(),
                 self._stream())
        return hist

    def finish(self, nq: int, ghist, beta: float, k: int):
        torch = self.torch
        dev = ghist.device
        d2 = torch.empty((nq, k), dtype=torch.float64, device=dev)
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        num = torch.empty(nq, dtype=torch.int64, device=dev)
        lvl = torch.empty(nq, dtype=torch.int32, device=dev)
        nat.call("taco_query_finish_device", self.dev.h, nq, ghist.data_ptr(), float(beta), int(k),
                 d2.data_ptr(), ids.data_ptr(), num.data_ptr(), lvl.data_ptr(), self._stream())
        return d2, ids, num, lvl

    def merge(self, d2_all, ids_all, k: int):
        torch = self.torch
        R, nq = d2_all.shape[0], d2_all.shape[1]
        out_i = torch.empty((nq, k), dtype=torch.int32, device=d2_all.device)
        out_d = torch.empty((nq, k), dtype=torch.float32, device=d2_all.device)
        nat.call("taco_topk_merge_device", R, nq, int(k), d2_all.data_ptr(), ids_all.data_ptr(),
                 out_i.data_ptr(), out_d.data_ptr(), self._stream())
        return out_i, out_d


def _split_count(backend, Qt, alpha: float, group=None):
    """Stage 1 with the replicated traversal divided by query: rank r walks
    rows [r*per, (r+1)*per) of the tile, an in-place all_gather gives every
    rank all popped cells (identical to walking them itself: the traversal
    reads only replicated state), then each rank counts its own ids.

    Returns (local histograms, the all-reduced longest walk as a device
    tensor): no host sync here; the caller checks the walks of the whole
    batch against the pop cap once (``sharded_query``)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m = Qt.shape[0]
    per = -(-m // world)
    rows = per * world
    lo, hi = min(m, rank * per), min(m, rank * per + per)
    need = backend.front_async(Qt, alpha, lo, hi, rows)
    _all_reduce(need, dist.ReduceOp.MAX, group)
    for buf in backend.pop_views(rows):
        _all_gather_into(buf, buf[rank * per:(rank + 1) * per], group)
    return backend.count_popped(m), need


def common_tile_size(backend, group=None, device=None) -> int:
    """The query tile every rank uses: the MIN of the ranks' own tile sizes
    (a rank's super-tile depends on its local chunk count, and the per-tile
    collectives must have equal shapes on every rank)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(backend.tile_size())], dtype=torch.int64, device=device)
    _all_reduce(t, dist.ReduceOp.MIN, group)
    return int(t.item())


def sharded_query(backend, Q, alpha: float, beta: float, k: int, group=None):
    """Batched k-ANN over a point-sharded index; every rank returns the full,
    identical result (ids int32 [nq,k], dists f32 [nq,k], cand_num, last_coll).

    One host sync per batch: the tiles' all-reduced longest walks are checked
    against the pop cap after the last tile; if any walk was truncated (rare:
    the cap adapts to the workload and is kept), every rank raises its cap to
    the same all-reduced need and the batch is re-run."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    nq = Q.shape[0]
    split = hasattr(backend, "front_async")
    T = getattr(backend, "common_tile", None)
    if T is None:
        T = common_tile_size(backend, group, Q.device)
        backend.common_tile = T
    for _attempt in range(2):
        outs, needs = [], []
        for q0 in range(0, nq, T):
            Qt = Q[q0:q0 + T]
            m = Qt.shape[0]
            if split:
                hist, need = _split_count(backend, Qt, alpha, group)
                needs.append(need)
            else:
                hist = backend.count(Qt, alpha)
            _all_reduce(hist, dist.ReduceOp.SUM, group)
            d2, ids, num, lvl = backend.finish(m, hist, beta, k)
            d2_all = torch.empty((world * m, k), dtype=d2.dtype, device=d2.device)
            ids_all = torch.empty((world * m, k), dtype=ids.dtype, device=ids.device)
            _all_gather_into(d2_all, d2.contiguous(), group)
            _all_gather_into(ids_all, ids.contiguous(), group)
            oi, od = backend.merge(d2_all.view(world, m, k), ids_all.view(world, m, k), k)
            outs.append((oi, od, num, lvl))
        if not needs:
            break
        longest = int(torch.cat(needs).max().item())   # the batch's one host sync
        if longest <= backend.pop_cap:
            break
        backend.raise_pop_cap(longest)   # same all-reduced value on every rank: caps stay equal
    cat = lambda i: torch.cat([o[i] for o in outs]) if outs else None  # noqa: E731
    return cat(0), cat(1), cat(2), cat(3)
