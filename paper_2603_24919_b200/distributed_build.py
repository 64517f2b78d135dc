"""Point-sharded collective index build (build collectives).

Each rank holds only its own contiguous rows X[lo, hi) (shards start on
multiples of the Gram block, ``aligned_shard_range``) and the ranks build the
index together; the result is bit-identical to the single-GPU
``build_index`` on the whole matrix:

  1. column mean (spectral.py:107, numpy's sequential per-column add): a
     RANK-ORDERED CHAIN -- rank r continues the running fp64 sums it receives
     from rank r-1 (``taco_shard_colsum``), the last rank's sums are broadcast
     and divided by n;  non-finite rows are reported globally (all-reduce MIN);
  2. centred Gram (spectral.py:108-109): the same chain over fixed blocks of
     rows (``taco_shard_gram``; the single-GPU build sums the same block
     partials in the same order);
  3. eigensolve + allocation on the host, replicated (identical inputs);
  4. transform of the local rows (local, T dimension-major);
  5. k-means (clustering.py:57-115): the 2*N_s halves are independent, so
     rank q OWNS a contiguous range of subspaces and runs the single-GPU
     k-means on them over all n points.  An all-to-all moves the transformed
     columns to their owners (each value moves once: n*D*4 bytes in total
     over NVLink), then the labels back to the point owners;
  6. cells (imi.py:70-81): each rank builds the CSR of its own rows; the
     per-cell sizes are all-reduced (SUM) into the global size table the
     traversal reads.

Codebooks, inertia histories and the transform are replicated (a few MB).
``Comm`` wraps torch.distributed: NCCL moves device tensors directly; with
gloo (CPU tests, the one-GPU two-process emulation) CUDA tensors are staged
through host memory.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import NumericError, ParameterError


def aligned_shard_range(n: int, rank: int, world: int, block: int):
    """Contiguous shard of rank r whose start is a multiple of ``block`` rows
    (the Gram chain's block), as equal as that allows."""
    per = -(-max(-(-n // world), 1) // block) * block
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def owned_subspaces(n_sub: int, rank: int, world: int):
    """Subspaces whose two k-means halves rank r runs (contiguous, in order)."""
    return [j for j in range(n_sub) if j * world // n_sub == rank]


class Comm:
    """The collectives the sharded build uses, over torch.distributed."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.gloo = dist.get_backend(group) == "gloo"

    def _out(self, t):
        return t.cpu() if (self.gloo and t.is_cuda) else t

    def _back(self, t, like):
        return t.to(like.device) if t.device != like.device else t

    def chain(self, fn, like):
        """Rank-ordered chain: rank r gets rank r-1's carry (None on rank 0),
        returns fn(carry); the last rank's result is broadcast to all."""
        torch, dist = self.torch, self.dist
        carry = None
        if self.rank > 0:
            buf = self._out(torch.empty_like(like))
            dist.recv(buf, src=self._global(self.rank - 1), group=self.group)
            carry = buf.cpu().numpy()
        out = np.ascontiguousarray(fn(carry))
        res = self._out(torch.from_numpy(out).to(like.device))
        if self.rank < self.world - 1:
            dist.send(res, dst=self._global(self.rank + 1), group=self.group)
        dist.broadcast(res, src=self._global(self.world - 1), group=self.group)
        return res.cpu().numpy()

    def _global(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def all_reduce(self, t, op="sum"):
        d = self.dist
        x = self._out(t)
        d.all_reduce(x, op={"sum": d.ReduceOp.SUM, "min": d.ReduceOp.MIN, "max": d.ReduceOp.MAX}[op],
                     group=self.group)
        return self._back(x, t)

    def all_to_all(self, send, recv_shapes, like):
        """send[q]: tensor for rank q (any shape, contiguous); returns the
        tensors received from every rank, shaped recv_shapes[r]."""
        torch = self.torch
        inp = self._out(torch.cat([s.reshape(-1) for s in send]) if send else torch.empty(0, dtype=like.dtype))
        in_split = [int(s.numel()) for s in send]
        out_split = [int(math.prod(sh)) for sh in recv_shapes]
        out = torch.empty(sum(out_split), dtype=like.dtype, device=inp.device)
        self.dist.all_to_all_single(out, inp.contiguous(), out_split, in_split, group=self.group)
        out = self._back(out, like)
        parts, o = [], 0
        for sh, c in zip(recv_shapes, out_split):
            parts.append(out[o:o + c].view(*sh))
            o += c
        return parts

    def all_gather_object(self, obj):
        res = [None] * self.world
        self.dist.all_gather_object(res, obj, group=self.group)
        return res


class ShardIndex:
    """One rank's part of a point-sharded index: its device shard (local CSR
    over rows [id_base, id_base + n_local), X and the replicated transform,
    codebooks and global cell sizes) plus the replicated host-side model."""

    def __init__(self, params, transform, codebooks, histories, n_global, id_base, n_local, backend):
        self.params = params
        self.transform = transform
        self.codebooks = codebooks          # [(cb1, cb2)] per subspace, f32
        self.histories = histories          # [(hist1, hist2)] per subspace
        self.n = n_global
        self.id_base = id_base
        self.n_local = n_local
        self.backend = backend
        self.metadata = {}

    @property
    def d(self):
        return self.transform.d


def sharded_build(backend, params, n_global: int, comm: Comm | None = None) -> ShardIndex:
    """Build the index collectively; every rank calls this with its backend
    (its rows already resident).  Returns the rank's ShardIndex."""
    import torch

    from .spectral import covariance_from_gram, model_from_covariance

    comm = comm or Comm()
    rank, world = comm.rank, comm.world
    d, n_local, id_base = backend.d, backend.n_local, backend.id_base
    n_sub, s = params.n_subspaces, params.subspace_dim
    block = backend.gram_block_rows()
    lo, hi = aligned_shard_range(n_global, rank, world, block)
    if hi <= lo:
        raise ParameterError(f"rank {rank} of {world} gets no rows of {n_global} (blocks of {block})")
    if (lo, hi) != (id_base, id_base + n_local):
        raise ParameterError(f"rank {rank} holds rows [{id_base}, {id_base + n_local}), the build shards "
                             f"as [{lo}, {hi}) (aligned_shard_range, block {block})")
    like_d = torch.zeros(d, dtype=torch.float64, device=backend.comm_device)
    like_dd = torch.zeros((d, d), dtype=torch.float64, device=backend.comm_device)

    # 1. column sums: rank-ordered chain, then the global non-finite check
    bad = [None]

    def colsum(carry):
        out, b = backend.colsum(carry)
        bad[0] = b
        return out

    sums = comm.chain(colsum, like_d)
    b = torch.tensor([bad[0] + id_base if bad[0] >= 0 else np.iinfo(np.int64).max], dtype=torch.int64,
                     device=backend.comm_device)
    b = int(comm.all_reduce(b, "min").item())
    if b != np.iinfo(np.int64).max:
        raise NumericError(f"non-finite value in row {b}")
    mean = sums / float(n_global)                      # numpy mean: sum / n (fp64)

    # 2. centred Gram: the same chain over the fixed row blocks
    gram = comm.chain(lambda carry: backend.gram(mean, block, carry), like_dd)

    # 3. eigensolve + allocation (host, replicated)
    model = model_from_covariance(covariance_from_gram(mean, gram, n_global), d, n_sub, s)

    # 4. local transform (dimension-major [D][n_local])
    T_loc = backend.transform(model)
    D = n_sub * s

    # 5. transformed columns to the subspace owners, k-means there, labels back
    owned = [owned_subspaces(n_sub, q, world) for q in range(world)]
    ranges = [aligned_shard_range(n_global, r, world, block) for r in range(world)]
    sizes = [h - l for l, h in ranges]
    send = [T_loc[owned[q][0] * s:(owned[q][-1] + 1) * s].contiguous() if owned[q] else T_loc[:0]
            for q in range(world)]
    mine = owned[rank]
    Dq = len(mine) * s
    parts = comm.all_to_all(send, [(Dq, sizes[r]) for r in range(world)], T_loc)
    res = None
    if mine:
        T_cols = torch.cat(parts, dim=1).contiguous()          # [Dq][n_global]
        res = backend.kmeans(mine, T_cols, n_global, params)
        labels_all = res["labels"]                             # [2|mine|][n_global] i32
    else:
        labels_all = torch.zeros((0, n_global), dtype=torch.int32, device=T_loc.device)
    send = [labels_all[:, ranges[r][0]:ranges[r][1]].contiguous() for r in range(world)]
    got = comm.all_to_all(send, [(2 * len(owned[q]), n_local) for q in range(world)], labels_all)
    labels_loc = torch.cat(got, dim=0).contiguous()            # [2 N_s][n_local], subspace order
    info = comm.all_gather_object(None if res is None else
                                  {"subspaces": mine, "cb": res["codebooks"], "hist": res["histories"]})
    codebooks, histories = [None] * n_sub, [None] * n_sub
    for ent in info:
        if ent is None:
            continue
        for jj, j in enumerate(ent["subspaces"]):
            codebooks[j] = ent["cb"][jj]
            histories[j] = ent["hist"][jj]

    # 6. local CSR + global cell sizes (all-reduce SUM)
    local_sizes = backend.finish(codebooks, labels_loc)
    gs = comm.all_reduce(torch.as_tensor(local_sizes).to(backend.comm_device), "sum")
    backend.set_global_sizes(gs.cpu().numpy())
    out = ShardIndex(params, model, codebooks, histories, n_global, id_base, n_local, backend)
    out.metadata["warnings"] = list(model.warnings)
    return out


def gather_serialized(index: ShardIndex, comm: Comm | None = None):
    """The whole index in the v1 file format (engine.py:345-384), assembled on
    every rank from the shards' local cells (global id = id_base + local id;
    shards are ordered, so each cell's ids stay ascending)."""
    from .clustering import KMeansModel
    from .engine import TacoIndex, serialize_index
    from .imi import InvertedMultiIndex

    comm = comm or Comm()
    p = index.params
    kp = p.codebook_size
    local = index.backend.local_cells()                     # per subspace (offsets[K2+1], ids)
    allc = comm.all_gather_object([(off, ids.astype(np.int64) + index.id_base) for off, ids in local])
    subs = []
    for j in range(p.n_subspaces):
        cells = {}
        for c in range(kp * kp):
            pieces = [ids[off[c]:off[c + 1]] for off, ids in (rk[j] for rk in allc) if off[c + 1] > off[c]]
            if pieces:
                cells[(c // kp, c % kp)] = np.concatenate(pieces).astype(np.uint32)
        cb1, cb2 = index.codebooks[j]
        subs.append(InvertedMultiIndex(codebook1=KMeansModel(cb1, None), codebook2=KMeansModel(cb2, None),
                                       cells=cells, codebook_size=kp, split=(p.subspace_dim + 1) // 2))
    full = TacoIndex(params=p, transform=index.transform, subspaces=subs, n=index.n)
    return serialize_index(full)


class CudaShardBuilder:
    """One rank's build backend on its GPU (libtaco_b200.so)."""

    def __init__(self, X_local: np.ndarray, id_base: int, n_global: int, params, device: int = 0):
        import torch

        from . import _native as nat

        self.torch, self.nat = torch, nat
        self.device = device
        self.comm_device = f"cuda:{device}"
        self.X = np.ascontiguousarray(X_local, dtype=np.float32)
        self.n_local, self.d = self.X.shape
        self.id_base, self.n_global, self.params = id_base, n_global, params
        p = params
        self.dev = nat.DeviceIndex(self.n_local, self.d, p.n_subspaces, p.subspace_dim, p.clusters,
                                   p.kmeans_iters, device=device, n_global=n_global, id_base=id_base)
        nat.call("taco_index_set_data", self.dev.h, nat.ptr(self.X))
        self.kdev = None

    def gram_block_rows(self) -> int:
        return int(self.nat.lib().taco_gram_block_rows())

    def colsum(self, carry):
        nat = self.nat
        out = np.empty(self.d)
        bad = np.zeros(1, np.int64)
        cin = None if carry is None else np.ascontiguousarray(carry, dtype=np.float64)
        nat.call("taco_shard_colsum", self.dev.h, nat.ptr(cin), nat.ptr(out), nat.ptr(bad))
        return out, int(bad[0])

    def gram(self, mean, block, carry):
        nat = self.nat
        out = np.empty((self.d, self.d))
        cin = None if carry is None else np.ascontiguousarray(carry, dtype=np.float64)
        nat.call("taco_shard_gram", self.dev.h, nat.ptr(np.ascontiguousarray(mean)), int(block), nat.ptr(cin),
                 nat.ptr(out))
        return out

    def transform(self, model):
        nat, torch = self.nat, self.torch
        M = np.ascontiguousarray(model.matrix, dtype=np.float32)
        nat.call("taco_index_set_transform", self.dev.h, nat.ptr(np.ascontiguousarray(model.mean, np.float32)),
                 nat.ptr(M))
        nat.call("taco_transform_data", self.dev.h)
        D = M.shape[1]
        T = torch.empty((D, self.n_local), dtype=torch.float32, device=self.comm_device)
        nat.call("taco_get_transformed_device", self.dev.h, T.data_ptr())
        return T

    def kmeans(self, subspaces, T_cols, n_global, params):
        """The single-GPU k-means (all halves of the owned subspaces at once)
        over all n_global points, seeds of the GLOBAL subspace numbers."""
        from .imi import run_kmeans_all
        from .seeding import derive_seed

        nat, torch = self.nat, self.torch
        p = params
        ns = len(subspaces)
        s = p.subspace_dim
        self.kdev = nat.DeviceIndex(n_global, ns * s, ns, s, p.clusters, p.kmeans_iters, device=self.device)
        nat.call("taco_index_set_transformed_device", self.kdev.h, T_cols.data_ptr())
        models = run_kmeans_all(self.kdev, n_global, ns, s, p.codebook_size, p.kmeans_iters,
                                lambda j, h: derive_seed(derive_seed(p.seed, subspaces[j]), h))
        lab = torch.empty((2 * ns, n_global), dtype=torch.int32, device=self.comm_device)
        nat.call("taco_get_labels_device", self.kdev.h, lab.data_ptr())
        cbs = [(m1.centroids, m2.centroids) for m1, m2 in models]
        hist = [(m1.inertia_history, m2.inertia_history) for m1, m2 in models]
        return {"labels": lab, "codebooks": cbs, "histories": hist}

    def finish(self, codebooks, labels_loc):
        nat = self.nat
        p = self.params
        self.kdev = None   # the owner-side k-means state is no longer needed
        cb1 = np.ascontiguousarray(np.stack([c[0] for c in codebooks]), np.float32)
        cb2 = np.ascontiguousarray(np.stack([c[1] for c in codebooks]), np.float32)
        nat.call("taco_index_set_codebooks", self.dev.h, nat.ptr(cb1), nat.ptr(cb2))
        nat.call("taco_index_set_labels_device", self.dev.h, labels_loc.data_ptr())
        nat.call("taco_build_cells", self.dev.h)
        sizes = np.zeros((p.n_subspaces, p.clusters), np.int64)
        nat.call("taco_get_local_sizes", self.dev.h, nat.ptr(sizes))
        return sizes

    def set_global_sizes(self, sizes):
        self.nat.call("taco_index_set_global_sizes", self.dev.h, self.nat.ptr(np.ascontiguousarray(sizes, np.int64)))

    def local_cells(self):
        nat = self.nat
        p = self.params
        out = []
        for j in range(p.n_subspaces):
            off = np.empty(p.clusters + 1, np.int64)
            ids = np.empty(self.n_local, np.uint32)
            nat.call("taco_get_cells", self.dev.h, j, nat.ptr(off), nat.ptr(ids))
            out.append((off, ids))
        return out
