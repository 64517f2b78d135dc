"""Config-scale parity of the GPU path against the CPU oracle (run on the GPU box).

    python tools/parity_configs.py --configs 1,2,3,4 --out gpurun_out/parity.json

For each BASELINE config (SURVEY 8(d) generator, seeded):
  * GPU build (build_index) and the whole query batch through the public
    batched API (knn_query_batch);
  * the oracle (oracle/taco_oracle.py, the numpy restatement pinned to the
    reference's golden vectors) answers the same queries on the GPU-built
    index (v1 bytes), on all host cores; ids, distances, candidate_num and
    last_collision are compared query by query;
  * the query transform: the reference transforms ONE query at a time
    (engine.py:208 -> a 1-row matmul, OpenBLAS dgemv order); the GPU
    transforms the batch with an fp64 FMA chain.  The script counts f32
    coordinates that differ and, for every query with a flip, whether the
    flip changed any subspace's popped-cell sequence (oracle traversal with
    both transforms);
  * config 1 only (--oracle-build): the oracle BUILD from the raw data (about
    20 s), compared with the GPU build byte for byte (v1 file); when the
    transform blocks differ in a few ulps, the stages after it are compared
    given the GPU's transform (k-means centroids, labels, cells).

The oracle here is the checker, never the thing measured.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def qt_flip_check(O, index, Q, qt_gpu, alpha, threads):
    """Per-query (reference-order) transform vs the GPU batch transform; for
    queries with a flipped coordinate, compare the popped-cell sequences."""
    from concurrent.futures import ThreadPoolExecutor

    oidx = index
    mean, blocks = oidx.mean, oidx.blocks
    nq = Q.shape[0]
    flips = np.zeros(nq, np.int64)

    def one(r):
        flips[r] = int((O.transform(mean, blocks, Q[r][None, :])[0] != qt_gpu[r]).sum())

    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(one, range(nq)))
    flipped = np.flatnonzero(flips)
    pop_diff = 0
    s, kp, sp = oidx.s, oidx.kprime, oidx.split
    for r in flipped:
        qr = O.transform(mean, blocks, Q[r][None, :])[0]
        for j in range(oidx.n_sub):
            cells = oidx.cells[j]
            size = (lambda a, b, cells=cells: cells[(a, b)].size if (a, b) in cells else 0)
            pa, _ = O.traverse(alpha, oidx.n, kp, *O.centroid_order(oidx.cb1[j], oidx.cb2[j], qr[j * s:(j + 1) * s], sp), size)
            pb, _ = O.traverse(alpha, oidx.n, kp, *O.centroid_order(oidx.cb1[j], oidx.cb2[j], qt_gpu[r][j * s:(j + 1) * s], sp), size)
            if [(a, b) for _, a, b in pa] != [(a, b) for _, a, b in pb]:
                pop_diff += 1
    return {"coords": int(nq * qt_gpu.shape[1]), "flipped_coords": int(flips.sum()),
            "queries_with_flip": int(flipped.size), "subspace_pop_sequences_changed": int(pop_diff)}


def oracle_build_check(O, T, X, meta, index):
    """Oracle build from the raw data vs the GPU build (config 1)."""
    out = {}
    t = time.perf_counter()
    oidx = O.build_index(X, meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"])
    out["oracle_build_seconds"] = time.perf_counter() - t
    gpu_blob = T.serialize_index(index)
    out["v1_bytes_identical"] = bool(O.serialize(oidx) == gpu_blob)
    gb = np.stack(index.transform.blocks)
    ob = np.stack(oidx.blocks)
    out["mean_identical"] = bool(np.array_equal(np.asarray(index.transform.mean), oidx.mean))
    out["blocks_identical"] = bool(np.array_equal(gb, ob))
    out["blocks_max_abs_diff"] = float(np.max(np.abs(gb.astype(np.float64) - ob)))
    out["blocks_coords_differing"] = int((gb != ob).sum())
    if not out["v1_bytes_identical"]:
        # stages after the transform, given the GPU's transform
        t = time.perf_counter()
        o2 = O.build_index(X, meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"],
                           model=(np.asarray(index.transform.mean, np.float32), [np.asarray(b) for b in index.transform.blocks]))
        out["oracle_stagewise_seconds"] = time.perf_counter() - t
        out["stagewise_v1_bytes_identical"] = bool(O.serialize(o2) == gpu_blob)
        lab_eq = cb_eq = 0
        for j, sub in enumerate(index.subspaces):
            l1, l2 = o2.labels[j]
            lab_eq += int(np.array_equal(sub.codebook1.assignments, l1)) + int(np.array_equal(sub.codebook2.assignments, l2))
            cb_eq += int(np.array_equal(sub.codebook1.centroids, o2.cb1[j])) + int(np.array_equal(sub.codebook2.centroids, o2.cb2[j]))
        out["stagewise_halves_labels_identical"] = f"{lab_eq}/{2 * meta['n_sub']}"
        out["stagewise_halves_centroids_identical"] = f"{cb_eq}/{2 * meta['n_sub']}"
    return out


def run_config(cfg, args, O, T):
    from paper_2603_24919_b200.workloads import make_config

    t = time.perf_counter()
    X, Q, meta = make_config(cfg)
    gen = time.perf_counter() - t
    params = T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"])
    t = time.perf_counter()
    index = T.build_index(X, params)
    build = time.perf_counter() - t
    qp = T.QueryParams(meta["alpha"], meta["beta"], meta["k"])
    ids, dists, num, lvl = T.knn_query_batch(index, X, Q, qp)
    nq = Q.shape[0]
    limit = {4: args.cfg4_queries}.get(cfg, nq)
    sel = np.arange(min(nq, limit))
    threads = os.cpu_count() or 1
    oidx = O.deserialize(T.serialize_index(index))
    t = time.perf_counter()
    oi, od, on, ol = O.knn_batch(oidx, X, Q[sel], meta["alpha"], meta["beta"], meta["k"], threads=threads)
    oracle_s = time.perf_counter() - t
    res = {
        "config": cfg, "n": meta["n"], "d": meta["d"], "n_sub": meta["n_sub"], "kprime": meta["kprime"],
        "batch": nq, "queries_checked": int(sel.size), "oracle_threads": threads,
        "oracle_query_seconds": oracle_s, "gen_seconds": gen, "gpu_build_seconds": build,
        "ids_mismatch_queries": int((ids[sel] != oi).any(axis=1).sum()),
        "dists_mismatch_queries": int((dists[sel] != od).any(axis=1).sum()),
        "candidate_num_mismatch": int((num[sel] != on).sum()),
        "last_collision_mismatch": int((lvl[sel] != ol).sum()),
        "mean_candidate_num": float(num.mean()),
    }
    res["identical"] = all(res[k] == 0 for k in ("ids_mismatch_queries", "dists_mismatch_queries",
                                                   "candidate_num_mismatch", "last_collision_mismatch"))
    qt_gpu = T.transform_points(index.transform, Q[sel])
    res["query_transform"] = qt_flip_check(O, oidx, Q[sel], qt_gpu, meta["alpha"], threads)
    gt = T.compute_ground_truth(X, Q, meta["k"], index=index)
    res["recall@10_full_batch"] = float(np.mean([len(set(ids[i]) & set(gt.ids[i])) / meta["k"]
                                                  for i in range(nq)]))
    if cfg == 1 and args.oracle_build:
        res["build"] = oracle_build_check(O, T, X, meta, index)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--cfg4-queries", type=int, default=2048)
    ap.add_argument("--no-oracle-build", dest="oracle_build", action="store_false")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import paper_2603_24919_b200 as T
    from oracle import taco_oracle as O

    out = {"host_cores": os.cpu_count(), "configs": []}
    for c in [int(x) for x in args.configs.split(",") if x]:
        t = time.perf_counter()
        r = run_config(c, args, O, T)
        r["seconds"] = time.perf_counter() - t
        print(json.dumps(r), flush=True)
        out["configs"].append(r)
        if args.out:
            with open(args.out, "w") as fh:
                json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
