"""Config 5 (n = 1e8, d = 128, K' = 256, k = 100) on ONE B200 (run on the GPU box).

    python tools/run_cfg5.py --nq-run 2000 --oracle-queries 16 --out gpurun_out/cfg5.json

BASELINE config 5 is stated for 2/4/8 GPUs; this run asks whether the whole
index fits one B200 (X 51.2 GB + transformed 51.2 GB + CSR 3.2 GB resident,
k-means halves sized to the free memory) and measures, at that scale:
  * the GPU build (build_index: covariance, eigensolve, transform, 16
    k-means halves of 1e8 points x 256 centroids, cells) with its stages;
  * a query sample (the first NQ of the 100,000-query batch) through the
    public batched API, timed with CUDA-synchronised wall clock around
    knn_query_batch (inputs host-resident: this is the e2e number);
  * parity: the CPU oracle (oracle/taco_oracle.py) answers the first
    ORACLE_QUERIES queries on the GPU-built index (v1 bytes) -- ids,
    distances, candidate_num, last_collision compared query by query;
  * recall@100 of the sample against the GPU exact ground truth.
The base matrix is generated with the workloads generator's per-chunk
streams (rng([1005, 0, chunk])), chunks in a thread pool; identical to
workloads.make_config(5) by construction (same streams, same order).

The oracle is the checker here, never the thing measured.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def host_gb_available():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except Exception:
        return float("nan")


def generate(cfg, n, nq, threads):
    from paper_2603_24919_b200 import workloads as W

    c = W.CONFIGS[cfg]
    d = c["d"]
    A, mu = W._mixture(cfg, d)
    X = np.empty((n, d), np.float32)
    nch = math.ceil(n / W.CHUNK)

    def one(b):
        lo, hi = b * W.CHUNK, min(n, (b + 1) * W.CHUNK)
        X[lo:hi] = W._draw(cfg, np.random.default_rng([1000 + cfg, 0, b]), hi - lo, A, mu)

    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(one, range(nch)))
    qr = np.random.default_rng([1000 + cfg, 1])
    if cfg in (1, 5):
        rows = qr.choice(n, size=nq, replace=False)
        Q = (X[rows].astype(np.float64) + 0.05 * qr.standard_normal((nq, d))).astype(np.float32)
    else:
        Q = W._draw(cfg, qr, nq, A, mu)
    return X, Q, W._meta(cfg, n, nq, d)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--nq-run", type=int, default=2000, help="queries of the batch answered on the GPU")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--oracle-queries", type=int, default=16)
    ap.add_argument("--gt-queries", type=int, default=200)
    ap.add_argument("--min-host-gb", type=float, default=0.0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = {"host_cores": os.cpu_count(), "host_gb_available_start": host_gb_available()}

    def dump():
        print(json.dumps(out), flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                json.dump(out, fh, indent=1)

    from paper_2603_24919_b200.workloads import CONFIGS
    n = args.n or CONFIGS[args.cfg]["n"]
    need = n * CONFIGS[args.cfg]["d"] * 4 / 2**30 * 1.25
    if out["host_gb_available_start"] == out["host_gb_available_start"] and \
            out["host_gb_available_start"] < max(need, args.min_host_gb):
        out["skipped"] = f"host memory {out['host_gb_available_start']:.0f} GB < {need:.0f} GB needed"
        dump()
        return
    import torch
    import paper_2603_24919_b200 as T

    nq_total = CONFIGS[args.cfg]["nq"]
    t = time.perf_counter()
    X, Q, meta = generate(args.cfg, n, nq_total, os.cpu_count() or 1)
    out["gen_seconds"] = time.perf_counter() - t
    out.update(config=args.cfg, n=n, d=meta["d"], n_sub=meta["n_sub"], s=meta["s"], kprime=meta["kprime"],
               alpha=meta["alpha"], beta=meta["beta"], k=meta["k"], batch=nq_total)
    free0, tot = torch.cuda.mem_get_info()
    out["device_free_gb_before_build"] = free0 / 2**30
    out["device_total_gb"] = tot / 2**30
    dump()
    params = T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"])
    torch.cuda.synchronize()
    t = time.perf_counter()
    index = T.build_index(X, params)
    torch.cuda.synchronize()
    out["build_seconds"] = time.perf_counter() - t
    out["build_stages"] = {k: index.metadata[k] for k in ("covariance_seconds", "eigensolve_seconds",
                                                          "transform_only_seconds", "kmeans_only_seconds",
                                                          "cells_seconds")}
    free1, _ = torch.cuda.mem_get_info()
    out["device_free_gb_after_build"] = free1 / 2**30
    out["device_peak_reserved_gb"] = (tot - free1) / 2**30
    dump()
    qp = T.QueryParams(meta["alpha"], meta["beta"], meta["k"])
    Qr = np.ascontiguousarray(Q[:args.nq_run])
    times = []
    for r in range(max(1, args.reps)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ids, dists, num, lvl = T.knn_query_batch(index, X, Qr, qp)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    out["query_seconds_all"] = times
    out["qps_e2e"] = args.nq_run / min(times)
    out["queries_run"] = int(args.nq_run)
    out["mean_candidate_num"] = float(num.mean())
    out["levels"] = np.bincount(lvl).tolist()
    dump()
    # one profiled pass: per-kernel CUDA-event times on the launching stream
    from paper_2603_24919_b200 import _native as nat
    nat.profile_enable(True)
    nat.profile_read(reset=True)
    T.knn_query_batch(index, X, Qr, qp)
    torch.cuda.synchronize()
    prof, stats = nat.profile_read(reset=True)
    nat.profile_enable(False)
    out["kernels_ms"] = {k: round(v[0], 3) for k, v in prof.items() if v[0] > 0}
    out["query_stats"] = stats
    dump()
    # recall@k of the sample against the GPU exact ground truth
    g = min(args.gt_queries, args.nq_run)
    if g <= 0:
        return
    t = time.perf_counter()
    gt = T.compute_ground_truth(X, Qr[:g], meta["k"], index=index)
    out["ground_truth_seconds"] = time.perf_counter() - t
    out[f"recall@{meta['k']}"] = float(np.mean([len(set(ids[i]) & set(gt.ids[i])) / meta["k"] for i in range(g)]))
    out["recall_queries"] = g
    dump()
    # oracle parity on the GPU-built index
    if args.oracle_queries > 0:
        from oracle import taco_oracle as O
        t = time.perf_counter()
        oidx = O.deserialize(T.serialize_index(index))
        out["oracle_index_load_seconds"] = time.perf_counter() - t
        sel = np.arange(min(args.oracle_queries, args.nq_run))
        t = time.perf_counter()
        oi, od, on, ol = O.knn_batch(oidx, X, Qr[sel], meta["alpha"], meta["beta"], meta["k"],
                                     threads=min(len(sel), os.cpu_count() or 1))
        out["oracle_query_seconds"] = time.perf_counter() - t
        out["oracle_queries_checked"] = int(sel.size)
        out["ids_mismatch_queries"] = int((ids[sel] != oi).any(axis=1).sum())
        out["dists_mismatch_queries"] = int((dists[sel] != od).any(axis=1).sum())
        out["candidate_num_mismatch"] = int((num[sel] != on).sum())
        out["last_collision_mismatch"] = int((lvl[sel] != ol).sum())
        out["identical"] = all(out[k] == 0 for k in ("ids_mismatch_queries", "dists_mismatch_queries",
                                                      "candidate_num_mismatch", "last_collision_mismatch"))
    dump()


if __name__ == "__main__":
    main()
