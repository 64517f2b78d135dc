"""Quality / throughput measurement on the batched GPU path.

The reference's ``taco.bench`` (pkg/src/taco/bench.py) times a per-query
loop (``_query_pass``, bench.py:120-129) over an (alpha, beta) grid.  This
module keeps its names, dataclasses, metric definitions and CSV layouts, but a
pass is ONE ``knn_query_batch`` call, so the QPS
column measures the B200 path.  ``taco.bench``'s diagnostics that are not on
the query path (pareto report, activation comparison) are out of scope.
"""

from __future__ import annotations

import csv
import statistics
import time
from dataclasses import dataclass, field

import numpy as np

from .dataio import GroundTruth
from .engine import TacoIndex, knn_query_batch, serialize_index, QueryParams
from .errors import ParameterError

_ZERO = 1e-12   # bench.py:37


def _fmt(v) -> str:
    return f"{v:.6g}" if isinstance(v, float) else str(v)


def recall(result, truth_ids, k: int) -> float:
    """|top-k found ∩ true top-k| / k (bench.py:47-55); -1 padding never matches."""
    truth_ids = np.asarray(truth_ids)
    if k > truth_ids.shape[0]:
        raise ParameterError(f"k {k} exceeds ground truth depth {truth_ids.shape[0]}")
    ids = np.asarray(result.ids if hasattr(result, "ids") else result)
    return np.intersect1d(ids[:k][ids[:k] >= 0], truth_ids[:k]).size / k


def mre_with_skips(result_dists, truth_dists, k: int) -> tuple[float, int]:
    """Mean relative distance error over the k ranks and the skipped-rank count
    (bench.py:58-87): both lists ascending; a ~0 true distance counts 0 when the
    result is ~0 too and is skipped otherwise; missing result ranks are skipped."""
    tru_all = np.asarray(truth_dists, dtype=np.float64)
    if k > tru_all.shape[0]:
        raise ParameterError(f"k {k} exceeds ground truth depth {tru_all.shape[0]}")
    res = np.asarray(result_dists, dtype=np.float64)
    res = np.sort(res[np.isfinite(res)])   # +inf = padding of a short result
    tru = np.sort(tru_all)[:k]
    total, used, skipped = 0.0, 0, 0
    for r in range(k):
        if r >= res.shape[0]:
            skipped += 1
        elif tru[r] < _ZERO:
            if res[r] < _ZERO:
                used += 1
            else:
                skipped += 1
        else:
            total += (res[r] - tru[r]) / tru[r]
            used += 1
    return (total / used if used else 0.0), skipped


def mre(result_dists, truth_dists, k: int) -> float:
    return mre_with_skips(result_dists, truth_dists, k)[0]


@dataclass
class Metrics:   # bench.py:94-113
    alpha: float
    beta: float
    k: int
    recall: float
    mre: float
    mre_skipped: int
    qps: float
    build_seconds: float
    index_bytes: int
    threads: int
    candidate_counts: np.ndarray
    candidate_budget_ratio: float

    @property
    def mean_candidates(self) -> float:
        return float(np.mean(self.candidate_counts))


@dataclass
class BenchmarkReport:
    rows: list
    metadata: dict = field(default_factory=dict)
    query_records: list = field(default_factory=list)


def run_benchmark(index: TacoIndex, data, queries, truth: GroundTruth, alphas, betas, k: int = 50,
                  threads: int = 1, warmup: int = 1, repeats: int = 3,
                  record_queries: bool = False) -> BenchmarkReport:
    """One metrics row per (alpha, beta) grid point (bench.py:132-194): quality
    from an untimed pass, QPS = median of ``repeats`` timed batched passes after
    ``warmup`` warm-up passes (the first untimed pass counts as one)."""
    queries = np.asarray(queries)
    if truth.k < k:
        raise ParameterError(f"ground truth depth {truth.k} is below k {k}")
    if queries.shape[0] != truth.ids.shape[0]:
        raise ParameterError(f"{queries.shape[0]} queries but {truth.ids.shape[0]} truth rows")
    report = BenchmarkReport(rows=[], metadata={
        "threads": threads, "warmup_passes": warmup, "timed_passes": repeats,
        "n_queries": int(queries.shape[0]), "query_removal": "after-subset-sampling",
        "path": "knn_query_batch (B200)",
    })
    index_bytes = len(serialize_index(index))
    build_seconds = float(index.metadata.get("build_seconds", float("nan")))
    for alpha in alphas:
        for beta in betas:
            qp = QueryParams(alpha=float(alpha), beta=float(beta), k=k)
            ids, dists, num, lvl = knn_query_batch(index, data, queries, qp)
            recalls, mres, skips = [], [], 0
            for qi in range(ids.shape[0]):
                recalls.append(recall(ids[qi], truth.ids[qi], k))
                v, sk = mre_with_skips(dists[qi], truth.dists[qi], k)
                mres.append(v)
                skips += sk
                if record_queries:
                    report.query_records.append({
                        "query": qi, "alpha": float(alpha), "beta": float(beta), "recall": recalls[-1],
                        "mre": v, "candidates": int(num[qi]), "last_collision": int(lvl[qi])})
            for _ in range(max(0, warmup - 1)):
                knn_query_batch(index, data, queries, qp)
            times = []
            for _ in range(repeats):
                t0 = time.perf_counter()
                knn_query_batch(index, data, queries, qp)
                times.append(time.perf_counter() - t0)
            report.rows.append(Metrics(
                alpha=float(alpha), beta=float(beta), k=k, recall=float(np.mean(recalls)),
                mre=float(np.mean(mres)), mre_skipped=skips, qps=ids.shape[0] / statistics.median(times),
                build_seconds=build_seconds, index_bytes=index_bytes, threads=threads,
                candidate_counts=num.astype(np.int64),
                candidate_budget_ratio=float(np.mean(num) / (float(beta) * index.n))))
    return report


def write_metrics_csv(report: BenchmarkReport, path) -> None:
    """Column layout of bench.py:197-210."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["alpha", "beta", "k", "recall", "mre", "mre_skipped", "qps", "build_seconds",
                    "index_bytes", "mean_candidates", "candidate_budget_ratio", "threads"])
        for r in report.rows:
            w.writerow([_fmt(v) for v in (r.alpha, r.beta, r.k, r.recall, r.mre, r.mre_skipped, r.qps,
                                          r.build_seconds, r.index_bytes, r.mean_candidates,
                                          r.candidate_budget_ratio, r.threads)])


def write_query_records_csv(report: BenchmarkReport, path) -> None:
    """Column layout of bench.py:213-224."""
    cols = ("query", "alpha", "beta", "recall", "mre", "candidates", "last_collision")
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(list(cols))
        for rec in report.query_records:
            w.writerow([_fmt(rec[c]) for c in cols])
