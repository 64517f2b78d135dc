"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The reference measures on DEEP/SIFT/GIST-style corpora that are not in this
container; SURVEY.md section 8(d) fixes a generator with the same shapes,
spectra and value distributions.  Every parameter is recorded in the
returned ``meta`` dict so runs can state what they measured.

Rows are generated in independent 1M-row chunks (``rng([1000+c, 0, b])``),
so shards and sampled checks can regenerate any chunk on its own.
"""

from __future__ import annotations

import math

import numpy as np

CHUNK = 1_000_000

# cfg -> (n, d, N_s, s, K', alpha, beta, k, nq, mixture C, power p, lambda_1)
CONFIGS = {
    1: dict(n=100_000, d=128, n_sub=8, s=16, kprime=50, alpha=0.05, beta=0.005, k=10,
            nq=1_000, comps=100, power=1.0, lam1=1.0),
    2: dict(n=1_000_000, d=128, n_sub=8, s=16, kprime=64, alpha=0.03, beta=0.003, k=10,
            nq=10_000, comps=1_000, power=1.2, lam1=3600.0),
    3: dict(n=1_000_000, d=960, n_sub=16, s=60, kprime=64, alpha=0.03, beta=0.002, k=10,
            nq=1_000, comps=1_000, power=1.5, lam1=1.0),
    4: dict(n=10_000_000, d=96, n_sub=8, s=12, kprime=128, alpha=0.01, beta=0.001, k=10,
            nq=10_000, comps=5_000, power=0.8, lam1=1.0),
    5: dict(n=100_000_000, d=128, n_sub=8, s=16, kprime=256, alpha=0.005, beta=0.0005, k=100,
            nq=100_000, comps=10_000, power=1.2, lam1=1.0),
}


def _mixture(cfg: int, d: int):
    c = CONFIGS[cfg]
    rng = np.random.default_rng([1000 + cfg, 2])
    q, r = np.linalg.qr(rng.standard_normal((d, d)))
    q = q * np.where(np.diag(r) < 0, -1.0, 1.0)
    lam = c["lam1"] * np.arange(1, d + 1, dtype=np.float64) ** (-c["power"])
    A = q * np.sqrt(lam)[None, :]
    if cfg == 2:
        mu = 22.0 + 40.0 * rng.standard_normal((c["comps"], d))
    else:
        mu = 2.0 * rng.standard_normal((c["comps"], d))
    return A, mu


def _post(cfg: int, x: np.ndarray) -> np.ndarray:
    if cfg == 2:
        x = np.clip(np.rint(np.maximum(x, 0.0)), 0.0, 255.0)
    elif cfg == 4:
        x = x / np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(np.float32)


def _draw(cfg: int, rng, size: int, A, mu):
    lab = rng.integers(mu.shape[0], size=size)
    return _post(cfg, mu[lab] + rng.standard_normal((size, A.shape[0])) @ A.T)


def base_chunk(cfg: int, b: int, size: int, d: int | None = None):
    c = CONFIGS[cfg]
    d = d or c["d"]
    A, mu = _mixture(cfg, d)
    return _draw(cfg, np.random.default_rng([1000 + cfg, 0, b]), size, A, mu)


def make_shard(cfg: int, lo: int, hi: int, n: int | None = None, nq: int | None = None,
               d: int | None = None):
    """(rows [lo, hi) of the base matrix, all queries, meta) -- what one rank
    of a point-sharded run generates; equal to make_config's X[lo:hi] and Q."""
    c = dict(CONFIGS[cfg])
    n = c["n"] if n is None else n
    nq = c["nq"] if nq is None else nq
    d = c["d"] if d is None else d
    A, mu = _mixture(cfg, d)
    X = np.empty((hi - lo, d), np.float32)
    for b in range(lo // CHUNK, math.ceil(hi / CHUNK)):
        c0 = b * CHUNK
        clen = min(CHUNK, n - c0)
        a0, a1 = max(lo, c0), min(hi, c0 + clen)
        X[a0 - lo:a1 - lo] = _draw(cfg, np.random.default_rng([1000 + cfg, 0, b]), clen, A, mu)[a0 - c0:a1 - c0]
    qr = np.random.default_rng([1000 + cfg, 1])
    if cfg in (1, 5):   # queries are base rows + noise: regenerate the chunks holding them
        rows = qr.choice(n, size=nq, replace=False)
        base = np.empty((nq, d), np.float32)
        for b in np.unique(rows // CHUNK):
            c0 = int(b) * CHUNK
            clen = min(CHUNK, n - c0)
            chunk = _draw(cfg, np.random.default_rng([1000 + cfg, 0, int(b)]), clen, A, mu)
            sel = rows // CHUNK == b
            base[sel] = chunk[rows[sel] - c0]
        Q = (base.astype(np.float64) + 0.05 * qr.standard_normal((nq, d))).astype(np.float32)
    else:
        Q = _draw(cfg, qr, nq, A, mu)
    return X, Q, _meta(cfg, n, nq, d)


def _meta(cfg, n, nq, d):
    c = CONFIGS[cfg]
    s = c["s"] if d == c["d"] else max(2, d // c["n_sub"])
    return dict(cfg=cfg, n=n, d=d, nq=nq, n_sub=c["n_sub"], s=s,
                clusters=c["kprime"] ** 2, kprime=c["kprime"], kmeans_iters=20, seed=0,
                alpha=c["alpha"], beta=c["beta"], k=c["k"], mixture=c["comps"],
                power=c["power"], lam1=c["lam1"],
                generator="SURVEY.md 8(d): rotated anisotropic Gaussian mixture, "
                          "rng([1000+cfg,0,chunk]) base / rng([1000+cfg,1]) queries")


def make_config(cfg: int, n: int | None = None, nq: int | None = None,
                d: int | None = None):
    """Return (base f32[n,d], queries f32[nq,d], meta).

    ``n``/``nq``/``d`` override the sizes for small parity cases; the
    distribution parameters stay those of ``cfg``."""
    c = dict(CONFIGS[cfg])
    n = c["n"] if n is None else n
    nq = c["nq"] if nq is None else nq
    d = c["d"] if d is None else d
    A, mu = _mixture(cfg, d)
    X = np.empty((n, d), np.float32)
    for b in range(math.ceil(n / CHUNK)):
        lo, hi = b * CHUNK, min(n, (b + 1) * CHUNK)
        X[lo:hi] = _draw(cfg, np.random.default_rng([1000 + cfg, 0, b]), hi - lo, A, mu)
    qr = np.random.default_rng([1000 + cfg, 1])
    if cfg in (1, 5):
        rows = qr.choice(n, size=nq, replace=False)
        Q = (X[rows].astype(np.float64) + 0.05 * qr.standard_normal((nq, d))).astype(np.float32)
    else:
        Q = _draw(cfg, qr, nq, A, mu)
    meta = _meta(cfg, n, nq, d)
    return X, Q, meta
