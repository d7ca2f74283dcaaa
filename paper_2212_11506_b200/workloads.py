"""Seeded synthetic workloads C0-C4 (BASELINE.json configs).

The paper's datasets (mouse-brain 1.3M, MNIST, ...) are not available; these
generators stand in for them with the shapes, sizes and value distributions
BASELINE.json names.  Used by bench.py and the tests; not part of the
optimisation path itself.
"""

from __future__ import annotations

import numpy as np


def c0(seed: int = 0) -> np.ndarray:
    """N=2048, D=10: 4 isotropic clusters x 512, centres U[-10,10]^10, sigma 1."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-10, 10, (4, 10))
    lab = np.repeat(np.arange(4), 512)
    x = centres[lab] + rng.standard_normal((2048, 10))
    return x.astype(np.float32)


def c1(seed: int = 0, n: int = 70_000, d: int = 50, k: int = 10) -> np.ndarray:
    """N=70k, D=50: 10 clusters, sizes 7000*(1+U(-.1,.1)), diagonal
    variances 0.9^d."""
    rng = np.random.default_rng(seed)
    base = n // k
    sizes = np.floor(base * (1 + rng.uniform(-0.1, 0.1, k))).astype(np.int64)
    sizes[-1] = n - sizes[:-1].sum()
    centres = rng.uniform(-10, 10, (k, d))
    std = np.sqrt(0.9 ** np.arange(d))
    parts = [centres[c] + rng.standard_normal((s, d)) * std
             for c, s in enumerate(sizes)]
    return np.vstack(parts).astype(np.float32)


def _rotation(rng, d):
    q, r = np.linalg.qr(rng.standard_normal((d, d)))
    return q * np.sign(np.diag(r))


def _rotated_mixture(rng, sizes, d, decay):
    centres = rng.uniform(-10, 10, (len(sizes), d))
    std = np.sqrt(decay ** np.arange(d))
    parts = []
    for c, s in enumerate(sizes):
        q = _rotation(rng, d)
        z = rng.standard_normal((int(s), d)) * std
        parts.append(centres[c] + z @ q.T)
    return np.vstack(parts)


def c2(seed: int = 0, n: int = 250_000, d: int = 50, k: int = 20) -> np.ndarray:
    """N=250k, D=50: 20 rotated clusters, eigenvalues 0.85^d, sizes ~ c^-1.5."""
    rng = np.random.default_rng(seed)
    w = np.arange(1, k + 1, dtype=np.float64) ** -1.5
    sizes = np.floor(n * w / w.sum()).astype(np.int64)
    sizes[0] += n - sizes.sum()
    return _rotated_mixture(rng, sizes, d, 0.85).astype(np.float32)


def c3(seed: int = 0, n: int = 1_300_000, d: int = 50, k: int = 40,
       noise_frac: float = 0.02) -> np.ndarray:
    """N=1.3M, D=50: 40 rotated clusters (log-normal sizes, eigenvalues 0.9^d)
    holding 98% of the points plus 2% uniform background noise."""
    rng = np.random.default_rng(seed)
    n_noise = int(round(n * noise_frac))
    n_cl = n - n_noise
    w = rng.lognormal(0.0, 1.0, k)
    sizes = np.floor(n_cl * w / w.sum()).astype(np.int64)
    sizes[np.argmax(sizes)] += n_cl - sizes.sum()
    x = _rotated_mixture(rng, sizes, d, 0.9)
    lo, hi = x.min(axis=0), x.max(axis=0)
    noise = rng.uniform(lo, hi, (n_noise, d))
    return np.vstack([x, noise]).astype(np.float32)


def c4_points(seed: int = 0, n: int = 4_000_000, k: int = 100) -> np.ndarray:
    """2-D microbench embedding: 100 centres U[-50,50]^2, multivariate
    Student-t (nu=2, scale 1) around each.  Returns (n, 2) f32."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-50, 50, (k, 2))
    lab = rng.integers(0, k, n)
    g = rng.standard_normal((n, 2))
    w = rng.chisquare(2.0, n) / 2.0
    y = centres[lab] + g / np.sqrt(w)[:, None]
    return y.astype(np.float32)


def c4_directed(seed: int, n: int, k: int = 90):
    """Random directed kNN-like graph for C4: per row k distinct uniform
    neighbours != i, values U(0,1]+1e-3 row-normalised.  Returns
    (indices int32 (n,k), cond f64 (n,k))."""
    rng = np.random.default_rng(seed + 1)
    idx = np.empty((n, k), np.int32)
    chunk = 1 << 18
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        m = e - s
        # draw with replacement then repair duplicates / self loops row-wise
        cand = rng.integers(0, n - 1, (m, k + 8), dtype=np.int64)
        rows = np.arange(s, e)[:, None]
        cand = cand + (cand >= rows)  # skip self
        cand.sort(axis=1)
        dup = np.zeros_like(cand, dtype=bool)
        dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
        cand[dup] = n + 1  # push duplicates to the end
        cand.sort(axis=1)
        bad = (cand[:, k - 1] >= n)
        for r in np.flatnonzero(bad):  # rare: redraw exactly
            i = s + r
            pick = rng.choice(n - 1, k, replace=False)
            pick = pick + (pick >= i)
            cand[r, :k] = np.sort(pick)
        idx[s:e] = cand[:, :k]
    vals = rng.uniform(0.0, 1.0, (n, k))
    vals = (1.0 - vals) + 1e-3  # U(0,1] + 1e-3
    vals /= vals.sum(axis=1, keepdims=True)
    return idx, vals


CONFIGS = {
    "c0": dict(n=2048, d=10, gen=c0),
    "c1": dict(n=70_000, d=50, gen=c1),
    "c2": dict(n=250_000, d=50, gen=c2),
    "c3": dict(n=1_300_000, d=50, gen=c3),
}
