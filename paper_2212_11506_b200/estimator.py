"""Scikit-learn-style estimator over the B200 engine.

Mirrors the reference's estimator surface -- BarnesHutTSNE.fitTransform in
pkg/frontend/src/estimator.ts:40-98 with the options of config.ts:45-96 --
as a Python class: same parameters and defaults, same validation messages
(ValueError instead of RangeError), ``kl_divergence_``, ``timings_`` and
``manifest_`` after a fit.  Unlike the TS estimator it runs in-process
(no CLI subprocess) and accepts a precomputed kNN graph.
"""

from __future__ import annotations

import hashlib

import numpy as np

from . import __version__
from .optimizer import REPORT_STAGES, TsneConfig, run


class BarnesHutTSNE:
    def __init__(self, perplexity=30.0, theta=0.5, n_iter=1000,
                 early_exaggeration=12.0, exaggeration_iters=250,
                 learning_rate=200.0, momentum_early=0.5, momentum_late=0.8,
                 min_gain=0.01, seed=0, kl_every=0, precision="f32",
                 code_bits=32):
        if not isinstance(n_iter, (int, np.integer)) or n_iter < 0:
            raise ValueError(
                f"nIter must be a non-negative integer, got {n_iter}")
        if not isinstance(seed, (int, np.integer)):
            raise ValueError(f"seed must be an integer, got {seed}")
        self.config = TsneConfig(
            perplexity=float(perplexity), theta=float(theta),
            n_iter=int(n_iter), early_exaggeration=float(early_exaggeration),
            exaggeration_iters=int(exaggeration_iters),
            learning_rate=float(learning_rate),
            momentum_early=float(momentum_early),
            momentum_late=float(momentum_late), min_gain=float(min_gain),
            seed=int(seed), kl_every=int(kl_every), precision=precision,
            code_bits=int(code_bits)).validate()
        self.kl_divergence_ = None
        self.timings_ = None
        self.manifest_ = None
        self.embedding_ = None
        self._running = False

    def fit(self, x, knn=None):
        self.fit_transform(x, knn=knn)
        return self

    def fit_transform(self, x, knn=None) -> np.ndarray:
        """Embed an N x D matrix into N x 2 (estimator.ts:57-98)."""
        data = np.ascontiguousarray(np.asarray(x, dtype=self.config.dtype))
        if data.ndim != 2:
            raise ValueError(f"expected a 2-D matrix, got {data.ndim}-D")
        if data.shape[0] < 2:
            raise ValueError(
                f"matrix must have at least 2 rows, got {data.shape[0]}")
        if not np.isfinite(data).all():
            r, c = np.argwhere(~np.isfinite(data))[0]
            raise ValueError(f"non-finite value at row {r}, column {c}")
        if self._running:
            raise RuntimeError("this estimator is already running a fit")
        self._running = True
        try:
            e, timings, kl = run(data, self.config, knn=knn)
        finally:
            self._running = False
        y = e.numpy()
        self.embedding_ = y
        self.kl_divergence_ = kl
        self.timings_ = timings.report()
        cfg = self.config
        self.manifest_ = {
            "tool": "paper_2212_11506_b200",
            "version": __version__,
            "input": {"sha256": hashlib.sha256(data.tobytes()).hexdigest(),
                      "shape": list(data.shape)},
            "config": {"perplexity": cfg.perplexity, "theta": cfg.theta,
                       "n_iter": cfg.n_iter,
                       "early_exaggeration": cfg.early_exaggeration,
                       "exaggeration_iters": cfg.exaggeration_iters,
                       "learning_rate": cfg.learning_rate,
                       "kl_every": cfg.kl_every, "code_bits": cfg.code_bits},
            "seed": cfg.seed,
            "precision": cfg.precision,
            "wall_s": timings.total_wall_s,
            "stage_totals_s": {s: timings.total(s) for s in REPORT_STAGES},
            "kl": kl,
            "kl_history": timings.kl_history,
        }
        return y
