"""Exact kNN on the B200 (knn.py:36-73 semantics).

The north star passes the reference's kNN graph in; this kernel exists so
that ``run(x, cfg)`` without a graph stays a drop-in.  Distances are f64
column-ordered sums as the reference computes them, ties -> lower id.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream
from .affinity import NeighborGraph


MAX_K = 128  # bh_knn: per-thread candidate list (csrc/knn.cu kKnnMaxK)
MAX_D = 64   # bh_knn: the query row held in registers


def knn_exact(x, k: int) -> NeighborGraph:
    """k exact neighbours; float64 data keeps float64 distances (knn.py:72),
    anything else runs in float32."""
    data = torch.as_tensor(np.ascontiguousarray(x)
                           if not isinstance(x, torch.Tensor) else x)
    dt = torch.float64 if data.dtype == torch.float64 else torch.float32
    data = data.to(_lib.device(), dt).contiguous()
    n, d = data.shape
    if not 1 <= k <= n - 1:
        raise ValueError(f"k must be in [1, {n - 1}], got {k}")
    if k > MAX_K or d > MAX_D:
        raise ValueError(
            f"the GPU exact kNN supports k <= {MAX_K} (perplexity < "
            f"{(MAX_K + 1) / 3:.0f}) and D <= {MAX_D}; got k={k}, D={d}. "
            "Pass a precomputed graph (run(..., knn=NeighborGraph) or "
            "--knn graph.npz), e.g. the reference's knn_exact, or reduce D "
            "(PCA) first")
    idx = torch.empty((n, k), dtype=torch.int64, device=data.device)
    sqd = torch.empty((n, k), dtype=dt, device=data.device)
    call(_lib.fn("bh_knn", dt), ptr(data), n, d, k, ptr(idx), ptr(sqd),
         stream())
    return NeighborGraph(idx, sqd)
