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


# bh_knn (query row in registers, top-k list in local memory) covers
# k <= 128 and D <= 64; bh_knn_general any k and D (slower)
MAX_K = 128
MAX_D = 64
BIG_K = 512  # bh_knn_f64_filtered keeps its lists thread-local up to here


def _f64_filter() -> bool:
    """BH_KNN_TILE=0 keeps the per-thread float64 kernel (A/B)."""
    import os
    return os.environ.get("BH_KNN_TILE", "1") != "0"


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
    idx = torch.empty((n, k), dtype=torch.int64, device=data.device)
    sqd = torch.empty((n, k), dtype=dt, device=data.device)
    if dt == torch.float64 and d <= MAX_D and _f64_filter():
        # float64 data: the float32 tile filter on a rounded copy, exact
        # sums on the float64 rows (the same graph, bit for bit)
        lib = _lib.load()
        ws = (_lib.workspace(lib.bh_knn_general_workspace_bytes(n, k))
              if k > BIG_K else None)
        call("bh_knn_f64_filtered", ptr(data), ptr(data.to(torch.float32)),
             n, d, k, ptr(idx), ptr(sqd), ptr(ws) if ws is not None else None,
             ws.numel() if ws is not None else 0, stream())
    elif k <= MAX_K and d <= MAX_D:
        call(_lib.fn("bh_knn", dt), ptr(data), n, d, k, ptr(idx), ptr(sqd),
             stream())
    else:  # any D / k: columns in chunks, the top-k list in scratch
        lib = _lib.load()
        ws = _lib.workspace(lib.bh_knn_general_workspace_bytes(n, k))
        call(_lib.fn("bh_knn_general", dt), ptr(data), n, d, k, ptr(idx),
             ptr(sqd), ptr(ws), ws.numel(), stream())
    return NeighborGraph(idx, sqd)
