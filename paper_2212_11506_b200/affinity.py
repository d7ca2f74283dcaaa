"""Perplexity calibration and the symmetric sparse P on the B200.

Mirrors bhtsne.affinity and bhtsne.knn's graph type (reference:
pkg/src/bhtsne/affinity.py, knn.py:20-33): ``NeighborGraph``,
``PerplexityResult``, ``SparseAffinity``, ``calibrate_perplexity``
(:99-118), ``symmetrize`` (:121-158), ``set_exaggeration`` (:161-173).

Device layout: CSR with int64 ``row_offsets``, int32 ``col_indices`` and
``base_values`` (the pristine, unexaggerated p_ij) in the run precision,
float32 or float64 (symmetrize's ``dtype``, affinity.py:121-158).  The
exaggeration factor is applied inside the kernels as ``base * dtype(factor)``
-- the same product set_exaggeration computes -- so rescaling never
rewrites the matrix and restoring factor 1 is bitwise exact.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream

DEFAULT_MAX_ITER = 200
DEFAULT_TOL_BITS = 1e-5


@dataclass(frozen=True)
class NeighborGraph:
    """k neighbour ids and squared distances per point, ascending per row
    (knn.py:20-33).  Accepts numpy or torch; stored on the device."""

    indices: torch.Tensor       # (N, k) int64
    sq_distances: torch.Tensor  # (N, k) float32 or float64 (the data's dtype)

    def __post_init__(self):
        dev = _lib.device()
        idx = torch.as_tensor(np.asarray(self.indices) if not isinstance(
            self.indices, torch.Tensor) else self.indices)
        sqd = torch.as_tensor(np.asarray(self.sq_distances) if not isinstance(
            self.sq_distances, torch.Tensor) else self.sq_distances)
        if idx.ndim != 2 or sqd.shape != idx.shape:
            raise ValueError("indices and sq_distances must be (N, k)")
        object.__setattr__(self, "indices",
                           idx.to(dev, torch.int64).contiguous())
        sdt = torch.float64 if sqd.dtype == torch.float64 else torch.float32
        object.__setattr__(self, "sq_distances",
                           sqd.to(dev, sdt).contiguous())

    @property
    def n_points(self) -> int:
        return self.indices.shape[0]

    @property
    def k(self) -> int:
        return self.indices.shape[1]


@dataclass(frozen=True)
class PerplexityResult:
    betas: torch.Tensor        # (N,) float64
    conditional: torch.Tensor  # (N, k) float64


@dataclass(frozen=True)
class SparseAffinity:
    """Symmetric p_ij in CSR form (affinity.py:40-58)."""

    n: int
    row_offsets: torch.Tensor  # (N+1,) int64
    col_indices: torch.Tensor  # (nnz,) int32
    base_values: torch.Tensor  # (nnz,) float32 | float64, exaggeration 1
    exaggeration: float = 1.0
    _padded: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def nnz(self) -> int:
        return self.col_indices.shape[0]

    @property
    def values(self) -> torch.Tensor:
        """Currently applied values (base * dtype(factor), affinity.py:171)."""
        if self.exaggeration == 1.0:
            return self.base_values
        return self.base_values * torch.tensor(
            self.exaggeration, dtype=self.base_values.dtype,
            device=self.base_values.device)

    @property
    def dtype(self) -> torch.dtype:
        return self.base_values.dtype

    def padded(self):
        """(row_ptr, col, val) with rows padded to multiples of 4 entries
        for the 128-bit attractive sweep (cached, built on the device)."""
        if "csr" not in self._padded:
            self._padded["csr"] = pad_csr(self.row_offsets, self.col_indices,
                                          self.base_values)
        return self._padded["csr"]

    def to_reference(self):
        return (self.row_offsets.cpu().numpy(),
                self.col_indices.cpu().numpy().astype(np.int64),
                self.values.cpu().numpy())


def as_graph(g) -> NeighborGraph:
    if isinstance(g, NeighborGraph):
        return g
    if isinstance(g, tuple) and len(g) == 2:
        return NeighborGraph(*g)
    if hasattr(g, "indices") and hasattr(g, "sq_distances"):
        return NeighborGraph(g.indices, g.sq_distances)
    raise TypeError("expected a NeighborGraph or (indices, sq_distances)")


def calibrate_perplexity(g, u: float, max_iter: int = DEFAULT_MAX_ITER,
                         tol: float = DEFAULT_TOL_BITS) -> PerplexityResult:
    """Per-row bisection on beta until 2^H is within 2^+-tol of u."""
    g = as_graph(g)
    k = g.k
    if u > k:
        raise ValueError(
            f"perplexity exceeds neighborhood size (u={u}, k={k})")
    if u <= 1:
        raise ValueError(f"perplexity must be > 1, got {u}")
    if tol <= 0:
        raise ValueError(f"tolerance must be > 0, got {tol}")
    n = g.n_points
    dev = g.indices.device
    cond = torch.empty((n, k), dtype=torch.float64, device=dev)
    betas = torch.empty(n, dtype=torch.float64, device=dev)
    call(_lib.fn("bh_bsp", g.sq_distances.dtype), ptr(g.sq_distances), n, k,
         float(u), float(tol), int(max_iter), ptr(betas), ptr(cond), stream())
    return PerplexityResult(betas=betas, conditional=cond)


def symmetrize(pr: PerplexityResult, g, dtype=np.float32) -> SparseAffinity:
    """p_ij = max((p_j|i + p_i|j) / 2N, eps64) as a ``dtype`` CSR."""
    g = as_graph(g)
    dt = _lib.torch_dtype(dtype)
    n, k = g.indices.shape
    if tuple(pr.conditional.shape) != (n, k):
        raise ValueError("perplexity result does not match neighbor graph")
    lib = _lib.load()
    dev = g.indices.device
    ws = _lib.workspace(lib.bh_symmetrize_workspace_bytes(n, k))
    nnz_t = torch.zeros(1, dtype=torch.int64, device=dev)
    call("bh_symmetrize_plan", ptr(g.indices), n, k, ptr(nnz_t), ptr(ws),
         ws.numel(), stream())
    nnz = int(nnz_t.item())
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=dt, device=dev)
    call(_lib.fn("bh_symmetrize_fill", dt), ptr(pr.conditional), n, k,
         ptr(nnz_t), ptr(row_ptr), ptr(col), ptr(val), ptr(ws), ws.numel(),
         stream())
    del ws
    return SparseAffinity(n=n, row_offsets=row_ptr, col_indices=col,
                          base_values=val, exaggeration=1.0)


def from_csr(row_offsets, col_indices, values, n=None) -> SparseAffinity:
    """Wrap a host/device CSR (e.g. the reference's SparseAffinity arrays);
    float64 values stay float64 (the f64 run mode), others become float32."""
    dev = _lib.device()
    ro = torch.as_tensor(np.asarray(row_offsets, np.int64)
                         if not isinstance(row_offsets, torch.Tensor)
                         else row_offsets).to(dev, torch.int64).contiguous()
    ci = torch.as_tensor(np.asarray(col_indices)
                         if not isinstance(col_indices, torch.Tensor)
                         else col_indices).to(dev, torch.int32).contiguous()
    va = torch.as_tensor(np.asarray(values)
                         if not isinstance(values, torch.Tensor) else values)
    vdt = torch.float64 if va.dtype == torch.float64 else torch.float32
    va = va.to(dev, vdt).contiguous()
    return SparseAffinity(n=int(n if n is not None else ro.shape[0] - 1),
                          row_offsets=ro, col_indices=ci, base_values=va)


def set_exaggeration(p: SparseAffinity, factor: float) -> SparseAffinity:
    """Rescale so values sum to ``factor``; factor 1 restores them bitwise."""
    if factor <= 0:
        raise ValueError(f"exaggeration factor must be > 0, got {factor}")
    return SparseAffinity(n=p.n, row_offsets=p.row_offsets,
                          col_indices=p.col_indices,
                          base_values=p.base_values,
                          exaggeration=float(factor), _padded=p._padded)


def pad_csr(row_ptr, col, val):
    """Device CSR -> rows padded to multiples of 4 (bh_pad_csr_*)."""
    lib = _lib.load()
    n = row_ptr.shape[0] - 1
    dev = row_ptr.device
    out_rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = _lib.workspace(lib.bh_pad_csr_workspace_bytes(n))
    call("bh_pad_csr_size", ptr(row_ptr), n, ptr(out_rp), ptr(total), ptr(ws),
         ws.numel(), stream())
    m = int(total.item())
    ocol = torch.empty(m, dtype=torch.int32, device=dev)
    oval = torch.empty(m, dtype=val.dtype, device=dev)
    call(_lib.fn("bh_pad_csr_fill", val.dtype), ptr(row_ptr), ptr(col),
         ptr(val), n, ptr(out_rp), ptr(ocol), ptr(oval), stream())
    return out_rp, ocol, oval
