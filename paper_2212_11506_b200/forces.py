"""Attractive and repulsive forces on the B200.

Mirrors bhtsne.forces (reference: pkg/src/bhtsne/forces.py):
``GradientBuffers`` (:30-53), ``attractive`` (:56-82), ``repulsive_bh``
(:85-150) and ``repulsive_exact`` (:153-182), with the same argument
meaning and error messages.  Buffers are (N, 2) float32 or float64 / (N,)
float64 CUDA tensors; ``z`` is kept on the device and read on access.

Precision: as in the reference, the arrays' dtype selects it -- float64
points (or a float64 P / tree) run the library's ``_f64`` kernels, whose
pair terms are float64 in the reference's operation order; float32 runs
the f32 kernels (f32 pair terms, f64 accumulation).  Mixed inputs are
promoted to float64 (exact), the reference's own arithmetic.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream
from .quadtree import MortonQuadtree, as_points


@dataclass
class GradientBuffers:
    """Per-point force accumulators and the normalisation term Z."""

    attr: torch.Tensor       # (N, 2) float32 | float64
    rep: torch.Tensor        # (N, 2), unnormalised repulsion
    z_partial: torch.Tensor  # (N,) float64 per-point contributions to Z
    z_dev: torch.Tensor = field(default=None)  # (1,) float64 on device

    @classmethod
    def allocate(cls, n: int, dtype=np.float32) -> "GradientBuffers":
        dt = _lib.torch_dtype(dtype)
        dev = _lib.device()
        f = lambda: torch.zeros((n, 2), dtype=dt, device=dev)
        return cls(attr=f(), rep=f(),
                   z_partial=torch.zeros(n, dtype=torch.float64, device=dev),
                   z_dev=torch.zeros(1, dtype=torch.float64, device=dev))

    @property
    def dtype(self) -> torch.dtype:
        return self.attr.dtype

    @property
    def z(self) -> float:
        return float(self.z_dev.item())

    attr0 = property(lambda s: s.attr[:, 0])
    attr1 = property(lambda s: s.attr[:, 1])
    rep0 = property(lambda s: s.rep[:, 0])
    rep1 = property(lambda s: s.rep[:, 1])


class _Out:
    """An (N, 2) result in the run precision ``dt``, stored into ``dst``
    (cast when the caller's buffers have another dtype, as numpy does when
    the reference's kernels write f64 results into f32 buffers)."""

    def __init__(self, dst: torch.Tensor, dt: torch.dtype):
        self.dst = dst
        self.t = dst if dst.dtype == dt else torch.empty(
            dst.shape, dtype=dt, device=dst.device)

    def done(self):
        if self.t is not self.dst:
            self.dst.copy_(self.t)


def attractive(p, y, out: GradientBuffers) -> None:
    """attr_i = sum_j p_ij (y_i - y_j) / (1 + |y_i - y_j|^2) -- forces.py:56."""
    pts = as_points(y)
    n = pts.shape[0]
    if p.n != n:
        raise ValueError(f"matrix is over {p.n} points, embedding has {n}")
    dt = (torch.float64 if torch.float64 in (pts.dtype, p.base_values.dtype)
          else torch.float32)
    res = _Out(out.attr, dt)
    pts = pts.to(dt)
    vals = p.base_values.to(dt)
    call(_lib.fn("bh_attractive", dt), ptr(p.row_offsets),
         ptr(p.col_indices), ptr(vals), n, 0, ptr(pts), 0, n,
         float(p.exaggeration), None, ptr(res.t), stream())
    res.done()


def repulsive_bh(t: MortonQuadtree, y, theta: float,
                 out: GradientBuffers) -> None:
    """Barnes-Hut repulsion over the summarized tree -- forces.py:134-150."""
    if not t.summarized:
        raise ValueError("tree must be summarized before computing repulsion")
    if theta < 0:
        raise ValueError(f"theta must be >= 0, got {theta}")
    dt = t.arrays.dtype
    pts = as_points(y, dt)
    n = pts.shape[0]
    if n != t.n_points:
        raise ValueError(f"tree is over {t.n_points} points, embedding has {n}")
    res = _Out(out.rep, dt)
    lib = _lib.load()
    ws = _lib.workspace(lib.bh_repulsive_workspace_bytes(n))
    call(_lib.fn("bh_repulsive", dt), t.arrays.sref(), ptr(t.bounds),
         float(theta), ptr(pts), 0, n, 0, ptr(res.t), ptr(out.z_partial),
         None, ptr(out.z_dev), None, ptr(ws), ws.numel(), stream())
    res.done()


def repulsive_counts(t: MortonQuadtree, theta: float) -> np.ndarray:
    """Per-point traversal counts (internal visits, leaf-node visits, leaf
    points, accepted) -- the roofline numerator."""
    n = t.n_points
    lib = _lib.load()
    dev = t.arrays.node.device
    dt = t.arrays.dtype
    rep = torch.empty((n, 2), dtype=dt, device=dev)
    cnt = torch.zeros((n, 4), dtype=torch.int32, device=dev)
    ws = _lib.workspace(lib.bh_repulsive_workspace_bytes(n))
    call(_lib.fn("bh_repulsive", dt), t.arrays.sref(), ptr(t.bounds),
         float(theta), None, 0, n, 0, ptr(rep), None, None, None, ptr(cnt),
         ptr(ws), ws.numel(), stream())
    return cnt.cpu().numpy()


def repulsive_exact(y, out: GradientBuffers) -> None:
    """Direct O(N^2) repulsion -- forces.py:153-182."""
    pts = as_points(y)
    n = pts.shape[0]
    if n < 2:
        raise ValueError("need at least 2 points")
    res = _Out(out.rep, pts.dtype)
    lib = _lib.load()
    ws = _lib.workspace(lib.bh_repulsive_exact_workspace_bytes(n))
    call(_lib.fn("bh_repulsive_exact", pts.dtype), ptr(pts), n, ptr(res.t),
         ptr(out.z_partial), ptr(out.z_dev), ptr(ws), ws.numel(), stream())
    res.done()
