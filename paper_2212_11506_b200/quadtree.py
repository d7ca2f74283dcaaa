"""Morton codes and the level-contiguous quadtree on the B200.

Mirrors bhtsne.quadtree (reference: pkg/src/bhtsne/quadtree.py) --
``compute_bounds``, ``morton_codes``, ``build_tree``, ``summarize``,
``morton_interleave``, ``MortonCodes``, ``MortonQuadtree`` -- with the arrays
resident in HBM and every step a CUDA kernel of libbhtsne_b200.so.

Code width: ``code_bits=32`` (default, 16 bits per dimension, depth <= 16,
the north-star layout) or ``64`` (the reference's own width, depth <= 32).
``MortonQuadtree.to_reference()`` returns the reference array layout
(quadtree.py:66-85) for parity checks.

Precision follows the points, as in the reference (whose kernels run on the
arrays' own dtype): float64 points build an f64 tree (f64 centres of mass,
32-byte records) and select the library's ``_f64`` entry points; anything
else runs in float32.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import BOUNDS_DTYPE, call, ptr, stream

DEFAULT_CODE_BITS = 32


def as_points(y, dtype=None) -> torch.Tensor:
    """(N, 2) or (y0, y1) -> contiguous (N, 2) CUDA tensor (quadtree.py:
    122-130 accepts both forms), float64 if the input is float64 (or
    ``dtype`` asks for it), else float32."""
    dev = _lib.device()
    if isinstance(y, tuple):
        y0, y1 = (torch.as_tensor(a) for a in y)
        t = torch.stack([y0.reshape(-1), y1.reshape(-1)], dim=1)
    else:
        t = torch.as_tensor(y)
        if t.ndim != 2 or t.shape[1] != 2:
            raise ValueError(f"expected (N, 2) points, got shape {tuple(t.shape)}")
    if dtype is None:
        dtype = torch.float64 if t.dtype == torch.float64 else torch.float32
    return t.to(device=dev, dtype=_lib.torch_dtype(dtype)).contiguous()


def _bounds_struct(center, r_span, code_bits, shift=(0.0, 0.0)):
    """Host-side bh_bounds_t with _morton_kernel's constants
    (quadtree.py:179-181), identical f64 arithmetic to the device path."""
    scale = (2.0 ** 31 if code_bits == 64 else 2.0 ** 15) / r_span
    return _lib.struct_tensor(BOUNDS_DTYPE, dict(
        c0=center[0], c1=center[1], r_span=r_span, root0=center[0] - r_span,
        root1=center[1] - r_span, scale=scale, shift0=shift[0],
        shift1=shift[1], nonfinite=0, code_bits=code_bits))


def compute_bounds(y, code_bits: int = DEFAULT_CODE_BITS):
    """Bounding square (center, r_span) -- quadtree.py:133-153, on device."""
    pts = as_points(y)
    n = pts.shape[0]
    if n < 1:
        raise ValueError("need at least one point")
    lib = _lib.load()
    out = _lib.struct_tensor(BOUNDS_DTYPE)
    ws = _lib.workspace(lib.bh_bounds_workspace_bytes(n))
    call(_lib.fn("bh_bounds", pts.dtype), ptr(pts), n, code_bits, ptr(out),
         ptr(ws), ws.numel(), stream())
    b = _lib.read_struct(out, BOUNDS_DTYPE)
    if b["nonfinite"]:
        raise ValueError("non-finite coordinate in embedding points")
    return (float(b["c0"]), float(b["c1"])), float(b["r_span"])


def morton_interleave(d0: int, d1: int) -> int:
    """Bit-interleave two integer coordinates (d0 -> even bits, d1 -> odd),
    quadtree.py:172-174 (host helper; the device kernel inlines it)."""
    out = 0
    for bit in range(32):
        out |= ((int(d0) >> bit) & 1) << (2 * bit)
        out |= ((int(d1) >> bit) & 1) << (2 * bit + 1)
    return out


@dataclass(frozen=True)
class MortonCodes:
    """Codes plus the stable Z-order permutation (quadtree.py:55-63).

    Tensors live on the device: ``codes``/``sorted_codes`` hold uint32
    (as int32) or uint64 (as int64) bit patterns; ``order`` is int32."""

    codes: torch.Tensor
    order: torch.Tensor
    center: tuple
    r_span: float
    sorted_codes: torch.Tensor = field(repr=False, default=None)
    code_bits: int = DEFAULT_CODE_BITS
    bounds: torch.Tensor = field(repr=False, default=None)

    def codes_u64(self, which="codes") -> np.ndarray:
        a = getattr(self, which).cpu().numpy()
        return (a.view(np.uint32).astype(np.uint64) if self.code_bits == 32
                else a.view(np.uint64))


def morton_codes(y, center, r_span: float,
                 code_bits: int = DEFAULT_CODE_BITS) -> MortonCodes:
    """Codes and stable radix-sort permutation -- quadtree.py:177-242."""
    if code_bits not in (32, 64):
        raise ValueError("code_bits must be 32 or 64")
    pts = as_points(y)
    n = pts.shape[0]
    lib = _lib.load()
    dt = torch.int32 if code_bits == 32 else torch.int64
    codes = torch.empty(n, dtype=dt, device=pts.device)
    sorted_codes = torch.empty_like(codes)
    order = torch.empty(n, dtype=torch.int32, device=pts.device)
    b = _bounds_struct(center, r_span, code_bits)
    call(_lib.fn("bh_morton", pts.dtype), ptr(pts), n, ptr(b), code_bits, 0,
         ptr(codes), stream())
    ws = _lib.workspace(lib.bh_sort_workspace_bytes(n, code_bits))
    call("bh_sort", ptr(codes), n, code_bits, ptr(sorted_codes), ptr(order),
         ptr(ws), ws.numel(), stream())
    return MortonCodes(codes=codes, order=order,
                       center=(float(center[0]), float(center[1])),
                       r_span=float(r_span), sorted_codes=sorted_codes,
                       code_bits=code_bits, bounds=b)


class TreeArrays:
    """Device storage of one bh_tree_t (caller-owned, reusable)."""

    def __init__(self, n: int, code_bits: int, device, capacity=None,
                 dtype=torch.float32):
        lib = _lib.load()
        self.n = n
        self.code_bits = code_bits
        self.max_depth = code_bits // 2
        self.dtype = _lib.torch_dtype(dtype)
        self.precision = 64 if self.dtype == torch.float64 else 32
        cap = int(capacity or lib.bh_tree_node_bound(n, code_bits))
        self.capacity = cap
        i32 = dict(dtype=torch.int32, device=device)
        # records: 4 x f32 (16 B) or 4 x f64 (32 B: com, then mass|info)
        self.node = torch.zeros((cap, 4), dtype=self.dtype, device=device)
        self.parent = torch.zeros(cap, **i32)
        self.node_start = torch.zeros(cap, **i32)
        self.leaf_end = torch.zeros(cap, **i32)
        self.level_off = torch.zeros(self.max_depth + 3, **i32)
        self.order = torch.zeros(n, **i32)
        self.sorted_codes = torch.zeros(
            n, dtype=torch.int32 if code_bits == 32 else torch.int64,
            device=device)
        self.ys = torch.zeros((n, 2), dtype=self.dtype, device=device)
        self.status = torch.zeros(1, **i32)
        self.ws = _lib.workspace(lib.bh_tree_workspace_bytes(n, code_bits))
        self.struct = _lib.TreeStruct(
            n_points=n, node_capacity=cap, code_bits=code_bits,
            max_depth=self.max_depth, node=self.node.data_ptr(),
            parent=self.parent.data_ptr(),
            node_start=self.node_start.data_ptr(),
            leaf_end=self.leaf_end.data_ptr(),
            level_off=self.level_off.data_ptr(),
            order=self.order.data_ptr(),
            sorted_codes=self.sorted_codes.data_ptr(), ys=self.ys.data_ptr(),
            status=self.status.data_ptr(), precision=self.precision)

    def sref(self):
        return C.byref(self.struct)

    def build(self, pts: torch.Tensor, st=None):
        if pts.dtype != self.dtype or tuple(pts.shape) != (self.n, 2):
            raise ValueError(f"tree is for ({self.n}, 2) {self.dtype} points, "
                             f"got {tuple(pts.shape)} {pts.dtype}")
        call("bh_build_tree", self.sref(), ptr(pts), ptr(self.ws),
             self.ws.numel(), st or stream())

    def summarize(self, st=None):
        call("bh_summarize", self.sref(), ptr(self.ws), self.ws.numel(),
             st or stream())

    def summarize_prefix(self, st=None):
        """All levels from the f64 prefix sums of the sorted points (f32
        trees; see bh_summarize_prefix)."""
        call("bh_summarize_prefix", self.sref(), ptr(self.ws),
             self.ws.numel(), st or stream())


class MortonQuadtree:
    """Level-contiguous quadtree in HBM (quadtree.py:66-119).

    Node records are 16 B {com.x, com.y, mass, info}; see
    include/bhtsne_b200.h.  Host-side views (``level_offsets``, ``mass``,
    ``com``, ...) synchronise; ``to_reference()`` rebuilds the reference
    arrays (start, end, children, is_leaf, cell_center, cell_radius, ...)."""

    def __init__(self, arrays: TreeArrays, mc: MortonCodes, pts: torch.Tensor):
        self.arrays = arrays
        self.mc = mc
        self.points = pts
        self.n_points = arrays.n
        self.center = mc.center
        self.r_span = mc.r_span
        self.code_bits = mc.code_bits
        self.max_depth = arrays.max_depth
        self.bounds = mc.bounds
        self.summarized = False
        st = int(arrays.status.item())
        if st == _lib.BH_ERR_CAPACITY:
            raise RuntimeError("quadtree node capacity exceeded")

    # -- reference-shaped accessors ----------------------------------------
    @property
    def order(self) -> torch.Tensor:
        return self.arrays.order

    @property
    def level_offsets(self) -> np.ndarray:
        lo = self.arrays.level_off.cpu().numpy().astype(np.int64)
        nl = int(lo[self.max_depth + 2])
        return lo[:nl + 1].copy()

    @property
    def n_levels(self) -> int:
        return self.level_offsets.shape[0] - 1

    @property
    def n_nodes(self) -> int:
        return int(self.level_offsets[-1])

    def depths(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_levels, dtype=np.int64),
                         np.diff(self.level_offsets))

    def to_reference(self) -> dict:
        """Arrays in the reference layout (quadtree.py:66-85), numpy."""
        lo = self.level_offsets
        m = int(lo[-1])
        rec = self.arrays.node[:m].cpu().numpy()
        if self.arrays.precision == 64:
            mi = np.ascontiguousarray(rec[:, 2]).view(np.uint32).reshape(m, 2)
            mass, info = (mi[:, 0].astype(np.int64), mi[:, 1].astype(np.int64))
        else:
            info = rec[:, 3].view(np.uint32).astype(np.int64)
            mass = rec[:, 2].astype(np.int64)  # f32 records: float count
        is_leaf = ((info & _lib.BH_LEAF_BIT) != 0).astype(np.uint8)
        start = self.arrays.node_start[:m].cpu().numpy().astype(np.int64)
        parent = self.arrays.parent[:m].cpu().numpy().astype(np.int64)
        leaf_end = self.arrays.leaf_end[:m].cpu().numpy().astype(np.int64)
        depth = self.depths()
        end = np.where(is_leaf == 1, leaf_end, -1)
        for lvl in range(self.n_levels - 1, 0, -1):
            sl = slice(lo[lvl], lo[lvl + 1])
            np.maximum.at(end, parent[sl], end[sl])
        sc = self.mc.codes_u64("sorted_codes")
        width = 2 * self.max_depth
        children = np.full((m, 4), -1, np.int64)
        center = np.empty((m, 2), np.float64)
        radius = np.empty(m, np.float64)
        center[0] = self.center
        radius[0] = self.r_span
        for lvl in range(1, self.n_levels):
            ids = np.arange(lo[lvl], lo[lvl + 1])
            p = parent[ids]
            v = ((sc[start[ids]] >> np.uint64(width - 2 * lvl))
                 & np.uint64(3)).astype(np.int64)
            children[p, v] = ids
            half = radius[p] * 0.5
            radius[ids] = half
            center[ids, 0] = center[p, 0] + np.where(v & 1, half, -half)
            center[ids, 1] = center[p, 1] + np.where(v & 2, half, -half)
        ys = self.arrays.ys.cpu().numpy()
        out = dict(level_offsets=lo, start=start, end=end, children=children,
                   is_leaf=is_leaf, cell_center=center, cell_radius=radius,
                   mass=mass if self.summarized else np.zeros(m, np.int64),
                   com=rec[:, :2].copy() if self.summarized
                   else np.zeros((m, 2), rec.dtype),
                   order=self.order.cpu().numpy().astype(np.int64),
                   ys0=ys[:, 0].copy(), ys1=ys[:, 1].copy(), depth=depth,
                   sorted_codes=sc)
        return out

    def dump(self) -> str:
        """quadtree.py:101-113 textual dump (depth, prefix, count, com)."""
        if not self.summarized:
            raise ValueError("tree must be summarized before dumping")
        r = self.to_reference()
        width = 2 * self.max_depth
        lines = []
        for nd in range(r["start"].shape[0]):
            d = int(r["depth"][nd])
            prefix = "-" if d == 0 else format(
                int(r["sorted_codes"][r["start"][nd]]) >> (width - 2 * d),
                f"0{2 * d}b")
            lines.append("{} {} {} {:.12g} {:.12g}".format(
                d, prefix, int(r["end"][nd] - r["start"][nd]),
                float(r["com"][nd, 0]), float(r["com"][nd, 1])))
        return "\n".join(lines)


def build_tree(mc: MortonCodes, y, capacity=None) -> MortonQuadtree:
    """Build the canonical quadtree over the sorted codes (quadtree.py:399)."""
    pts = as_points(y)
    arrays = TreeArrays(pts.shape[0], mc.code_bits, pts.device, capacity,
                        dtype=pts.dtype)
    arrays.order.copy_(mc.order)
    arrays.sorted_codes.copy_(mc.sorted_codes)
    arrays.build(pts)
    return MortonQuadtree(arrays, mc, pts)


def summarize(t: MortonQuadtree) -> MortonQuadtree:
    """Fill mass and centre of mass bottom-up (quadtree.py:511-519)."""
    t.arrays.summarize()
    t.summarized = True
    return t
