"""CPU oracle for the B200 Barnes-Hut t-SNE hot path.

TEST INFRASTRUCTURE ONLY.  Imported by ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s CPU-baseline leg as the checker; never by the product
package ``paper_2212_11506_b200``.

The compute lives in ``bh_oracle.c`` (a C/OpenMP restatement of the reference
``bhtsne`` kernels, loaded through ctypes); this module adds the numpy parts
of the reference that are plain array programs:

* ``knn_exact``       -- knn.py:36-59 (f64 distances, ties -> lower id)
* ``symmetrize``      -- affinity.py:121-158 (lexsort/reduceat CSR)
* ``set_exaggeration``-- affinity.py:161-173
* ``init_embedding``  -- optimizer.py:147-158 (numpy Philox)

Parity pin: tests/test_oracle.py checks all of it against golden vectors made
by the unmodified reference (tests/golden/make_golden.py).  All paths above
are relative to /root/reference/pkg/src/bhtsne/.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libbh_oracle.so")
_lib = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile bh_oracle.c with the committed Makefile (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH)
            < os.path.getmtime(os.path.join(_HERE, "bh_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    L.or_set_threads.argtypes = [C.c_int]
    L.or_set_threads.restype = C.c_int
    L.or_num_threads.restype = C.c_int
    L.or_bounds.argtypes = [_f32p, _f32p, C.c_int64, _f64p]
    L.or_bounds.restype = C.c_int
    L.or_interleave.argtypes = [C.c_uint64, C.c_uint64]
    L.or_interleave.restype = C.c_uint64
    L.or_morton.argtypes = [_f32p, _f32p, C.c_int64, C.c_double, C.c_double,
                            C.c_double, C.c_int, _u64p]
    L.or_radix_argsort.argtypes = [_u64p, C.c_int64, C.c_int, _i64p, _u64p]
    L.or_build_tree.argtypes = [_u64p, C.c_int64, C.c_int, C.c_double,
                                C.c_double, C.c_double]
    L.or_build_tree.restype = C.c_void_p
    L.or_tree_free.argtypes = [C.c_void_p]
    L.or_tree_dims.argtypes = [C.c_void_p, _i64p]
    L.or_tree_copy.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _i64p, _u8p,
                               _f64p, _f64p, _i64p, _f32p]
    L.or_summarize.argtypes = [C.c_void_p, _f32p, _f32p]
    L.or_attractive.argtypes = [_i64p, _i64p, _f32p, _f32p, _f32p, C.c_int64,
                                _f32p, _f32p]
    L.or_repulsive_bh.argtypes = [C.c_void_p, _i64p, _f32p, _f32p, _f32p,
                                  _f32p, C.c_int64, C.c_double, _f32p, _f32p,
                                  _f64p, C.c_void_p]
    L.or_repulsive_exact.argtypes = [_f32p, _f32p, C.c_int64, _f32p, _f32p,
                                     _f64p]
    L.or_calibrate.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_double,
                               C.c_double, C.c_int64, _f64p, _f64p]
    L.or_kl_rows.argtypes = [_i64p, _i64p, _f32p, _f32p, _f32p, C.c_int64,
                             C.c_double, _f64p]
    L.or_update.argtypes = [_f32p] * 10 + [C.c_double, C.c_int64, C.c_double,
                                           C.c_double, C.c_double]
    L.or_update.restype = C.c_int64
    L.or_gradient_step.argtypes = [_f32p] * 6 + [_i64p, _i64p, _f32p,
                                                 C.c_int64, C.c_double,
                                                 C.c_double, C.c_double,
                                                 C.c_double, C.c_int,
                                                 C.c_void_p]
    L.or_gradient_step.restype = C.c_int64
    _lib = L
    return L


def set_threads(t: int | None) -> int:
    return lib().or_set_threads(int(t or 0))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def split_xy(y):
    if isinstance(y, tuple):
        return _f32(y[0]), _f32(y[1])
    y = np.asarray(y)
    return _f32(y[:, 0]), _f32(y[:, 1])


# --- bounds / morton / sort (quadtree.py:133-242) ---------------------------

def compute_bounds(y):
    y0, y1 = split_xy(y)
    out = np.zeros(3)
    rc = lib().or_bounds(y0, y1, y0.shape[0], out)
    if rc == -1:
        raise ValueError("non-finite coordinate in embedding points")
    if rc != 0:
        raise ValueError("need at least one point")
    return (float(out[0]), float(out[1])), float(out[2])


def morton_interleave(d0: int, d1: int) -> int:
    return int(lib().or_interleave(d0, d1))


def morton_codes(y, center, r_span, code_bits: int = 64):
    y0, y1 = split_xy(y)
    n = y0.shape[0]
    codes = np.empty(n, np.uint64)
    lib().or_morton(y0, y1, n, float(center[0]), float(center[1]),
                    float(r_span), code_bits, codes)
    order = np.empty(n, np.int64)
    sc = np.empty(n, np.uint64)
    lib().or_radix_argsort(codes, n, code_bits, order, sc)
    return codes, order, sc


# --- tree (quadtree.py:399-519) ---------------------------------------------

@dataclass
class OracleTree:
    """Reference-layout tree arrays (quadtree.py:66-85)."""

    n_points: int
    max_depth: int
    level_offsets: np.ndarray
    start: np.ndarray
    end: np.ndarray
    children: np.ndarray
    is_leaf: np.ndarray
    cell_center: np.ndarray
    cell_radius: np.ndarray
    mass: np.ndarray
    com: np.ndarray
    order: np.ndarray
    sorted_codes: np.ndarray
    ys0: np.ndarray
    ys1: np.ndarray
    _handle: int = 0

    @property
    def n_nodes(self):
        return self.start.shape[0]

    @property
    def n_levels(self):
        return self.level_offsets.shape[0] - 1

    def depths(self):
        return np.repeat(np.arange(self.n_levels, dtype=np.int64),
                         np.diff(self.level_offsets))

    def __del__(self):
        if self._handle and _lib is not None:
            _lib.or_tree_free(self._handle)
            self._handle = 0


def build_tree(y, code_bits: int = 64, summarized: bool = True):
    """bounds -> codes -> stable sort -> tree (-> summarize), reference-style."""
    y0, y1 = split_xy(y)
    center, r_span = compute_bounds((y0, y1))
    codes, order, sc = morton_codes((y0, y1), center, r_span, code_bits)
    return tree_from_sorted(sc, order, (y0, y1), center, r_span, code_bits,
                            summarized=summarized, codes=codes)


def tree_from_sorted(sc, order, y, center, r_span, code_bits=64,
                     summarized=True, codes=None):
    y0, y1 = split_xy(y)
    L = lib()
    n = y0.shape[0]
    h = L.or_build_tree(np.ascontiguousarray(sc, np.uint64), n, code_bits,
                        float(center[0]), float(center[1]), float(r_span))
    dims = np.zeros(4, np.int64)
    L.or_tree_dims(h, dims)
    m, nl = int(dims[1]), int(dims[2])
    lo = np.empty(nl + 1, np.int64)
    start = np.empty(m, np.int64)
    end = np.empty(m, np.int64)
    ch = np.empty((m, 4), np.int64)
    leaf = np.empty(m, np.uint8)
    cen = np.empty((m, 2), np.float64)
    rad = np.empty(m, np.float64)
    ys0 = np.ascontiguousarray(y0[order])
    ys1 = np.ascontiguousarray(y1[order])
    if summarized:
        L.or_summarize(h, ys0, ys1)
    mass = np.empty(m, np.int64)
    com = np.empty((m, 2), np.float32)
    L.or_tree_copy(h, lo, start, end, ch, leaf, cen, rad, mass, com)
    t = OracleTree(n_points=n, max_depth=int(dims[3]), level_offsets=lo,
                   start=start, end=end, children=ch, is_leaf=leaf,
                   cell_center=cen, cell_radius=rad, mass=mass, com=com,
                   order=np.ascontiguousarray(order, np.int64),
                   sorted_codes=np.ascontiguousarray(sc, np.uint64),
                   ys0=ys0, ys1=ys1, _handle=h)
    t.codes = codes
    return t


def tree_dump(t: OracleTree) -> str:
    """quadtree.py:101-113 dump format (depth, prefix bits, count, com)."""
    depths = t.depths()
    width = 2 * t.max_depth
    lines = []
    for nd in range(t.n_nodes):
        d = int(depths[nd])
        prefix = "-" if d == 0 else format(
            int(t.sorted_codes[t.start[nd]]) >> (width - 2 * d), f"0{2 * d}b")
        lines.append("{} {} {} {:.12g} {:.12g}".format(
            d, prefix, int(t.end[nd] - t.start[nd]), float(t.com[nd, 0]),
            float(t.com[nd, 1])))
    return "\n".join(lines)


# --- forces (forces.py) -----------------------------------------------------

def attractive(row_offsets, col_indices, values, y, n_rows=None):
    """forces.py:56-82; rows [0, n_rows) (default: one per point)."""
    y0, y1 = split_xy(y)
    n = y0.shape[0] if n_rows is None else int(n_rows)
    a0 = np.empty(n, np.float32)
    a1 = np.empty(n, np.float32)
    lib().or_attractive(np.ascontiguousarray(row_offsets, np.int64),
                        np.ascontiguousarray(col_indices, np.int64),
                        _f32(values), y0, y1, n, a0, a1)
    return a0, a1


def repulsive_bh(t: OracleTree, y, theta: float, counts: bool = False):
    y0, y1 = split_xy(y)
    n = y0.shape[0]
    r0 = np.empty(n, np.float32)
    r1 = np.empty(n, np.float32)
    zp = np.empty(n, np.float64)
    cnt = np.zeros((n, 6), np.int64) if counts else None
    lib().or_repulsive_bh(t._handle, t.order, t.ys0, t.ys1, y0, y1, n,
                          float(theta), r0, r1, zp,
                          cnt.ctypes.data if counts else None)
    out = (r0, r1, zp, float(np.sum(zp)))
    return out + (cnt,) if counts else out


def repulsive_exact(y):
    y0, y1 = split_xy(y)
    n = y0.shape[0]
    r0 = np.empty(n, np.float32)
    r1 = np.empty(n, np.float32)
    zp = np.empty(n, np.float64)
    lib().or_repulsive_exact(y0, y1, n, r0, r1, zp)
    return r0, r1, zp, float(np.sum(zp))


# --- affinities (affinity.py, knn.py) ---------------------------------------

def knn_exact(x: np.ndarray, k: int):
    """Restates knn.py:36-59: f64 squared distances summed over columns in
    order, k smallest per row, ties -> lower id (stable sort), self excluded.
    Returns (indices int64 (N,k), sq_distances in x.dtype)."""
    x = np.ascontiguousarray(x)
    n = x.shape[0]
    xd = x.astype(np.float64)
    idx = np.empty((n, k), np.int64)
    sqd = np.empty((n, k), np.float64)
    block = max(1, min(n, 2_000_000 // max(n, 1)))
    for s in range(0, n, block):
        e = min(n, s + block)
        acc = np.zeros((e - s, n))
        for c in range(x.shape[1]):
            diff = xd[s:e, c][:, None] - xd[None, :, c]
            acc += diff * diff
        acc[np.arange(e - s), np.arange(s, e)] = np.inf
        order = np.argsort(acc, axis=1, kind="stable")[:, :k]
        idx[s:e] = order
        sqd[s:e] = np.take_along_axis(acc, order, axis=1)
    return idx, sqd.astype(x.dtype)


def calibrate_perplexity(sqd, u: float, max_iter: int = 200,
                         tol: float = 1e-5):
    sqd = _f32(sqd)
    n, k = sqd.shape
    cond = np.empty((n, k), np.float64)
    betas = np.empty(n, np.float64)
    lib().or_calibrate(sqd, n, k, math.log(u), tol * math.log(2.0), max_iter,
                       cond, betas)
    return betas, cond


def symmetrize(indices, cond, dtype=np.float32):
    """affinity.py:121-158 restated: (row_offsets int64, cols int64, vals)."""
    n, k = indices.shape
    rows = np.repeat(np.arange(n, dtype=np.int64), k)
    cols = np.asarray(indices).ravel().astype(np.int64)
    vals = np.asarray(cond, np.float64).ravel()
    ri = np.concatenate([rows, cols])
    ci = np.concatenate([cols, rows])
    vi = np.concatenate([vals, vals])
    order = np.lexsort((ci, ri))
    ri, ci, vi = ri[order], ci[order], vi[order]
    first = np.ones(ri.shape[0], dtype=bool)
    first[1:] = (ri[1:] != ri[:-1]) | (ci[1:] != ci[:-1])
    starts = np.flatnonzero(first)
    summed = np.add.reduceat(vi, starts)
    values = np.maximum(summed / (2.0 * n),
                        np.finfo(np.float64).eps).astype(dtype)
    out_rows = ri[starts]
    row_offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(out_rows, minlength=n), out=row_offsets[1:])
    return row_offsets, ci[starts].copy(), values


def exaggerate(values, factor: float):
    """affinity.py:161-173: base * dtype(factor); factor 1 -> pristine."""
    values = np.asarray(values)
    return values if factor == 1.0 else values * values.dtype.type(factor)


def init_embedding(n: int, seed: int, dtype=np.float32):
    """optimizer.py:147-158: Philox(seed) standard normal * 1e-4."""
    rng = np.random.Generator(np.random.Philox(seed))
    y = (rng.standard_normal((n, 2)) * 1e-4).astype(dtype)
    return np.ascontiguousarray(y[:, 0]), np.ascontiguousarray(y[:, 1])


def kl_divergence(row_offsets, col_indices, values, y, z=None):
    """optimizer.py:242-270, exact mode: Z from the O(N^2) pass."""
    y0, y1 = split_xy(y)
    if z is None:
        z = repulsive_exact((y0, y1))[3]
    n = y0.shape[0]
    part = np.empty(n, np.float64)
    lib().or_kl_rows(np.ascontiguousarray(row_offsets, np.int64),
                     np.ascontiguousarray(col_indices, np.int64),
                     _f32(values), y0, y1, n, float(z), part)
    return float(np.sum(part))


# --- optimizer (optimizer.py:161-224) ---------------------------------------

@dataclass
class State:
    y0: np.ndarray
    y1: np.ndarray
    v0: np.ndarray
    v1: np.ndarray
    g0: np.ndarray
    g1: np.ndarray
    iteration: int = 0

    @classmethod
    def init(cls, n, seed):
        y0, y1 = init_embedding(n, seed)
        z = lambda: np.zeros(n, np.float32)
        o = lambda: np.ones(n, np.float32)
        return cls(y0, y1, z(), z(), o(), o())

    def copy(self):
        return State(*(a.copy() for a in (self.y0, self.y1, self.v0, self.v1,
                                          self.g0, self.g1)), self.iteration)


def update(s: State, attr, rep, z, momentum, lr=200.0, min_gain=0.01):
    rc = lib().or_update(s.y0, s.y1, s.v0, s.v1, s.g0, s.g1,
                         _f32(attr[0]), _f32(attr[1]), _f32(rep[0]),
                         _f32(rep[1]), float(z), s.y0.shape[0],
                         float(momentum), float(lr), float(min_gain))
    if rc < 0:
        raise ValueError(f"non-finite gradient at point {-1 - rc} "
                         f"(iteration {s.iteration})")
    s.iteration += 1


def gradient(y, row_offsets, cols, vals, theta, code_bits=64):
    """Forces of one iteration: (grad0, grad1, attr, rep, z) in f32 numpy
    semantics (optimizer.py:203-207)."""
    y0, y1 = split_xy(y)
    t = build_tree((y0, y1), code_bits=code_bits)
    a0, a1 = attractive(row_offsets, cols, vals, (y0, y1))
    r0, r1, zp, z = repulsive_bh(t, (y0, y1), theta)
    zf = np.float32(z)
    g0 = np.float32(4.0) * (a0 - r0 / zf)
    g1 = np.float32(4.0) * (a1 - r1 / zf)
    return g0, g1, (a0, a1), (r0, r1), z


def gradient_step(s: State, row_offsets, cols, vals, theta=0.5,
                  momentum_early=0.5, momentum_late=0.8, lr=200.0,
                  min_gain=0.01, code_bits=64, stage_s=None):
    momentum = momentum_early if s.iteration < 250 else momentum_late
    st = np.zeros(5) if stage_s is None else stage_s
    rc = lib().or_gradient_step(
        s.y0, s.y1, s.v0, s.v1, s.g0, s.g1,
        np.ascontiguousarray(row_offsets, np.int64),
        np.ascontiguousarray(cols, np.int64), _f32(vals), s.y0.shape[0],
        float(theta), float(momentum), float(lr), float(min_gain),
        int(code_bits), st.ctypes.data)
    if rc == -2:
        raise ValueError("non-finite coordinate in embedding points")
    if rc < 0:
        raise ValueError(f"non-finite gradient at point {-1 - rc} "
                         f"(iteration {s.iteration})")
    s.iteration += 1
    return st


def run(indices, sqd, n_iter=1000, perplexity=30.0, theta=0.5,
        early_exaggeration=12.0, exaggeration_iters=250, lr=200.0,
        momentum_early=0.5, momentum_late=0.8, min_gain=0.01, seed=0,
        code_bits=64, kl=True):
    """optimizer.py:289-332 on a precomputed kNN graph (f32 run mode)."""
    betas, cond = calibrate_perplexity(sqd, perplexity)
    ro, co, va = symmetrize(indices, cond, np.float32)
    n = indices.shape[0]
    s = State.init(n, seed)
    exag = n_iter > 0 and exaggeration_iters > 0
    for it in range(n_iter):
        v = exaggerate(va, early_exaggeration) if (
            exag and it < exaggeration_iters) else va
        gradient_step(s, ro, co, v, theta, momentum_early, momentum_late, lr,
                      min_gain, code_bits)
    out = kl_divergence(ro, co, va, (s.y0, s.y1)) if kl else None
    return s, out, (ro, co, va, betas)
