"""ctypes binding of libbhtsne_b200.so (include/bhtsne_b200.h).

The library is the only compute path: there is no CPU fallback.  Loading
fails loudly when the shared object is missing or no CUDA device is present.
torch supplies device memory and streams; no torch type crosses the ABI.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# BH_LIB overrides the library path (A/B builds in tools/microbench.py)
LIB_PATH = os.environ.get("BH_LIB") or os.path.join(HERE, "libbhtsne_b200.so")

_lib = None

BH_LEAF_BIT = 0x80000000
BH_CHILD_MASK = 0x1FFFFFFF
BH_NKIDS_SHIFT = 29
BH_ERR_CAPACITY = -3

# device-resident structs, viewed through numpy structured dtypes
BOUNDS_DTYPE = np.dtype([
    ("c0", "f8"), ("c1", "f8"), ("r_span", "f8"), ("root0", "f8"),
    ("root1", "f8"), ("scale", "f8"), ("shift0", "f4"), ("shift1", "f4"),
    ("nonfinite", "i4"), ("code_bits", "i4"), ("shift0_f64", "f8"),
    ("shift1_f64", "f8")])
SCHED_DTYPE = np.dtype([
    ("iteration", "i4"), ("exaggeration_iters", "i4"),
    ("momentum_switch", "i4"), ("pad0", "i4"), ("exaggeration", "f4"),
    ("momentum_early", "f4"), ("momentum_late", "f4"),
    ("learning_rate", "f4"), ("min_gain", "f4"), ("pad1", "f4"),
    ("bad", "i8"), ("z", "f8"), ("exaggeration_f64", "f8"),
    ("momentum_early_f64", "f8"), ("momentum_late_f64", "f8"),
    ("learning_rate_f64", "f8"), ("min_gain_f64", "f8")])
assert BOUNDS_DTYPE.itemsize == 80 and SCHED_DTYPE.itemsize == 96
INT64_MAX = np.iinfo(np.int64).max


class TreeStruct(C.Structure):
    """bh_tree_t: host struct of device pointers."""

    _fields_ = [
        ("n_points", C.c_int64), ("node_capacity", C.c_int64),
        ("code_bits", C.c_int32), ("max_depth", C.c_int32),
        ("node", C.c_void_p), ("parent", C.c_void_p),
        ("node_start", C.c_void_p), ("leaf_end", C.c_void_p),
        ("level_off", C.c_void_p), ("order", C.c_void_p),
        ("sorted_codes", C.c_void_p), ("ys", C.c_void_p),
        ("status", C.c_void_p),
        ("rank", C.c_void_p),
        ("precision", C.c_int32), ("pad", C.c_int32),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_SZ = C.c_size_t

SIGNATURES = {
    "bh_last_error": ([], C.c_char_p),
    "bh_abi_version": ([], C.c_int),
    "bh_tree_node_bound": ([_I64, C.c_int], _I64),
    "bh_bounds_workspace_bytes": ([_I64], _SZ),
    "bh_bounds": ([_P, _I64, C.c_int, _P, _P, _SZ, _P], C.c_int),
    "bh_morton": ([_P, _I64, _P, C.c_int, C.c_int, _P, _P], C.c_int),
    "bh_hilbert": ([_P, _I64, _P, C.c_int, C.c_int, _P, _P], C.c_int),
    "bh_hilbert_f64": ([_P, _I64, _P, C.c_int, C.c_int, _P, _P], C.c_int),
    "bh_sort_workspace_bytes": ([_I64, C.c_int], _SZ),
    "bh_sort": ([_P, _I64, C.c_int, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_sort_pairs": ([_P, _P, _I64, C.c_int, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_tree_workspace_bytes": ([_I64, C.c_int], _SZ),
    "bh_build_tree": ([C.POINTER(TreeStruct), _P, _P, _SZ, _P], C.c_int),
    "bh_summarize": ([C.POINTER(TreeStruct), _P, _SZ, _P], C.c_int),
    "bh_summarize_prefix": ([C.POINTER(TreeStruct), _P, _SZ, _P], C.c_int),
    "bh_attractive": ([_P, _P, _P, _I64, C.c_int, _P, _I64, _I64, C.c_float,
                       _P, _P, _P], C.c_int),
    "bh_repulsive_workspace_bytes": ([_I64], _SZ),
    "bh_repulsive": ([C.POINTER(TreeStruct), _P, C.c_double, _P, _I64, _I64,
                      C.c_int, _P, _P, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_forces": ([C.POINTER(TreeStruct), _P, C.c_double, _I64, _I64, C.c_int,
                   _P, _P, _P, _P, _SZ, _P, _P, _P, _I64, C.c_int, _P, _I64,
                   _I64, C.c_float, _P, _P, _P], C.c_int),
    "bh_sum_partials": ([_P, _I64, _P, _P], C.c_int),
    "bh_forces_f64": ([C.POINTER(TreeStruct), _P, C.c_double, _I64, _I64,
                       C.c_int, _P, _P, _P, _P, _SZ, _P, _P, _P, _I64, C.c_int,
                       _P, _I64, _I64, C.c_double, _P, _P, _P], C.c_int),
    "bh_attractive_f64": ([_P, _P, _P, _I64, C.c_int, _P, _I64, _I64,
                           C.c_double, _P, _P, _P], C.c_int),
    "bh_repulsive_f64": ([C.POINTER(TreeStruct), _P, C.c_double, _P, _I64,
                          _I64, C.c_int, _P, _P, _P, _P, _P, _P, _SZ, _P],
                         C.c_int),
    "bh_repulsive_exact_f64": ([_P, _I64, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_kl_rows_f64": ([_P, _P, _P, _I64, C.c_int, _P, _P, _P, _P, _SZ, _P],
                       C.c_int),
    "bh_bounds_f64": ([_P, _I64, C.c_int, _P, _P, _SZ, _P], C.c_int),
    "bh_morton_f64": ([_P, _I64, _P, C.c_int, C.c_int, _P, _P], C.c_int),
    "bh_update_f64": ([_P, _P, _P, _P, _P, _P, _I64, _P, _P, C.c_int, _P,
                       _SZ, _P], C.c_int),
    "bh_center_f64": ([_P, _I64, _P, _P], C.c_int),
    "bh_bsp_f64": ([_P, _I64, _I64, C.c_double, C.c_double, _I64, _P, _P,
                    _P], C.c_int),
    "bh_symmetrize_fill_f64": ([_P, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P],
                               C.c_int),
    "bh_pad_csr_fill_f64": ([_P, _P, _P, _I64, _P, _P, _P, _P], C.c_int),
    "bh_permute_csr_f64": ([_P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _SZ,
                            _P], C.c_int),
    "bh_knn_f64": ([_P, _I64, _I64, _I64, _P, _P, _P], C.c_int),
    "bh_repulsive_exact_workspace_bytes": ([_I64], _SZ),
    "bh_repulsive_exact": ([_P, _I64, _P, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_kl_workspace_bytes": ([_I64], _SZ),
    "bh_kl_rows": ([_P, _P, _P, _I64, C.c_int, _P, _P, _P, _P, _SZ, _P],
                   C.c_int),
    "bh_update_workspace_bytes": ([_I64], _SZ),
    "bh_update": ([_P, _P, _P, _P, _P, _P, _I64, _P, _P, C.c_int, _P, _SZ,
                   _P], C.c_int),
    "bh_center": ([_P, _I64, _P, _P], C.c_int),
    "bh_bsp": ([_P, _I64, _I64, C.c_double, C.c_double, _I64, _P, _P, _P],
               C.c_int),
    "bh_symmetrize_workspace_bytes": ([_I64, _I64], _SZ),
    "bh_symmetrize_plan": ([_P, _I64, _I64, _P, _P, _SZ, _P], C.c_int),
    "bh_symmetrize_fill": ([_P, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P],
                           C.c_int),
    "bh_pad_csr_workspace_bytes": ([_I64], _SZ),
    "bh_pad_csr_size": ([_P, _I64, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_pad_csr_fill": ([_P, _P, _P, _I64, _P, _P, _P, _P], C.c_int),
    "bh_knn": ([_P, _I64, _I64, _I64, _P, _P, _P], C.c_int),
    "bh_knn_general_workspace_bytes": ([_I64, _I64], _SZ),
    "bh_knn_general": ([_P, _I64, _I64, _I64, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_knn_general_f64": ([_P, _I64, _I64, _I64, _P, _P, _P, _SZ, _P],
                           C.c_int),
    "bh_knn_f64_filtered": ([_P, _P, _I64, _I64, _I64, _P, _P, _P, _SZ, _P],
                            C.c_int),
    "bh_gather_rows": ([_P, _P, _I64, C.c_int, _P, _P], C.c_int),
    "bh_scatter_rows": ([_P, _P, _I64, C.c_int, _P, _P], C.c_int),
    "bh_invert_perm": ([_P, _I64, _P, _P], C.c_int),
    "bh_partition": ([_P, _I64, C.c_int, C.c_double, C.c_double, _I64, _P,
                      _P, _P], C.c_int),
    "bh_step_attractive": ([_P, _P, _P, C.c_int, _P, _P, _I64, _P, _P, _P],
                           C.c_int),
    "bh_step_attractive_f64": ([_P, _P, _P, C.c_int, _P, _P, _I64, _P, _P,
                                _P], C.c_int),
    "bh_step_forces": ([C.POINTER(TreeStruct), _P, C.c_double, _P, _P, _P,
                        _P, _I64, C.c_int, _P, _P, _P, _SZ, _P, _P, _P,
                        C.c_int, _P, _P, _P], C.c_int),
    "bh_step_forces_f64": ([C.POINTER(TreeStruct), _P, C.c_double, _P, _P,
                            _P, _P, _I64, C.c_int, _P, _P, _P, _SZ, _P, _P,
                            _P, C.c_int, _P, _P, _P], C.c_int),
    "bh_step_qlist_workspace_bytes": ([_I64], _SZ),
    "bh_step_qlist": ([_P, _I64, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_step_zsum_workspace_bytes": ([_I64], _SZ),
    "bh_step_zsum": ([_P, _P, _I64, _I64, _P, _P, _P, _SZ, _P], C.c_int),
    "bh_step_update": ([_P, _P, _P, _P, _P, _P, _I64, _P, _P, C.c_int,
                        C.c_int, _P, _P, _SZ, _P], C.c_int),
    "bh_step_update_f64": ([_P, _P, _P, _P, _P, _P, _I64, _P, _P, C.c_int,
                            C.c_int, _P, _P, _SZ, _P], C.c_int),
    "bh_step_finish": ([_P, _I64, _P, _P, C.c_int, _P, _SZ, _P], C.c_int),
    "bh_step_finish_f64": ([_P, _I64, _P, _P, C.c_int, _P, _SZ, _P],
                           C.c_int),
    "bh_pack_rows": ([_P, _P, _I64, C.c_int, _P, _P], C.c_int),
    "bh_unpack_rows": ([_P, _I64, _P, C.c_int, C.c_int, _P, _P], C.c_int),
    "bh_permute_csr_workspace_bytes": ([_I64], _SZ),
    "bh_permute_csr": ([_P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _SZ, _P],
                       C.c_int),
}


def load(require_device: bool = True):
    """Load the CUDA library (raises if it is missing; no fallback)."""
    global _lib
    if require_device and not torch.cuda.is_available():
        raise RuntimeError("paper_2212_11506_b200 needs a CUDA device (B200, "
                           "sm_100a); there is no CPU fallback")
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.bh_abi_version() != 1:
        raise RuntimeError("libbhtsne_b200 ABI version mismatch")
    _lib = lib
    return lib


def load_symbols_only():
    """Load without requiring a device (used by the CPU ABI tests)."""
    return load(require_device=False)


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = _lib.bh_last_error().decode(errors="replace") if _lib else ""
        if rc == -1:
            raise ValueError(msg or what)
        raise RuntimeError(f"{what}: {msg} (code {rc})")


def call(name: str, *args):
    lib = load()
    check(getattr(lib, name)(*args), name)


# Run precision: the reference's dtype (io.py:21-30).  f64 tensors select the
# library's `_f64` entry points.
DTYPES = {"f32": torch.float32, "f64": torch.float64}


def is_f64(t) -> bool:
    dt = t.dtype if isinstance(t, torch.Tensor) else t
    return dt in (torch.float64, np.float64, np.dtype(np.float64))


def fn(name: str, dtype) -> str:
    """Entry point for a run precision: bh_x or bh_x_f64."""
    return name + "_f64" if is_f64(dtype) else name


def torch_dtype(dtype) -> torch.dtype:
    """numpy/torch/str precision -> torch.float32 | torch.float64."""
    if isinstance(dtype, str):
        if dtype not in DTYPES:
            raise ValueError(f"unknown precision {dtype!r}; expected one of "
                             f"{sorted(DTYPES)}")
        return DTYPES[dtype]
    if isinstance(dtype, torch.dtype):
        dt = dtype
    else:
        dt = {np.dtype(np.float32): torch.float32,
              np.dtype(np.float64): torch.float64}.get(np.dtype(dtype))
    if dt not in (torch.float32, torch.float64):
        raise ValueError(f"unsupported dtype {dtype}; expected float32 or "
                         "float64")
    return dt


def ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def device() -> torch.device:
    load()
    return torch.device("cuda", torch.cuda.current_device())


def workspace(nbytes: int) -> torch.Tensor:
    """Zero-filled scratch (the library leaves its counters at zero)."""
    return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8,
                       device=device())


def struct_tensor(dtype: np.dtype, values: dict | None = None) -> torch.Tensor:
    host = np.zeros(1, dtype)
    for k, v in (values or {}).items():
        host[k] = v
    t = torch.from_numpy(host.view(np.uint8).copy())
    return t.to(device())


def read_struct(t: torch.Tensor, dtype: np.dtype):
    return t.cpu().numpy().view(dtype)[0]
