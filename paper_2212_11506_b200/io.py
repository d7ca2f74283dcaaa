"""Dense matrix files: the reference's BHTM binary and CSV formats.

Same on-disk formats as bhtsne.io (reference pkg/src/bhtsne/io.py:1-30,
131-190) so files move freely between the two packages and the TypeScript
estimator (frontend/src/binary.ts):

* BHTM: magic ``b"BHTM"``, one u8 dtype tag (0 = f64, 1 = f32), u64 rows,
  u64 columns, then the values row-major, all little-endian;
* CSV: one row per line, comma separated, optional header line.

Host-side file I/O only (no compute).
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"BHTM"
_HEADER = struct.Struct("<4sBQQ")
_TAGS = {0: np.dtype("<f8"), 1: np.dtype("<f4")}
PRECISIONS = {"f32": np.dtype(np.float32), "f64": np.dtype(np.float64)}


def precision_dtype(precision: str) -> np.dtype:
    try:
        return PRECISIONS[precision]
    except KeyError:
        raise ValueError(f"unknown precision {precision!r}; expected one of "
                         f"{sorted(PRECISIONS)}") from None


@dataclass(frozen=True)
class InputMatrix:
    """A validated dense N x D dataset (io.py:33-65 rules)."""

    data: np.ndarray

    def __post_init__(self):
        a = self.data
        if a.ndim != 2:
            raise ValueError(f"expected a 2-D matrix, got {a.ndim}-D")
        if a.shape[0] < 2:
            raise ValueError(f"matrix must have at least 2 rows, got {a.shape[0]}")
        if a.shape[1] < 1:
            raise ValueError("matrix must have at least 1 column")
        if a.dtype not in (np.float32, np.float64):
            raise ValueError(f"unsupported dtype {a.dtype}")
        bad = np.argwhere(~np.isfinite(a))
        if bad.size:
            r, c = bad[0]
            raise ValueError(f"non-finite value at row {r}, column {c}")

    @property
    def n_points(self) -> int:
        return self.data.shape[0]

    @property
    def n_dims(self) -> int:
        return self.data.shape[1]


def sniff_format(path) -> str:
    with open(path, "rb") as fh:
        return "bin" if fh.read(4) == MAGIC else "csv"


def read_bhtm(path) -> np.ndarray:
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
        if len(head) < _HEADER.size:
            raise ValueError(f"{path}: not a BHTM binary matrix file")
        magic, tag, n, d = _HEADER.unpack(head)
        if magic != MAGIC:
            raise ValueError(f"{path}: not a BHTM binary matrix file")
        if tag not in _TAGS:
            raise ValueError(f"{path}: unknown dtype tag {tag}")
        flat = np.fromfile(fh, dtype=_TAGS[tag], count=n * d)
    if flat.size != n * d:
        raise ValueError(f"{path}: truncated payload, expected {n * d} values, "
                         f"got {flat.size}")
    return flat.astype(_TAGS[tag].newbyteorder("="), copy=False).reshape(n, d)


def write_bhtm(arr: np.ndarray, path) -> None:
    arr = np.ascontiguousarray(arr)
    if arr.dtype == np.float64:
        tag = 0
    elif arr.dtype == np.float32:
        tag = 1
    else:
        raise ValueError(f"unsupported dtype {arr.dtype}")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, tag, arr.shape[0], arr.shape[1]))
        arr.astype(_TAGS[tag], copy=False).tofile(fh)


def read_csv(path, has_header: bool = False) -> np.ndarray:
    out, width = [], None
    with open(path) as fh:
        for lineno, line in enumerate(fh, start=1):
            if has_header and lineno == 1:
                continue
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if width is None:
                width = len(parts)
            elif len(parts) != width:
                raise ValueError(f"{path}: row {lineno} has {len(parts)} "
                                 f"columns, expected {width}")
            try:
                out.append([float(v) for v in parts])
            except ValueError:
                raise ValueError(f"{path}: row {lineno} contains a "
                                 f"non-numeric field") from None
    if not out:
        raise ValueError(f"{path}: no data rows")
    return np.asarray(out, dtype=np.float64)


def write_csv(arr: np.ndarray, path) -> None:
    with open(path, "w") as fh:
        for row in np.asarray(arr):
            fh.write(",".join(repr(float(v)) for v in row) + "\n")


def load_matrix(path, format: str | None = None, precision: str = "f32",
                has_header: bool = False) -> InputMatrix:
    fmt = format or sniff_format(path)
    if fmt == "bin":
        raw = read_bhtm(path)
    elif fmt == "csv":
        raw = read_csv(path, has_header)
    else:
        raise ValueError(f"unknown format {fmt!r}; expected 'csv' or 'bin'")
    return InputMatrix(np.ascontiguousarray(raw, dtype=precision_dtype(precision)))


def save_matrix(m, path, format: str | None = None) -> None:
    arr = m.data if isinstance(m, InputMatrix) else np.asarray(m)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    if arr.ndim == 2 and arr.shape[0] >= 2:
        InputMatrix(arr)
    fmt = format or ("csv" if os.fspath(path).endswith(".csv") else "bin")
    if fmt == "bin":
        write_bhtm(arr, path)
    elif fmt == "csv":
        write_csv(arr, path)
    else:
        raise ValueError(f"unknown format {fmt!r}; expected 'csv' or 'bin'")


def load_labels(path) -> np.ndarray:
    """One integer class id per non-empty line -- the first comma-separated
    field, "3" and "3.0" alike (io.py:120-128; used by the plot only)."""
    ids = []
    with open(path) as fh:
        for lineno, line in enumerate(fh, start=1):
            field = line.strip().split(",")[0]
            if not line.strip():
                continue
            try:
                ids.append(int(float(field)))
            except ValueError:
                raise ValueError(f"labels file {path}: line {lineno}: "
                                 f"{field!r} is not a class id") from None
    return np.asarray(ids, dtype=np.int64)
