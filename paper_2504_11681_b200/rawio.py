"""Raw complex tensor container — the reference's wire format
(reporting.py:236-282): little-endian header of four uint32 dims followed by
interleaved (re, im) float32 pairs in row-major order; weights are stored as
dims [rows, cols, 1, 1] with a row-major payload.  Byte-compatible with the
reference, so files move between the two implementations unchanged."""

from __future__ import annotations

import numpy as np

from .cgemm import ComplexMatrix
from .core import COMPLEX_DTYPE, FnofuseError

_HEADER_DTYPE = np.dtype("<u4")
_DATA_DTYPE = np.dtype("<c8")


def write_raw_tensor(path: str, arr) -> None:
    arr = np.ascontiguousarray(arr, dtype=COMPLEX_DTYPE)
    if arr.ndim != 4:
        raise FnofuseError(f"raw tensors are 4-D, got {arr.ndim}-D")
    with open(path, "wb") as f:
        np.asarray(arr.shape, dtype=_HEADER_DTYPE).tofile(f)
        arr.astype(_DATA_DTYPE, copy=False).tofile(f)


def read_raw_tensor(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        dims = np.fromfile(f, dtype=_HEADER_DTYPE, count=4)
        if dims.size != 4:
            raise FnofuseError(f"{path}: truncated header")
        count = int(np.prod(dims.astype(np.int64)))
        data = np.fromfile(f, dtype=_DATA_DTYPE, count=count)
        if data.size != count:
            raise FnofuseError(f"{path}: expected {count} complex elements, found {data.size}")
        if f.read(1):
            raise FnofuseError(f"{path}: trailing bytes after payload")
    return data.astype(COMPLEX_DTYPE).reshape(tuple(int(d) for d in dims))


def write_raw_matrix(path: str, mat: ComplexMatrix) -> None:
    write_raw_tensor(path, np.ascontiguousarray(mat.values).reshape(mat.rows, mat.cols, 1, 1))


def read_raw_matrix(path: str) -> ComplexMatrix:
    arr = read_raw_tensor(path)
    if arr.shape[2:] != (1, 1):
        raise FnofuseError(f"{path}: weight container must have dims [rows, cols, 1, 1], got {arr.shape}")
    return ComplexMatrix(arr.reshape(arr.shape[0], arr.shape[1]))
