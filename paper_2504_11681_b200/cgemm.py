"""Complex GEMM API — mirror of ``fnofuse.cgemm`` (cgemm.py:1-124):
``ComplexMatrix`` (column-major complex64), ``GemmProblem``, ``gemm_tiled``
and ``gemm_kloop``, computed on the GPU by the FP32 SIMT CGEMM kernel
(``tfno_cgemm``, csrc/kernels.cu), k ascending with fp32 accumulation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device
from ._lib import check, lib
from .core import COMPLEX_DTYPE, DEFAULT_TILES, ShapeMismatch, TileConfig, tile_violations


@dataclass(frozen=True)
class ComplexMatrix:
    """Column-major complex64 matrix (cgemm.py:21-58)."""

    values: np.ndarray

    def __post_init__(self):
        v = self.values
        if hasattr(v, "detach"):
            v = v.detach().cpu().numpy()
        arr = np.asfortranarray(v, dtype=COMPLEX_DTYPE)
        if arr.ndim != 2:
            raise ShapeMismatch(f"expected a 2-D matrix, got {arr.ndim}-D")
        object.__setattr__(self, "values", arr)

    @property
    def rows(self) -> int:
        return self.values.shape[0]

    @property
    def cols(self) -> int:
        return self.values.shape[1]

    @property
    def data(self) -> np.ndarray:
        return self.values.ravel(order="F")

    @classmethod
    def zeros(cls, rows: int, cols: int) -> "ComplexMatrix":
        return cls(np.zeros((rows, cols), dtype=COMPLEX_DTYPE, order="F"))

    @classmethod
    def identity(cls, n: int) -> "ComplexMatrix":
        return cls(np.eye(n, dtype=COMPLEX_DTYPE, order="F"))

    @classmethod
    def random(cls, rows: int, cols: int, rng: np.random.Generator) -> "ComplexMatrix":
        re = rng.standard_normal((rows, cols), dtype=np.float32)
        im = rng.standard_normal((rows, cols), dtype=np.float32)
        return cls(re + 1j * im)


@dataclass(frozen=True)
class GemmProblem:
    m: int
    n: int
    k: int
    tiles: TileConfig = DEFAULT_TILES


def _check_shapes(p: GemmProblem, a: ComplexMatrix, b: ComplexMatrix) -> None:
    """cgemm.py:71-80."""
    if (a.rows, a.cols) != (p.m, p.k):
        raise ShapeMismatch(f"A is {a.rows}x{a.cols}, problem wants {p.m}x{p.k}")
    if (b.rows, b.cols) != (p.k, p.n):
        raise ShapeMismatch(f"B is {b.rows}x{b.cols}, problem wants {p.k}x{p.n}")
    if min(p.m, p.n, p.k) < 1:
        raise ShapeMismatch(f"degenerate problem {p.m}x{p.n}x{p.k}")
    bad = tile_violations(p.tiles)
    if bad:
        raise ShapeMismatch("; ".join(str(v) for v in bad))


def cgemm_device(a, b, out=None, alpha: float = 1.0, precision: str = "fp32"):
    """Device API: C = alpha * a @ b for CUDA complex64 tensors of any
    strides (2-D, or 3-D batched along dim 0).  precision "tf32" / "tf32x3"
    runs the tcgen05 tensor-core contraction (mode layout required: a and the
    output m-contiguous, b row-major with N <= 128)."""
    t = _device.torch()
    batched = a.dim() == 3
    A = a if batched else a.unsqueeze(0)
    Bm = b if b.dim() == 3 else b.unsqueeze(0)
    bsz, M, K = A.shape
    K2, N = Bm.shape[1], Bm.shape[2]
    if K != K2:
        raise ShapeMismatch(f"inner dims differ: {K} vs {K2}")
    if out is None:
        out = t.empty((bsz, N, M), dtype=t.complex64, device=a.device).transpose(1, 2)
    C = out if out.dim() == 3 else out.unsqueeze(0)
    w_bs = Bm.stride(0) if Bm.shape[0] > 1 else 0
    from ._lib import PREC_CODES
    rc = lib().tfno_cgemm_prec(M, N, K, bsz, A.data_ptr(), A.stride(1), A.stride(2), A.stride(0),
                               Bm.data_ptr(), Bm.stride(1), Bm.stride(2), w_bs,
                               C.data_ptr(), C.stride(1), C.stride(2), C.stride(0), float(alpha),
                               PREC_CODES[precision], _device.stream_ptr())
    check(rc, "tfno_cgemm_prec")
    return out if batched else C[0]


def _host_gemm(av: np.ndarray, bv: np.ndarray) -> np.ndarray:
    dev = _device.require_cuda()
    t = _device.torch()
    A = t.from_numpy(np.asfortranarray(av, dtype=COMPLEX_DTYPE).T.copy()).to(dev).T  # column-major view
    Bm = t.from_numpy(np.ascontiguousarray(bv, dtype=COMPLEX_DTYPE)).to(dev)
    C = cgemm_device(A, Bm)
    return np.asfortranarray(C.cpu().numpy())


def gemm_kloop(a: np.ndarray, b: np.ndarray, k_tb: int) -> np.ndarray:
    """cgemm.py:83-95 — fp32 product, k ascending (GPU)."""
    return np.ascontiguousarray(_host_gemm(np.asarray(a), np.asarray(b)))


def gemm_tiled(p: GemmProblem, a: ComplexMatrix, b: ComplexMatrix) -> ComplexMatrix:
    """cgemm.py:98-114 — blocked fp32 CGEMM with bounds-checked edge tiles (GPU)."""
    _check_shapes(p, a, b)
    return ComplexMatrix(_host_gemm(a.values, b.values))
