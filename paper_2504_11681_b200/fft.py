"""Truncating / zero-padded / pruned FFT API — mirror of ``fnofuse.fft``
(fft.py:1-315): ``plan``, ``FftPlan`` (prune masks, op and twiddle budgets),
``full_op_count``, ``execute`` and ``batched_execute``.

Plans are analysed natively (``tfno_plan_counts``, csrc/plan.cpp); the
transforms run on the GPU (``tfno_fft_execute``, the mixed-radix
Stockham engine in csrc/fft_engine.cuh) — never on the CPU.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _device
from ._lib import check, lib
from .core import COMPLEX_DTYPE, FnofuseError, is_power_of_two

FORWARD = "forward"
INVERSE = "inverse"


class InvalidLength(FnofuseError):
    pass


class InvalidKeep(FnofuseError):
    pass


class InvalidSrcLen(FnofuseError):
    pass


class LengthMismatch(FnofuseError):
    pass


class StrideOverlap(FnofuseError):
    pass


@dataclass(frozen=True)
class OpCount:
    """fft.py:62-75."""

    butterflies: int
    twiddle_muls: int
    skipped: int

    def scaled(self, pencils: int) -> "OpCount":
        return OpCount(self.butterflies * pencils, self.twiddle_muls * pencils, self.skipped * pencils)


@dataclass(frozen=True)
class StageSpec:
    stride: int
    twiddle_offset: int


class FftPlan:
    """Immutable plan (fft.py:87-191): same attributes as the reference."""

    def __init__(self, n: int, direction: str, keep: int, src_len: int):
        if not is_power_of_two(n):
            raise InvalidLength(f"transform length {n} is not a power of two")
        if direction not in (FORWARD, INVERSE):
            raise FnofuseError(f"direction must be {FORWARD!r} or {INVERSE!r}")
        if not 1 <= keep <= n:
            raise InvalidKeep(f"keep={keep} outside [1, {n}]")
        if not 1 <= src_len <= n:
            raise InvalidSrcLen(f"src_len={src_len} outside [1, {n}]")
        self.n, self.direction, self.keep, self.src_len = n, direction, keep, src_len
        ns = n.bit_length() - 1
        self.full_ops = n * ns
        sign = -1.0 if direction == FORWARD else 1.0
        self.stages = tuple(StageSpec(stride=1 << j, twiddle_offset=(1 << j) - 1) for j in range(ns))
        tables = [np.exp(sign * 1j * math.pi * np.arange(1 << j, dtype=np.float64) / (1 << j))
                  .astype(COMPLEX_DTYPE) for j in range(ns)]
        self.twiddles = np.concatenate(tables) if tables else np.zeros(0, COMPLEX_DTYPE)
        self.twiddles.setflags(write=False)
        masks = np.zeros(max(ns, 1) * n, dtype=np.uint8)
        ob, tb, fo = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        rc = lib().tfno_plan_counts(n, -1 if direction == FORWARD else 1, keep, src_len,
                                    ctypes.byref(ob), ctypes.byref(tb), ctypes.byref(fo),
                                    masks.ctypes.data_as(ctypes.c_void_p))
        if rc != 0:
            raise FnofuseError(f"plan analysis failed (code {rc})")
        mlist = []
        for j in range(ns):
            m = masks[j * n:(j + 1) * n].astype(bool)
            m.setflags(write=False)
            mlist.append(m)
        self.prune_mask = tuple(mlist)
        self.op_budget = int(ob.value)
        self.twiddle_budget = int(tb.value)

    def op_count(self, pencils: int = 1) -> OpCount:
        return OpCount(self.op_budget, self.twiddle_budget, self.full_ops - self.op_budget).scaled(pencils)

    def __repr__(self):
        return (f"FftPlan(n={self.n}, direction={self.direction!r}, keep={self.keep}, "
                f"src_len={self.src_len}, op_budget={self.op_budget})")


_PLAN_CACHE = {}


def plan(n: int, direction: str = FORWARD, keep: Optional[int] = None,
         src_len: Optional[int] = None) -> FftPlan:
    """fft.py:194-202 (plans are cached: they are immutable)."""
    key = (n, direction, n if keep is None else keep, n if src_len is None else src_len)
    p = _PLAN_CACHE.get(key)
    if p is None:
        p = FftPlan(*key)
        if isinstance(n, int):
            _PLAN_CACHE[key] = p
    return p


def full_op_count(n: int) -> int:
    """fft.py:205-209."""
    if not is_power_of_two(n):
        raise InvalidLength(f"transform length {n} is not a power of two")
    return n * (n.bit_length() - 1)


def _gpu_rows(p: FftPlan, rows_dev, out_dev, in_pencil_stride, in_es, out_pencil_stride, out_es, P):
    """Run P pencils on device tensors (element offsets in complex units)."""
    rc = lib().tfno_fft_execute(p.n, -1 if p.direction == FORWARD else 1, p.keep, p.src_len, P,
                                rows_dev.data_ptr(), 1, in_pencil_stride, 0, in_es,
                                out_dev.data_ptr(), 1, out_pencil_stride, 0, out_es,
                                _device.stream_ptr())
    check(rc, "tfno_fft_execute")


def execute_device(p: FftPlan, pencils, out=None):
    """Device API: pencils is a CUDA complex64 tensor (P, src_len) with any
    strides; returns a (P, keep) tensor (or writes into ``out``)."""
    t = _device.torch()
    if pencils.dim() != 2 or pencils.shape[1] != p.src_len:
        raise LengthMismatch(f"pencil length {pencils.shape[-1]} != plan src_len {p.src_len}")
    P = pencils.shape[0]
    if out is None:
        out = t.empty((P, p.keep), dtype=t.complex64, device=pencils.device)
    if P:
        _gpu_rows(p, pencils, out, pencils.stride(0), pencils.stride(1), out.stride(0), out.stride(1), P)
    return out


def _run_host(p: FftPlan, block: np.ndarray) -> np.ndarray:
    dev = _device.require_cuda()
    t = _device.torch()
    src = _device.to_device_c64(np.ascontiguousarray(block, dtype=COMPLEX_DTYPE), dev)
    out = execute_device(p, src)
    res = out.cpu().numpy()
    t.cuda.current_stream().synchronize()
    return res


def execute(p: FftPlan, x: np.ndarray, out: Optional[np.ndarray] = None):
    """fft.py:258-276 — one pencil through the plan (on the GPU)."""
    x = np.asarray(x)
    if x.ndim != 1 or x.shape[0] != p.src_len:
        raise LengthMismatch(f"input length {x.shape} != plan src_len {p.src_len}")
    res = _run_host(p, x[None, :])[0]
    if out is None:
        out = res
    else:
        if out.shape[0] < p.keep:
            raise LengthMismatch(f"out capacity {out.shape[0]} < keep {p.keep}")
        out[:p.keep] = res
    return out, p.op_count()


def _view_aliases(view: np.ndarray) -> bool:
    nr, nc = view.shape
    sr, sc = view.strides
    idx = np.arange(nr, dtype=np.int64)[:, None] * sr + np.arange(nc, dtype=np.int64)[None, :] * sc
    return np.unique(idx).size != nr * nc


def batched_execute(p: FftPlan, batch: np.ndarray, out: Optional[np.ndarray] = None):
    """fft.py:288-315 — strided view of pencils sharing one plan."""
    batch = np.asarray(batch)
    if batch.ndim != 2:
        raise LengthMismatch("batch must be a 2-D view of pencils")
    if batch.shape[1] != p.src_len:
        raise LengthMismatch(f"pencil length {batch.shape[1]} != plan src_len {p.src_len}")
    if _view_aliases(batch):
        raise StrideOverlap("two pencils alias the same element")
    bs = batch.shape[0]
    res = _run_host(p, batch) if bs else np.empty((0, p.keep), COMPLEX_DTYPE)
    if out is None:
        out = res
    else:
        if out.shape != (bs, p.keep):
            raise LengthMismatch(f"out shape {out.shape} != {(bs, p.keep)}")
        if _view_aliases(out):
            raise StrideOverlap("two output pencils alias the same element")
        out[:] = res
    return out, p.op_count(bs)
