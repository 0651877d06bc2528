"""ctypes binding of libturbofno.so (include/turbofno.h).

The library is built in-tree (``python -m paper_2504_11681_b200.build``).
There is no fallback: if the library or a CUDA device is missing, compute
entry points raise ``NativeUnavailable`` loudly.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libturbofno.so")

MODE_CODES = {"staged": 0, "fft_optimized": 1, "fused_fft_gemm": 2,
              "fused_gemm_ifft": 3, "fully_fused": 4}
PREC_CODES = {"fp32": 0, "tf32": 1, "bf16": 2, "tf32x3": 3}
VIOLATION_BITS = {1: "InvalidRankShape", 2: "NonPowerOfTwoLength", 4: "TruncationExceedsLength",
                  8: "TileDivisibilityViolation", 16: "BatchSizeMismatch"}


class NativeUnavailable(RuntimeError):
    """libturbofno.so (or a CUDA device) is missing: no CPU fallback exists."""


class TfnoCfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("batch", "hidden_dim", "output_dim", "dim_x", "dim_y", "keep_x", "keep_y", "rank")]


class TfnoTiles(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("m_tb", "n_tb", "k_tb", "m_w", "n_w", "m_t", "n_t")]


_I64 = ctypes.c_int64
_VP = ctypes.c_void_p
_SIGS = {
    "tfno_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "tfno_version": (ctypes.c_char_p, []),
    "tfno_config_violations": (ctypes.c_uint32, [ctypes.POINTER(TfnoCfg), ctypes.POINTER(TfnoTiles), ctypes.c_int]),
    "tfno_plan_counts": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64), _VP]),
    "tfno_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(TfnoCfg), ctypes.c_int, ctypes.c_int]),
    "tfno_layer_forward": (ctypes.c_int, [ctypes.POINTER(TfnoCfg), ctypes.c_int, ctypes.c_int, _VP, _VP, _VP,
                                          _VP, ctypes.c_size_t, _VP]),
    "tfno_packed_weight_bytes": (ctypes.c_size_t, [ctypes.POINTER(TfnoCfg), ctypes.c_int]),
    "tfno_prepare_weights": (ctypes.c_int, [ctypes.POINTER(TfnoCfg), ctypes.c_int, _VP, _VP, _VP]),
    "tfno_layer_forward_packed": (ctypes.c_int, [ctypes.POINTER(TfnoCfg), ctypes.c_int, ctypes.c_int, _VP, _VP, _VP,
                                                 _VP, _VP, ctypes.c_size_t, _VP]),
    "tfno_fft_execute": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _I64, _VP,
                                        _I64, _I64, _I64, _I64, _VP, _I64, _I64, _I64, _I64, _VP]),
    "tfno_cgemm": (ctypes.c_int, [_I64, _I64, _I64, _I64, _VP, _I64, _I64, _I64, _VP, _I64, _I64, _I64,
                                  _VP, _I64, _I64, _I64, ctypes.c_float, _VP]),
    "tfno_spectrum_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(TfnoCfg), ctypes.c_int]),
    "tfno_spectrum_forward": (ctypes.c_int, [ctypes.POINTER(TfnoCfg), _VP, _VP, _VP, ctypes.c_size_t, _VP]),
    "tfno_spectrum_inverse": (ctypes.c_int, [ctypes.POINTER(TfnoCfg), _VP, _VP, ctypes.c_float, _VP,
                                             ctypes.c_size_t, _VP]),
    "tfno_cgemm_prec": (ctypes.c_int, [_I64, _I64, _I64, _I64, _VP, _I64, _I64, _I64, _VP, _I64, _I64, _I64,
                                       _VP, _I64, _I64, _I64, ctypes.c_float, ctypes.c_int, _VP]),
    "tfno_batch_sum": (ctypes.c_int, [_VP, _I64, _I64, _VP, _VP]),
    "tfno_permode_mix": (ctypes.c_int, [_I64, _I64, _I64, _I64, _VP, _VP, _VP, ctypes.c_float, _VP]),
    "tfno_modulate": (ctypes.c_int, [_I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     _VP, _VP, ctypes.c_float, _VP]),
    "tfno_real_to_complex": (ctypes.c_int, [_VP, _VP, _I64, _VP]),
    "tfno_half_spectrum_weight": (ctypes.c_int, [_VP, _I64, ctypes.c_int, ctypes.c_int, _VP]),
    "tfno_real_epilogue": (ctypes.c_int, [_VP, _VP, _VP, _I64, ctypes.c_int, _I64, ctypes.c_int, _VP, _VP]),
    "tfno_launch_count": (ctypes.c_longlong, []),
    "tfno_set_stage_events": (None, [_VP, ctypes.c_int]),
    "tfno_layer_schedule": (ctypes.c_int, [ctypes.POINTER(TfnoCfg), ctypes.c_int, ctypes.c_int,
                                           ctypes.c_char_p, ctypes.c_size_t]),
}
EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load (once) and return the native library; raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; build it with `python -m paper_2504_11681_b200.build` "
                "(there is no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def cfg_struct(cfg) -> TfnoCfg:
    return TfnoCfg(cfg.batch, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y,
                   cfg.keep_x, cfg.keep_y, cfg.rank)


def tiles_struct(t) -> TfnoTiles:
    return TfnoTiles(t.m_tb, t.n_tb, t.k_tb, t.m_w, t.n_w, t.m_t, t.n_t)


def check(code: int, what: str) -> None:
    if code != 0:
        msg = lib().tfno_strerror(code).decode()
        raise NativeUnavailable(f"{what} failed: {msg} (code {code})") if code == 3 else \
            RuntimeError(f"{what} failed: {msg} (code {code})")
