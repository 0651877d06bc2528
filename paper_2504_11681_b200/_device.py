"""Device plumbing (PyTorch for memory and streams only)."""

from __future__ import annotations

import numpy as np

from ._lib import NativeUnavailable

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise NativeUnavailable("a CUDA device is required: the TurboFNO layer has no CPU fallback")
    return t.device(device if device is not None else f"cuda:{t.cuda.current_device()}")


def to_device_c64(a, device):
    """numpy / torch -> contiguous complex64 CUDA tensor (zero-copy if already one)."""
    t = torch()
    if isinstance(a, t.Tensor):
        if a.device == device and a.dtype == t.complex64 and a.is_contiguous():
            return a
        return a.to(device=device, dtype=t.complex64).contiguous()
    arr = np.ascontiguousarray(a, dtype=np.complex64)
    return t.from_numpy(arr).to(device, non_blocking=False)


def stream_ptr(stream=None) -> int:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return int(s.cuda_stream)


_WS = {}


def workspace(nbytes: int, device, stream=None):
    """Cached uint8 device workspace of at least nbytes (grown on demand),
    one per (device, stream): calls on different streams may run
    concurrently, so they never share scratch memory.  The buffer is
    allocated on (and its lifetime tracked against) that stream."""
    t = torch()
    sp = stream_ptr(stream)
    key = (str(device), sp)
    buf = _WS.get(key)
    if nbytes == 0:
        return None
    if buf is None or buf.numel() < nbytes:
        _WS.pop(key, None)
        if stream is not None:
            with t.cuda.stream(stream):
                buf = t.empty(nbytes, dtype=t.uint8, device=device)
        else:
            buf = t.empty(nbytes, dtype=t.uint8, device=device)
        _WS[key] = buf
    return buf


def release_workspace():
    _WS.clear()
