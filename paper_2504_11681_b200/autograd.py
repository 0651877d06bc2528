"""Backward pass of the Fourier layer (SURVEY.md §8f row 4 "the backward
pass"; the reference ``fnofuse`` is forward-only, so this extension is pinned
by its own float64 oracle: ``tests/test_gpu_autograd.py`` differentiates a
float64 torch.fft composition of SURVEY.md Appendix A with autograd).

The layer is linear in x and in W (Appendix A):

    y[b,n] = (1/(dx*dy)) * E^H ( sum_h W[h,n] * E x[b,h] )

with E the truncating (first-keep-bins, unnormalised) 2D DFT and E^H the
zero-padded inverse.  With PyTorch's complex-gradient convention (the
returned gradient is dL/d(conj z)), the adjoints are

    grad_x[b,h] = (1/(dx*dy)) * E^H ( sum_n conj(W[h,n]) * E gy[b,n] )
                = run_layer(cfg with H <-> N, gy, W^H)            (same kernels)
    grad_W[h,n] = (1/(dx*dy)) * sum_b sum_modes conj(A[b,h,m]) * G[b,n,m],
                  A = E x (spectrum of the input), G = E gy,

so backward is two spectrum transforms, one channel-mix reduction over
(batch, modes) and one forward layer with the conjugate-transposed weights,
all on the sm_100a kernels of the forward path.
"""

from __future__ import annotations

from . import _device
from ._lib import check, lib
from .core import FnoLayerConfig
from .multigpu import spectrum_forward
from .pipeline import run_layer_device


def _transposed(cfg: FnoLayerConfig) -> FnoLayerConfig:
    return FnoLayerConfig(cfg.batch, cfg.output_dim, cfg.hidden_dim, cfg.dim_x, cfg.dim_y,
                          cfg.keep_x, cfg.keep_y, cfg.rank)


def layer_backward(cfg: FnoLayerConfig, x, w, grad_y, need_x: bool = True, need_w: bool = True,
                   precision: str = "fp32"):
    """(grad_x, grad_w) of the layer at (x, w) for the output gradient grad_y.
    x [B,H,dx,dy], w [H,N], grad_y [B,N,dx,dy]: complex64 CUDA tensors."""
    t = _device.torch()
    grad_x = grad_w = None
    gy = grad_y.contiguous()
    if need_x:
        wh = w.conj().transpose(0, 1).contiguous().resolve_conj()  # W^H as [N][H]
        grad_x = run_layer_device(_transposed(cfg), gy, wh, precision=precision)
    if need_w:
        B, H, N = cfg.batch, cfg.hidden_dim, cfg.output_dim
        MQ = cfg.keep_x * cfg.keep_y
        A = spectrum_forward(cfg, x.contiguous())                  # [B,H,kx,ky]
        G = spectrum_forward(_transposed(cfg), gy)                 # [B,N,kx,ky]
        Ac = A.conj_physical()
        part = t.empty((B, H, N), dtype=t.complex64, device=x.device)
        # part[b][h][n] = sum_m conj(A)[b][h][m] * G[b][n][m] / (dx*dy): M = H, K = modes, N = N
        rc = lib().tfno_cgemm(H, N, MQ, B, Ac.data_ptr(), MQ, 1, H * MQ, G.data_ptr(), 1, MQ, N * MQ,
                              part.data_ptr(), N, 1, H * N, 1.0 / (cfg.dim_x * cfg.dim_y),
                              _device.stream_ptr(None))
        check(rc, "tfno_cgemm")
        grad_w = t.empty((H, N), dtype=t.complex64, device=x.device)
        check(lib().tfno_batch_sum(part.data_ptr(), B, H * N, grad_w.data_ptr(), _device.stream_ptr(None)),
              "tfno_batch_sum")
    return grad_x, grad_w


def _autograd_function():
    torch = _device.torch()

    class SpectralLayerFunction(torch.autograd.Function):
        """y = Fourier layer(x; W) with the sm_100a forward and backward kernels."""

        @staticmethod
        def forward(ctx, x, w, cfg, mode, precision):
            ctx.cfg, ctx.precision = cfg, precision
            ctx.save_for_backward(x, w)
            return run_layer_device(cfg, x.contiguous(), w.contiguous(), mode=mode, precision=precision)

        @staticmethod
        def backward(ctx, gy):
            x, w = ctx.saved_tensors
            gx, gw = layer_backward(ctx.cfg, x, w, gy, ctx.needs_input_grad[0], ctx.needs_input_grad[1],
                                    precision=ctx.precision)
            return gx, gw, None, None, None

    return SpectralLayerFunction


_FN = None


def spectral_layer(x, w, cfg: FnoLayerConfig = None, mode: str = "fully_fused", precision: str = "fp32"):
    """Differentiable Fourier layer: ``y = spectral_layer(x, w)`` with x
    [B,H,dx,dy] and w [H,N] complex64 CUDA tensors (rank 1: dx = 1)."""
    global _FN
    if _FN is None:
        _FN = _autograd_function()
    if cfg is None:
        raise ValueError("cfg (FnoLayerConfig with keep_x / keep_y) is required")
    return _FN.apply(x, w, cfg, mode, precision)
