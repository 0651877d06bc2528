"""Real-field Fourier layer and FNO block — R2C/C2R input/output, pointwise
bypass, bias and activation (extensions beyond the
reference, whose ``run_layer`` is complex-to-complex only, Appendix A).

    real_layer:  y = irfft2(einsum(bhpq,hn->bnpq, rfft2(x)[..., :kx, :ky], W), s=(dx, dy))
                 (rank 1: irfft(rfft(x)[..., :ky] W, n=dy));  ky <= dy/2 + 1
    fno_block:   y = act(real_layer(x) + einsum(bhxy,hn->bnxy, x, W_bypass) + bias[n])

Composed on the spectrum C-ABI (include/turbofno.h): x + 0i
(``tfno_real_to_complex``) -> first-keep forward DFT (``tfno_spectrum_forward``,
== the rfft bins kept) -> per-bin weights c_k = 2 for 0 < k < dy/2
(``tfno_half_spectrum_weight``) -> channel mix (``tfno_cgemm``) -> padded
inverse (``tfno_spectrum_inverse``) -> Re + bypass + bias + activation
(``tfno_real_epilogue``), since irfft of bins 0..ky-1 equals
Re(sum_k c_k Z_k e^{2 pi i k t/dy})/dy.  The bypass channel mix is a plain real
GEMM (cuBLAS through torch.matmul).  Pinned by its own float64 oracle
(torch.fft.rfft2/irfft2 in tests/test_gpu_realfield.py; the identity itself in
tests/test_realfield_math.py).
"""

from __future__ import annotations

import contextlib

from . import _device
from ._lib import check, lib
from .core import FnoLayerConfig, FnofuseError, ShapeMismatch
from .multigpu import spectrum_forward, spectrum_inverse

ACTIVATIONS = {None: 0, "none": 0, "relu": 1, "gelu": 2}


def _check_real_cfg(cfg: FnoLayerConfig):
    if cfg.keep_y > cfg.dim_y // 2 + 1:
        raise FnofuseError(f"real layer needs keep_y <= dim_y/2 + 1 (got keep_y={cfg.keep_y}, dim_y={cfg.dim_y})")


def real_spectral(cfg: FnoLayerConfig, x, w, stream=None):
    """Complex planes z[B,N,dx,dy] with Re(z) == real_layer(cfg, x, w).  x: real
    float32 [B,H,dx,dy] CUDA; w: complex64 [H,N] CUDA."""
    t = _device.torch()
    _check_real_cfg(cfg)
    B, H, N = cfg.batch, cfg.hidden_dim, cfg.output_dim
    if tuple(x.shape) != (B, H, cfg.dim_x, cfg.dim_y) or x.dtype != t.float32:
        raise ShapeMismatch(f"x must be float32 {(B, H, cfg.dim_x, cfg.dim_y)}, got {x.dtype} {tuple(x.shape)}")
    if tuple(w.shape) != (H, N):
        raise ShapeMismatch(f"w shape {tuple(w.shape)} != {(H, N)}")
    sp = _device.stream_ptr(stream)
    # temporaries allocated on the stream the kernels run on (no cross-stream reuse)
    with (t.cuda.stream(stream) if stream is not None else contextlib.nullcontext()):
        x = x.contiguous()
        w = w.to(t.complex64).contiguous()
        xc = t.empty(x.shape, dtype=t.complex64, device=x.device)
        check(lib().tfno_real_to_complex(x.data_ptr(), xc.data_ptr(), x.numel(), sp), "tfno_real_to_complex")
        A = spectrum_forward(cfg, xc, stream)                                   # [B,H,kx,ky]
        del xc
        MQ = cfg.keep_x * cfg.keep_y
        check(lib().tfno_half_spectrum_weight(A.data_ptr(), B * H * cfg.keep_x, cfg.keep_y, cfg.dim_y, sp),
              "tfno_half_spectrum_weight")
        C = t.empty((B, N, cfg.keep_x, cfg.keep_y), dtype=t.complex64, device=x.device)
        check(lib().tfno_cgemm(MQ, N, H, B, A.data_ptr(), 1, MQ, H * MQ, w.data_ptr(), N, 1, 0,
                               C.data_ptr(), 1, MQ, N * MQ, 1.0, sp), "tfno_cgemm")
        return spectrum_inverse(cfg, C, (B, N), scale=1.0, stream=stream)


def fno_block(cfg: FnoLayerConfig, x, w, bypass_w=None, bias=None, activation=None, out=None, stream=None):
    """act(real_layer(x) + einsum(bhxy,hn->bnxy, x, bypass_w) + bias) as float32 [B,N,dx,dy].

    bypass_w: real [H,N] or None; bias: real [N] or None; activation: None/"relu"/"gelu"."""
    t = _device.torch()
    if activation not in ACTIVATIONS:
        raise FnofuseError(f"unknown activation {activation!r}; expected one of none/relu/gelu")
    B, H, N = cfg.batch, cfg.hidden_dim, cfg.output_dim
    P = cfg.dim_x * cfg.dim_y
    z = real_spectral(cfg, x, w, stream)
    byp = None
    if bypass_w is not None:
        if tuple(bypass_w.shape) != (H, N):
            raise ShapeMismatch(f"bypass_w shape {tuple(bypass_w.shape)} != {(H, N)}")
        # [B,N,P] = W_b^T [N,H] @ x [B,H,P]  (plain real GEMM, cuBLAS)
        with (t.cuda.stream(stream) if stream is not None else contextlib.nullcontext()):
            byp = t.matmul(bypass_w.to(t.float32).t().contiguous(), x.contiguous().reshape(B, H, P))
    if bias is not None:
        if tuple(bias.shape) != (N,):
            raise ShapeMismatch(f"bias shape {tuple(bias.shape)} != {(N,)}")
        bias = bias.to(t.float32).contiguous()
    if out is None:
        out = t.empty((B, N, cfg.dim_x, cfg.dim_y), dtype=t.float32, device=x.device)
    check(lib().tfno_real_epilogue(z.data_ptr(), byp.data_ptr() if byp is not None else None,
                                   bias.data_ptr() if bias is not None else None, B, N, P,
                                   ACTIVATIONS[activation], out.data_ptr(), _device.stream_ptr(stream)),
          "tfno_real_epilogue")
    return out


def real_layer(cfg: FnoLayerConfig, x, w, out=None, stream=None):
    """irfft2(einsum(bhpq,hn->bnpq, rfft2(x)[..., :kx, :ky], W), s=(dx, dy)) as float32."""
    return fno_block(cfg, x, w, out=out, stream=stream)
