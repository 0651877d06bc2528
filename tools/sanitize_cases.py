"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck):  tools/sanitize.sh"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_11681_b200 as T  # noqa: E402
from paper_2504_11681_b200 import multigpu as MG  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)


def rnd(*shape):
    return torch.from_numpy((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)).to(dev)


cases = [((1, 2, 2, 128, 128, 16, 16, 2), ["fully_fused"]),            # plane2d G128
         ((1, 1, 1, 512, 512, 64, 64, 2), ["fully_fused"]),            # plane2d G512 (TMA ring, producer warp)
         ((2, 3, 2, 32, 64, 8, 16, 2), list(T.MODES)),                  # paper schedule + generic kernels
         ((2, 8, 8, 1, 1024, 1, 128, 1), ["fully_fused", "fft_optimized"]),  # warp fused / warp rows
         ((3, 8, 8, 1, 256, 1, 32, 1), ["fully_fused", "fft_optimized"]),
         ((1, 4, 4, 1, 4096, 1, 512, 1), ["fully_fused"]),               # team rows
         ((2, 8, 8, 1, 128, 1, 32, 1), ["fully_fused", "fused_fft_gemm", "fused_gemm_ifft"]),  # CT rows fused
         ((3, 64, 64, 1, 256, 1, 32, 1), ["fully_fused"]),               # fused1d, output-channel split 2
         ((200, 32, 64, 1, 256, 1, 32, 1), ["fully_fused"]),             # fused1d, several items per CTA
         ((150, 16, 64, 1, 1024, 1, 128, 1), ["fully_fused"]),           # fused1d L = 32
         ((3, 20, 19, 256, 256, 32, 32, 2), ["fully_fused"]),            # generic plane / fused mix (TFNO_PLANE_FUSEDMIX=1)
         ((300, 2, 9, 64, 64, 16, 16, 2), ["fully_fused"])]              # more mix tasks than CTAs (rings wrap)
for shape, modes in cases:
    cfg = T.FnoLayerConfig(*shape)
    x, w = rnd(cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), rnd(cfg.hidden_dim, cfg.output_dim)
    for mode in modes:
        T.run_layer_device(cfg, x, w, mode=mode)
        torch.cuda.synchronize()
        print("ok", shape, mode, flush=True)
for shape in ((2, 8, 8, 512, 512, 64, 64, 2), (3, 12, 20, 1, 1024, 1, 128, 1)):  # tcgen05 layer (W' image)
    cfg = T.FnoLayerConfig(*shape)
    x, w = rnd(cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), rnd(cfg.hidden_dim, cfg.output_dim)
    for prec in ("tf32x3", "tf32"):
        T.run_layer_device(cfg, x, w, mode="fully_fused", precision=prec)
        torch.cuda.synchronize()
        print("ok tc layer", shape, prec, flush=True)
from paper_2504_11681_b200.autograd import layer_backward  # noqa: E402
from paper_2504_11681_b200.symmetric import run_layer_symmetric  # noqa: E402
cfg = T.FnoLayerConfig(2, 4, 6, 64, 64, 8, 8, 2)
x, w, gy = rnd(2, 4, 64, 64), rnd(4, 6), rnd(2, 6, 64, 64)
layer_backward(cfg, x, w, gy)
run_layer_symmetric(cfg, x, w)
torch.cuda.synchronize()
print("ok backward / symmetric", flush=True)
for shape in ((2, 4, 6, 64, 64, 8, 8, 2), (3, 2, 3, 1, 2, 1, 2, 1)):  # real layer + block epilogue (vector/scalar)
    cfg = T.FnoLayerConfig(*shape)
    xr = torch.randn(cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y, device="cuda")
    T.fno_block(cfg, xr, rnd(cfg.hidden_dim, cfg.output_dim), bypass_w=torch.randn(cfg.hidden_dim, cfg.output_dim,
                device="cuda"), bias=torch.randn(cfg.output_dim, device="cuda"), activation="gelu")
    torch.cuda.synchronize()
    print("ok real block", shape, flush=True)
for prec in ("tf32", "tf32x3", "bf16"):
    A = rnd(2, 64, 256).transpose(1, 2)
    T.cgemm_device(A, rnd(64, 96), precision=prec)
    torch.cuda.synchronize()
    print("ok cgemm", prec, flush=True)
cfg = T.FnoLayerConfig(1, 4, 4, 256, 256, 32, 32, 2)
MG.spectrum_inverse(cfg, MG.spectrum_forward(cfg, rnd(1, 4, 256, 256)), (1, 4))
torch.cuda.synchronize()
print("ok spectrum")
for shape in ((16, 64, 64, 1, 128, 1, 32, 1), (64, 64, 64, 1, 256, 1, 32, 1), (3, 20, 70, 1, 1024, 1, 100, 1)):
    cfg = T.FnoLayerConfig(*shape)  # tiny1d (the last one only with TFNO_TINY1D=1; default fused1d otherwise)
    x, w = rnd(cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), rnd(cfg.hidden_dim, cfg.output_dim)
    T.run_layer_device(cfg, x, w)
    torch.cuda.synchronize()
    print("ok tiny1d", shape, flush=True)
