"""Backward pass of the Fourier layer (paper_2504_11681_b200.autograd) vs a
float64 oracle: SURVEY.md Appendix A written with torch.fft in complex128
and differentiated by autograd (the reference package is forward-only, so
this extension has its own oracle).  Gradients are linear maps of the output
gradient like the forward is of x: FP32 tolerance 1e-5 (max_rel_error)."""

import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _ref_layer(x, w, cfg):
    import torch
    if cfg.rank == 2:
        X = torch.fft.fft2(x)[..., :cfg.keep_x, :cfg.keep_y]
        C = torch.einsum("bhpq,hn->bnpq", X, w)
        return torch.fft.ifft2(C, s=(cfg.dim_x, cfg.dim_y))
    X = torch.fft.fft(x, dim=-1)[..., :cfg.keep_y]
    C = torch.einsum("bhpq,hn->bnpq", X, w)
    return torch.fft.ifft(C, n=cfg.dim_y, dim=-1)


CASES = [
    (3, 8, 6, 1, 256, 1, 32, 1),       # 1D: fused1d forward, warp-FFT spectra
    (2, 16, 16, 1, 128, 1, 32, 1),     # 1D N = 128
    (2, 4, 5, 64, 64, 8, 8, 2),        # 2D generic row/pencil kernels, H != N
    (1, 2, 3, 256, 256, 32, 32, 2),    # 2D plane kernels (C3 plane shape)
]


@pytest.mark.parametrize("case", CASES)
def test_backward_vs_float64_autograd(case):
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200.autograd import spectral_layer
    cfg = T.FnoLayerConfig(*case)
    g = torch.Generator().manual_seed(sum(case))
    shp_x = (cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y)
    shp_y = (cfg.batch, cfg.output_dim, cfg.dim_x, cfg.dim_y)
    x = torch.view_as_complex(torch.randn(shp_x + (2,), generator=g))
    w = torch.view_as_complex(torch.randn((cfg.hidden_dim, cfg.output_dim, 2), generator=g))
    v = torch.view_as_complex(torch.randn(shp_y + (2,), generator=g))
    # float64 oracle
    xr = x.to(torch.complex128).requires_grad_(True)
    wr = w.to(torch.complex128).requires_grad_(True)
    yr = _ref_layer(xr, wr, cfg)
    yr.backward(v.to(torch.complex128))
    # sm_100a forward + backward
    xd = x.cuda().requires_grad_(True)
    wd = w.cuda().contiguous().requires_grad_(True)
    yd = spectral_layer(xd, wd, cfg)
    yd.backward(v.cuda())
    torch.cuda.synchronize()
    assert T.max_rel_error(yd.detach().cpu().numpy(), yr.detach().numpy()) < TOL
    ex = T.max_rel_error(xd.grad.cpu().numpy(), xr.grad.numpy())
    ew = T.max_rel_error(wd.grad.cpu().numpy(), wr.grad.numpy())
    assert ex < TOL, ex
    assert ew < TOL, ew


def test_backward_only_weights():
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200.autograd import layer_backward
    cfg = T.FnoLayerConfig(2, 8, 8, 1, 256, 1, 32, 1)
    x = torch.randn(2, 8, 1, 256, dtype=torch.complex64, device="cuda")
    w = torch.randn(8, 8, dtype=torch.complex64, device="cuda")
    gy = torch.randn(2, 8, 1, 256, dtype=torch.complex64, device="cuda")
    gx, gw = layer_backward(cfg, x, w, gy, need_x=False, need_w=True)
    assert gx is None and gw.shape == (8, 8)
