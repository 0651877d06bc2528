"""CPU check of the adjoint formulas the GPU backward (paper_2504_11681_b200.autograd)
is built from, in float64 with the oracle's naive-DFT layer (tests/oracles.py
composition) against torch autograd of the same layer:

    grad_x = layer(cfg with H <-> N, gy, W^H)
    grad_W = (1/(dx*dy)) * sum_{b,modes} conj(E x) (E gy)^T
"""

import numpy as np
import pytest


def _spectrum(cfg, x):
    from oracle import fnofuse_port as O
    t = np.asarray(x, np.complex128)
    if cfg.rank == 2:
        t = np.einsum("jx,bhxy->bhjy", O.dft_matrix(cfg.dim_x), t)[:, :, :cfg.keep_x, :]
    return np.einsum("jy,bhxy->bhxj", O.dft_matrix(cfg.dim_y), t)[..., :cfg.keep_y]


@pytest.mark.parametrize("case", [(2, 3, 4, 1, 16, 1, 5, 1), (2, 3, 2, 8, 8, 3, 4, 2)])
def test_adjoint_formulas_vs_torch_autograd(case):
    import torch

    import paper_2504_11681_b200 as T
    from oracle import fnofuse_port as O
    cfg = T.FnoLayerConfig(*case)
    cfgT = T.FnoLayerConfig(cfg.batch, cfg.output_dim, cfg.hidden_dim, cfg.dim_x, cfg.dim_y,
                            cfg.keep_x, cfg.keep_y, cfg.rank)
    rng = np.random.default_rng(3)
    cplx = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
    x = cplx(cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y)
    w = cplx(cfg.hidden_dim, cfg.output_dim)
    gy = cplx(cfg.batch, cfg.output_dim, cfg.dim_x, cfg.dim_y)

    def layer_t(xt, wt):  # Appendix A with torch (differentiable), float64
        if cfg.rank == 2:
            X = torch.fft.fft2(xt)[..., :cfg.keep_x, :cfg.keep_y]
            return torch.fft.ifft2(torch.einsum("bhpq,hn->bnpq", X, wt), s=(cfg.dim_x, cfg.dim_y))
        X = torch.fft.fft(xt, dim=-1)[..., :cfg.keep_y]
        return torch.fft.ifft(torch.einsum("bhpq,hn->bnpq", X, wt), n=cfg.dim_y, dim=-1)

    xt = torch.tensor(x, requires_grad=True)
    wt = torch.tensor(w, requires_grad=True)
    yt = layer_t(xt, wt)
    assert np.abs(yt.detach().numpy() - O.reference_layer(cfg, x, w)).max() < 1e-10
    yt.backward(torch.tensor(gy))
    gx = O.reference_layer(cfgT, gy, np.conj(w).T)
    A, G = _spectrum(cfg, x), _spectrum(cfgT, gy)
    gw = np.einsum("bhpq,bnpq->hn", np.conj(A), G) / (cfg.dim_x * cfg.dim_y)
    assert np.abs(gx - xt.grad.numpy()).max() < 1e-10
    assert np.abs(gw - wt.grad.numpy()).max() < 1e-10
