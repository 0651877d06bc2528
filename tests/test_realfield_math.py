"""CPU check (float64, numpy) of the identity the real-field layer
(paper_2504_11681_b200.realfield) is composed from:

    irfft2(rfft2(x)[:kx, :ky] W, s=(dx, dy)) == Re(iDFT_pad(c * (DFT_trunc(x + 0i) W)))

with c_k = 2 for 0 < k < dy/2 (else 1) on the y bins — first-keep truncation of the
complex forward equals the kept rfft bins, and the complex padded inverse of the weighted
bins, real part, equals irfft.  DFT_trunc / iDFT_pad are the oracle's float64 DFT matrices
(tests/oracles.py composition in oracle/fnofuse_port.py)."""

import numpy as np
import pytest


def _weights(ky, dy):
    k = np.arange(ky)
    return np.where((k > 0) & (2 * k < dy), 2.0, 1.0)


@pytest.mark.parametrize("case", [
    (2, 3, 4, 1, 16, 1, 5, 1), (2, 3, 2, 1, 16, 1, 9, 1), (1, 2, 2, 1, 1, 1, 1, 1), (1, 2, 2, 1, 2, 1, 2, 1),
    (2, 3, 4, 8, 8, 3, 4, 2), (2, 2, 3, 8, 16, 8, 9, 2), (1, 2, 2, 4, 2, 2, 2, 2),
])
def test_real_layer_identity(case):
    import paper_2504_11681_b200 as T
    from oracle import fnofuse_port as O
    cfg = T.FnoLayerConfig(*case)
    rng = np.random.default_rng(sum(case))
    x = rng.standard_normal((cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y))
    w = rng.standard_normal((cfg.hidden_dim, cfg.output_dim)) + 1j * rng.standard_normal((cfg.hidden_dim,
                                                                                          cfg.output_dim))
    kx, ky = cfg.keep_x, cfg.keep_y
    # numpy real-FFT definition
    X = np.fft.rfft2(x)[..., :kx, :ky]
    ref = np.fft.irfft2(np.einsum("bhpq,hn->bnpq", X, w), s=(cfg.dim_x, cfg.dim_y))
    # the composition on complex first-keep transforms (oracle DFT matrices)
    Fx, Fy = O.dft_matrix(cfg.dim_x), O.dft_matrix(cfg.dim_y)
    A = np.einsum("jx,ky,bhxy->bhjk", Fx[:kx], Fy[:ky], x.astype(np.complex128))
    C = np.einsum("bhpq,hn->bnpq", A * _weights(ky, cfg.dim_y), w)
    y = np.einsum("xj,yk,bnjk->bnxy", np.conj(Fx[:kx]).T, np.conj(Fy[:ky]).T, C) / (cfg.dim_x * cfg.dim_y)
    assert np.abs(np.real(y) - ref).max() < 1e-12 * max(1.0, np.abs(ref).max())


def test_keep_beyond_half_spectrum_rejected():
    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200.realfield import _check_real_cfg
    with pytest.raises(T.FnofuseError):
        _check_real_cfg(T.FnoLayerConfig(1, 2, 2, 1, 16, 1, 10, 1))
    _check_real_cfg(T.FnoLayerConfig(1, 2, 2, 1, 16, 1, 9, 1))
