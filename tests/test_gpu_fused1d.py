"""GPU parity of the fused 1D layer kernel (fused1d.cu: FFT -> truncate ->
channel CGEMM -> zero-pad -> iFFT in one launch, TMA producer warp) against
the numpy oracle restatement of ``fnofuse.pipeline.run_layer`` and against
the unfused schedule of the same library (y-FFT | CGEMM | y-iFFT).

Shapes: the BASELINE C2 sweep's (N, H) grid with keep = N/8 at small batch,
plus ragged keep (masked bins), rank-2 rows (the x-FFT/x-iFFT passes around
the fused rows kernel) and a multi-item-per-CTA batch.  Tolerance: FP32 1e-5
(max_rel_error, core.py:39-50)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5


@pytest.fixture(scope="module")
def T():
    import paper_2504_11681_b200 as T
    return T


@pytest.fixture(scope="module")
def O():
    from oracle import fnofuse_port as O
    return O


CASES = [
    # (batch, H, N_out, dim_x, dim_y, keep_x, keep_y, rank)
    (3, 64, 64, 1, 256, 1, 32, 1),
    (2, 128, 128, 1, 256, 1, 32, 1),
    (2, 256, 256, 1, 256, 1, 32, 1),
    (2, 64, 64, 1, 1024, 1, 128, 1),
    (2, 64, 64, 1, 1024, 1, 64, 1),      # N = 1024, keep 64 (KP = 2)
    (2, 64, 128, 1, 256, 1, 16, 1),      # H != N_out, keep <= 16
    (2, 32, 64, 1, 256, 1, 20, 1),       # ragged keep (masked bins), H = 2 chunks
    (2, 128, 64, 1, 256, 1, 50, 1),      # keep 50 -> KP = 4 tile
    (2, 64, 64, 4, 256, 2, 32, 2),       # rank 2: x passes around the fused rows
    (16, 64, 64, 1, 128, 1, 32, 1),      # C1 exactly: N = 128 rows (16 lanes x 8), split 4
    (3, 32, 64, 1, 128, 1, 20, 1),       # N = 128, ragged keep
    (4, 128, 128, 1, 1024, 1, 128, 1),   # N_out 128 at N = 1024: forced output split (2 x 64)
]


def _schedule(T, cfg):
    return T.layer_schedule(cfg, "fully_fused")[1]


@pytest.mark.parametrize("case", CASES)
def test_fused1d_vs_oracle(T, O, case):
    cfg = T.FnoLayerConfig(*case)
    # C1-sized layers (one wave of (batch, 8-channel) CTAs) take the tiny1d kernel instead
    assert "fused1d" in _schedule(T, cfg) or "tiny1d" in _schedule(T, cfg), _schedule(T, cfg)
    x, w = O.random_inputs(cfg, 2000 + sum(case))
    out, led = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
    ref = O.run_layer_values(cfg, x, w)
    err = T.max_rel_error(out.data, ref)
    assert err < FP32_TOL, (case, err)
    exact = O.reference_layer(cfg, x, w)
    assert T.max_rel_error(out.data, exact) < FP32_TOL


@pytest.mark.parametrize("n,h,keep", [(256, 64, 32), (256, 256, 32), (1024, 64, 128), (128, 64, 32)])
def test_fused1d_many_items_vs_unfused(T, n, h, keep):
    """Batch >> #SMs (several items per persistent CTA, ring phases wrap):
    fused == unfused schedule within FP32 tolerance, and deterministic."""
    import torch
    cfg = T.FnoLayerConfig(700, h, h, 1, n, 1, keep, 1)
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    x = torch.view_as_complex(torch.randn((cfg.batch, h, 1, n, 2), generator=g, device="cuda"))
    w = torch.view_as_complex(torch.randn((h, h, 2), generator=g, device="cuda")).contiguous()
    y1 = T.run_layer_device(cfg, x, w, mode="fully_fused").clone()
    y2 = T.run_layer_device(cfg, x, w, mode="fft_optimized")
    y3 = T.run_layer_device(cfg, x, w, mode="fully_fused")
    torch.cuda.synchronize()
    a, b = y1.cpu().numpy(), y2.cpu().numpy()
    assert T.max_rel_error(a, b) < FP32_TOL
    assert torch.equal(y1, y3)
    assert np.isfinite(a).all()


TINY = [
    (16, 64, 64, 1, 128, 1, 32, 1),   # C1 exactly
    (3, 64, 64, 1, 128, 1, 32, 1),
    (5, 37, 21, 1, 128, 1, 20, 1),    # ragged H, N (last CTA has 5 channels), ragged keep
    (2, 128, 8, 1, 128, 1, 64, 1),    # keep 64 (4 bin groups), H = 128
    (4, 16, 30, 1, 128, 1, 1, 1),     # keep 1
    (1, 200, 3, 1, 128, 1, 33, 1),    # H not a multiple of the 64-row batches of the teams
    (64, 64, 64, 1, 256, 1, 32, 1),   # C2 N256-H64-B64 (32 channels per CTA)
    (64, 128, 128, 1, 256, 1, 32, 1), # C2 N256-H128-B64 (64 channels per CTA)
    (64, 64, 64, 1, 1024, 1, 128, 1), # C2 N1024-H64-B64 (32-lane teams)
    (7, 50, 70, 1, 256, 1, 20, 1),    # ragged N / keep, 8 channels per CTA
    (40, 33, 100, 1, 1024, 1, 100, 1),  # keep 100 -> 4 bin groups, 64 channels per CTA, ragged tail
    (5, 20, 40, 1, 256, 1, 64, 1),    # keep 64 at N = 256
]


def test_tiny1d_default_selection(T):
    """tiny1d is the default only where it was measured faster (N <= 256, H <= 64, <= 32 channels per CTA)."""
    for case, want in [((16, 64, 64, 1, 128, 1, 32, 1), "tiny1d"), ((64, 64, 64, 1, 256, 1, 32, 1), "tiny1d"),
                       ((64, 128, 128, 1, 256, 1, 32, 1), "fused1d"), ((64, 64, 64, 1, 1024, 1, 128, 1), "fused1d")]:
        assert _schedule(T, T.FnoLayerConfig(*case)).startswith(want), case


_TINY_CODE = r"""
import numpy as np, paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
for case in CASES:
    cfg = T.FnoLayerConfig(*case)
    assert T.layer_schedule(cfg, "fully_fused")[1] == "tiny1d-fft-cgemm-ifft", case
    x, w = O.random_inputs(cfg, 3000 + sum(case))
    out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
    err = T.max_rel_error(out.data, O.run_layer_values(cfg, x, w))
    assert err < 1e-5, (case, err)
    again, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
    assert np.array_equal(out.data, again.data), case
print("ok")
"""


def test_tiny1d_forced_every_shape():
    """TFNO_TINY1D=1: the kernel on every shape it fits (N = 128 / 256 / 1024, 8 / 32 / 64 channels
    per CTA, ragged N and keep, 1..4 bin groups) vs the oracle, bitwise determinism."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _TINY_CODE.replace("CASES", repr(TINY))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PYTHONPATH=root, TFNO_TINY1D="1"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("case", TINY)
def test_tiny1d_vs_oracle(T, O, case):
    """The default schedule (tiny1d where it wins, else fused1d) on the tiny
    shapes vs the oracle; bitwise determinism."""
    cfg = T.FnoLayerConfig(*case)
    x, w = O.random_inputs(cfg, 3000 + sum(case))
    out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
    err = T.max_rel_error(out.data, O.run_layer_values(cfg, x, w))
    assert err < FP32_TOL, (case, err)
    again, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
    assert np.array_equal(out.data, again.data)


def test_tiny1d_off_keeps_fused1d():
    import os
    import subprocess
    import sys
    code = r"""
import paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
cfg = T.FnoLayerConfig(16, 64, 64, 1, 128, 1, 32, 1)
assert T.layer_schedule(cfg, "fully_fused")[1] == "fused1d-fft-cgemm-ifft"
x, w = O.random_inputs(cfg, 1)
out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
assert T.max_rel_error(out.data, O.run_layer_values(cfg, x, w)) < 1e-5
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PYTHONPATH=root, TFNO_TINY1D="0"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("mode", ["fused_fft_gemm", "fused_gemm_ifft"])
@pytest.mark.parametrize("case", [c for c in CASES if c[6] % 2 == 0])
def test_fused1d_partial_modes(T, O, case, mode):
    """K4 (fused_fft_gemm: the fused kernel's FFT + GEMM half writes C, then the
    padded y-iFFT pass) and K5 (fused_gemm_ifft: the y-FFT pass writes A, the
    kernel's GEMM + iFFT half reads it) vs the oracle of the same mode."""
    cfg = T.FnoLayerConfig(*case)
    sched = T.layer_schedule(cfg, mode)[1]
    assert "fused1d" in sched, sched
    x, w = O.random_inputs(cfg, 5000 + sum(case))
    out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode=mode)
    err = T.max_rel_error(out.data, O.run_layer_values(cfg, x, w, mode))
    assert err < FP32_TOL, (case, mode, err)


@pytest.mark.parametrize("case", [(3, 128, 128, 1, 1024, 1, 128, 1), (100, 256, 256, 1, 1024, 1, 128, 1),
                                  (2, 256, 256, 1, 1024, 1, 96, 1), (5, 128, 512, 1, 1024, 1, 128, 1),
                                  (80, 96, 128, 1, 1024, 1, 128, 1)])
def test_fused_gemm_ifft_channel_split(T, O, case):
    """K5 where the full C tile does not fit one CTA (N = 1024 with 128+ output
    channels): the output channels are split across items at any batch (each
    split streams the same A rows, nothing is recomputed) — vs the oracle."""
    cfg = T.FnoLayerConfig(*case)
    assert T.layer_schedule(cfg, "fused_gemm_ifft")[1] == "y-fft|fused1d-cgemm-ifft"
    x, w = O.random_inputs(cfg, 7000 + sum(case))
    out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fused_gemm_ifft")
    err = T.max_rel_error(out.data, O.run_layer_values(cfg, x, w, "fused_gemm_ifft"))
    assert err < FP32_TOL, (case, err)
