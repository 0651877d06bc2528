"""GPU parity of the generic per-plane 2D kernels (csrc/plane_g.cuh): every
power-of-two dy in 64..1024, dx up to 1024 (square and non-square), keeps up to
128 per axis incl. ragged keeps (padded to KP, masked bins written as zeros)
and keep == dim -- against the float64 composition of the reference layer
(oracle.reference_layer == tests/oracles.py:78-94) and the fp32 oracle port of
fnofuse.run_layer.  Covers the reference acceptance grid's rank-2 geometries
(test_acceptance.py:97-105: dims 128/256 x keeps 64/128).  FP32 bar 1e-5."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
# FP32 default: channel mix fused into the inverse; TFNO_PLANE_FUSEDMIX=0 keeps the standalone CGEMM
PLANES = ("plane-fft2d|plane-mix-ifft2d", "plane-fft2d|cgemm-modes|plane-ifft2d")

# (B, H, N, dx, dy, kx, ky)
SHAPES = [
    # reference acceptance grid, rank 2 (dims 128/256, keep 64/128; hidden 16..128)
    (1, 16, 16, 128, 128, 64, 64),
    (1, 32, 32, 128, 128, 128, 128),
    (1, 16, 16, 256, 256, 64, 64),
    (1, 16, 16, 256, 256, 128, 128),
    (1, 128, 128, 128, 128, 64, 64),
    # every row length, several keeps
    (2, 3, 5, 64, 64, 8, 8),
    (2, 3, 4, 64, 64, 32, 32),
    (1, 4, 3, 64, 64, 64, 64),
    (2, 3, 2, 128, 128, 16, 16),
    (2, 2, 3, 128, 128, 32, 32),
    (1, 3, 2, 256, 256, 8, 8),
    (2, 2, 2, 512, 512, 16, 16),
    (1, 2, 3, 512, 512, 32, 32),
    (1, 2, 2, 512, 512, 128, 128),
    (1, 2, 3, 1024, 1024, 64, 64),
    (1, 2, 2, 1024, 1024, 8, 8),
    (1, 1, 2, 1024, 1024, 128, 128),
    # non-square planes
    (2, 3, 4, 64, 512, 16, 16),
    (1, 2, 3, 1024, 128, 32, 32),
    (2, 2, 3, 256, 64, 8, 8),
    (1, 3, 2, 128, 1024, 64, 64),
    # ragged keeps (masked to kx x ky inside the padded KP x KP tile)
    (2, 3, 5, 256, 256, 20, 12),
    (2, 3, 3, 128, 512, 9, 100),
    (1, 2, 3, 512, 256, 33, 20),
    (2, 4, 4, 64, 64, 1, 5),
    (1, 3, 3, 256, 128, 128, 3),
    # more planes than CTAs (persistent loop wraps many times)
    (64, 8, 8, 64, 64, 8, 8),
    (16, 16, 16, 128, 128, 16, 16),
]


@pytest.fixture(scope="module")
def T():
    import paper_2504_11681_b200 as T
    return T


@pytest.fixture(scope="module")
def O():
    from oracle import fnofuse_port as O
    return O


def _ids(s):
    return "B{}H{}N{}_{}x{}_k{}x{}".format(*s)


@pytest.mark.parametrize("shape", SHAPES, ids=_ids)
def test_generic_plane_layer(T, O, shape):
    B, H, N, dx, dy, kx, ky = shape
    cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, rank=2)
    assert T.layer_schedule(cfg, "fully_fused", "fp32")[1] in PLANES, shape
    x, w = O.random_inputs(cfg, 1000 + sum(shape))
    out, led = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    exact = O.reference_layer(cfg, x, w)
    err = T.max_rel_error(out.data, exact)
    assert err < FP32_TOL, (shape, err)
    if B * H * dx * dy <= (1 << 20):
        ref = O.run_layer_values(cfg, x, w)
        assert T.max_rel_error(out.data, ref) < FP32_TOL


def test_generic_plane_deterministic(T, O):
    cfg = T.FnoLayerConfig(3, 5, 4, 256, 128, 24, 40, rank=2)
    x, w = O.random_inputs(cfg, 5)
    a, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    b, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    assert np.array_equal(a.data, b.data)


def test_generic_plane_zero_and_identity(T, O):
    cfg = T.FnoLayerConfig(2, 4, 4, 128, 128, 128, 128, rank=2)  # keep == dim, W = I: the layer is the identity
    x, _ = O.random_inputs(cfg, 9)
    w = np.eye(4, dtype=np.complex64)
    out, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    assert T.max_rel_error(out.data, x) < FP32_TOL
    z, _ = T.run_fused(cfg, T.SpectralTensor(np.zeros_like(x)), T.ComplexMatrix(w))
    assert not np.any(z.data)


@pytest.mark.parametrize("mix", ["1", "2", "3"])
def test_generic_kernels_on_tuned_geometries(mix):
    """TFNO_PLANE_GENERIC=<mix> routes the four hand-tuned geometries (C3/C4/C5
    planes) through the generic forward (bit 0) and/or inverse (bit 1), the
    other kernel being the tuned one in natural mode order: same parity bar."""
    code = r"""
import numpy as np, paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
for s in [(1, 3, 4, 512, 512, 64, 64), (2, 3, 2, 256, 256, 32, 32), (2, 2, 3, 256, 256, 16, 16), (2, 3, 3, 128, 128, 16, 16)]:
    cfg = T.FnoLayerConfig(*s, rank=2)
    x, w = O.random_inputs(cfg, 3)
    out, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    err = T.max_rel_error(out.data, O.reference_layer(cfg, x, w))
    assert err < 1e-5, (s, err)
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TFNO_PLANE_GENERIC=mix, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


_FUSEDMIX_CODE = r"""
import numpy as np, paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
FM, PREC, TOL = "@FM@", "@PREC@", @TOL@
want = "plane-fft2d|plane-mix-ifft2d" if FM == "1" else "plane-fft2d|cgemm-modes|plane-ifft2d"
for s in [(2, 3, 13, 512, 512, 64, 64), (64, 8, 64, 64, 64, 16, 16), (40, 21, 19, 128, 128, 32, 32),
          (3, 70, 9, 256, 128, 20, 12), (2, 5, 8, 64, 512, 16, 16), (1, 300, 17, 128, 64, 16, 16),
          (2, 2, 3, 256, 256, 16, 16), (600, 2, 5, 64, 64, 8, 8)]:
    cfg = T.FnoLayerConfig(*s, rank=2)
    d = T.layer_schedule(cfg, "fully_fused", PREC)[1]
    kp = max(8, 1 << (max(s[5], s[6]) - 1).bit_length())
    assert d == want or kp not in (16, 32, 64), (s, d)
    x, w = O.random_inputs(cfg, 7 + s[0])
    out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused", precision=PREC)
    err = T.max_rel_error(out.data, O.reference_layer(cfg, x, w))
    assert err < TOL, (s, err)
    b, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused", precision=PREC)
    assert np.array_equal(out.data, b.data), s
print("ok")
"""


@pytest.mark.parametrize("fusedmix,prec,tol", [("0", "fp32", 1e-5), ("1", "fp32", 1e-5), ("1", "tf32x3", 1e-5),
                                               ("1", "tf32", 1e-3), ("0", "tf32x3", 1e-5)])
def test_fused_mix_inverse(fusedmix, prec, tol):
    """plane_invmix_g (channel mix inside the inverse kernel, C in a per-CTA
    two-task ring) and the standalone-CGEMM schedule: ragged N (tasks of 8
    output channels), H not a multiple of the A chunk, more tasks than CTAs
    (the C ring and the A ring wrap many times), every fused KP (16/32/64),
    non-square planes, the C4 plane shape; FP32 bar vs the float64
    composition, bitwise determinism.  prec tf32 / tf32x3: the tcgen05 mix
    (TMEM accumulators, K-major canonical A / W' tiles), bars 1e-3 / 1e-5."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TFNO_PLANE_FUSEDMIX=fusedmix, PYTHONPATH=root)
    code = _FUSEDMIX_CODE.replace("@FM@", fusedmix).replace("@PREC@", prec).replace("@TOL@", repr(tol))
    r = subprocess.run([sys.executable, "-c", code], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("shape", [(2, 3, 4, 256, 256, 64, 64), (1, 2, 3, 128, 512, 32, 32)], ids=_ids)
def test_generic_plane_spectrum_api(T, O, shape):
    """tfno_spectrum_forward / inverse on the generic kernels (natural [kx][ky] modes)."""
    import torch
    B, H, N, dx, dy, kx, ky = shape
    cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, rank=2)
    x, _ = O.random_inputs(cfg, 11)
    from paper_2504_11681_b200 import multigpu as MG
    xd = torch.from_numpy(x).cuda()
    modes = MG.spectrum_forward(cfg, xd)
    want = np.fft.fft2(x.astype(np.complex128))[:, :, :kx, :ky]
    assert T.max_rel_error(modes.cpu().numpy(), want) < FP32_TOL
    cfgi = T.FnoLayerConfig(B, H, H, dx, dy, kx, ky, rank=2)
    back = MG.spectrum_inverse(cfgi, modes, (B, H))
    spec = np.zeros((B, H, dx, dy), np.complex128)
    spec[:, :, :kx, :ky] = want
    assert T.max_rel_error(back.cpu().numpy(), np.fft.ifft2(spec)) < FP32_TOL


@pytest.mark.parametrize("shape", [(2, 3, 13, 512, 512, 64, 64), (3, 5, 9, 256, 256, 32, 32), (4, 6, 7, 128, 256, 20, 12),
                                   (2, 4, 4, 256, 256, 16, 16)], ids=_ids)
def test_plane_fused_gemm_ifft_mode(T, O, shape):
    """mode fused_gemm_ifft on rank-2 planes = plane forward + the fused channel
    mix / inverse kernel (the GEMM-iFFT fusion), vs the oracle of that mode."""
    B, H, N, dx, dy, kx, ky = shape
    cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, rank=2)
    assert T.layer_schedule(cfg, "fused_gemm_ifft")[1] == "plane-fft2d|plane-mix-ifft2d"
    x, w = O.random_inputs(cfg, 60 + sum(shape))
    out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fused_gemm_ifft")
    assert T.max_rel_error(out.data, O.run_layer_values(cfg, x, w, "fused_gemm_ifft")) < FP32_TOL


_SKEW_CODE = r"""
import sys, numpy as np, paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
res = {}
# the tuned geometries (C3 / C5 planes, 128^2 keep 16) with more planes than CTAs, and the
# spectrum API (the forward kernel's modes alone)
for s in [(40, 8, 5, 256, 256, 32, 32), (80, 4, 3, 256, 256, 16, 16), (64, 5, 2, 128, 128, 16, 16),
          (1, 3, 2, 256, 256, 32, 32)]:
    cfg = T.FnoLayerConfig(*s, rank=2)
    x, w = O.random_inputs(cfg, 11 + s[0])
    out, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    err = T.max_rel_error(out.data, O.reference_layer(cfg, x, w))
    assert err < 1e-5, (s, err)
    for _ in range(4):  # a hand-off race between the class buffers would show as run-to-run noise
        again, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
        assert np.array_equal(again.data, out.data), s
    res[str(s)] = out.data
np.savez(sys.argv[1], **res)
print("ok")
"""


def test_forward_skewed_class_tail_bitwise(tmp_path):
    """The tuned forward's software-pipelined class tail (TFNO_PLANE_SKEW=1,
    default: column pass 1 of class c-1 and pass 2 of class c-2 beside the rows
    of class c, one barrier per class) and the inverse's pipelined class head
    (TFNO_PLANE_ISKEW=1: pass 2 of class c+1 and pass 1 of class c+2 beside the
    rows of class c, double-buffered mode tile) run the same operations in the
    same order as the three-barrier versions (=0): bitwise-equal layers."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("0", "1"):
        f = str(tmp_path / f"skew{v}.npz")
        env = dict(os.environ, TFNO_PLANE_SKEW=v, TFNO_PLANE_ISKEW=v, PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", _SKEW_CODE, f], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
        outs.append(np.load(f))
    for k in outs[0].files:
        assert np.array_equal(outs[0][k], outs[1][k]), k
