"""GPU (single device): the per-rank compute of the multi-GPU drivers.
Batch shards are bitwise equal to the unsharded run (batch elements are
independent); hidden-split partials summed over ranks equal the full layer;
the spectrum-level entry points match the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2504_11681_b200 as T
    from oracle import fnofuse_port as O
    from paper_2504_11681_b200 import multigpu as MG
    return T, O, MG, torch


@pytest.mark.parametrize("shape", [(6, 8, 8, 256, 256, 32, 32, 2), (5, 16, 12, 1, 256, 1, 32, 1),
                                   (4, 6, 5, 32, 64, 8, 16, 2)])
def test_batch_shards_bitwise_equal_unsharded(env, shape):
    T, O, MG, torch = env
    cfg = T.FnoLayerConfig(*shape)
    x, w = O.random_inputs(cfg, 3)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    full = T.run_layer_device(cfg, xd, wd)
    for world in (2, 3):
        parts = []
        for r in range(world):
            sh = MG.BatchSharded(cfg, world, r)
            b0, b1 = sh.bounds
            parts.append(sh.forward(xd[b0:b1].contiguous(), wd))
        assert torch.equal(torch.cat(parts), full)


@pytest.mark.parametrize("shape", [(2, 16, 8, 256, 256, 32, 32, 2), (3, 12, 6, 32, 64, 8, 16, 2),
                                   (3, 10, 4, 1, 128, 1, 32, 1)])
def test_hidden_split_partials_sum_to_layer(env, shape):
    T, O, MG, torch = env
    cfg = T.FnoLayerConfig(*shape)
    x, w = O.random_inputs(cfg, 4)
    ref = O.run_layer_values(cfg, x, w)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    world = 2
    C = None
    for r in range(world):
        h0, h1 = MG.shard_bounds(cfg.hidden_dim, world, r)
        part = MG.hidden_split_partial(cfg, xd[:, h0:h1].contiguous(), wd[h0:h1])
        C = part if C is None else C + part       # what all_reduce(SUM) computes over NVLink
    oc = T.FnoLayerConfig(cfg.batch, 1, cfg.output_dim, cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y, cfg.rank)
    y = MG.spectrum_inverse(oc, C, (cfg.batch, cfg.output_dim))
    assert T.max_rel_error(y.cpu().numpy(), ref) < 1e-5


@pytest.mark.parametrize("shape", [(2, 3, 3, 512, 512, 64, 64, 2), (2, 3, 3, 64, 32, 8, 4, 2), (3, 2, 2, 1, 64, 1, 8, 1)])
def test_spectrum_entry_points_vs_oracle(env, shape):
    T, O, MG, torch = env
    cfg = T.FnoLayerConfig(*shape)
    x, _ = O.random_inputs(cfg, 5)
    modes = MG.spectrum_forward(cfg, torch.from_numpy(x).cuda())
    want = O.dft_oracle(x) if cfg.rank == 1 else None
    t = x.astype(np.complex128)
    if cfg.rank == 2:
        t = np.einsum("jx,bhxy->bhjy", O.dft_matrix(cfg.dim_x), t)[:, :, :cfg.keep_x, :]
    want = np.einsum("jy,bhxy->bhxj", O.dft_matrix(cfg.dim_y), t)[..., :cfg.keep_y]
    assert T.max_rel_error(modes.cpu().numpy(), want) < 1e-5
    oc = T.FnoLayerConfig(cfg.batch, 1, cfg.hidden_dim, cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y, cfg.rank)
    y = MG.spectrum_inverse(oc, modes, (cfg.batch, cfg.hidden_dim), scale=2.0)
    spec = np.zeros(x.shape, np.complex128)
    spec[:, :, :cfg.keep_x, :cfg.keep_y] = want
    yr = 2.0 * np.fft.ifft2(spec, axes=(2, 3))
    assert T.max_rel_error(y.cpu().numpy(), yr) < 1e-5


def test_chain_graph_matches_chained_layers(env):
    """4-layer chain (BASELINE configs[4] shape, reduced batch) captured in a
    CUDA graph == chained reference run_layer calls (oracle)."""
    T, O, MG, torch = env
    from paper_2504_11681_b200.chain import FnoChain
    cfg = T.FnoLayerConfig(2, 8, 8, 256, 256, 16, 16, rank=2)
    x, _ = O.random_inputs(cfg, 21)
    rng = np.random.default_rng(3)
    ws = [(rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))).astype(np.complex64) for _ in range(4)]
    xd = torch.from_numpy(x).cuda()
    ch = FnoChain(cfg, [torch.from_numpy(w).cuda() for w in ws]).capture(xd)
    assert ch.kernels_per_forward == 12
    y = ch.forward(xd).cpu().numpy()
    ref = x
    for w in ws:
        ref = O.run_layer_values(cfg, ref, w)
    assert T.max_rel_error(y, ref) < 1e-5
    y2 = ch.forward(xd).cpu().numpy()
    assert np.array_equal(y, y2)


_NCCL_WORKER = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
import paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
from paper_2504_11681_b200 import multigpu as MG
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", rank=rank, world_size=world)
cfg = T.FnoLayerConfig(2, 8, 4 * world, 64, 64, 16, 16, 2)
x, w = O.random_inputs(cfg, 12)
ref = O.run_layer_values(cfg, x, w)
h0, h1 = MG.shard_bounds(cfg.hidden_dim, world, rank)
xd = torch.from_numpy(x[:, h0:h1].copy()).cuda()
wd = torch.from_numpy(w[h0:h1].copy()).cuda()
s = torch.cuda.Stream()  # a non-current stream: partial CGEMM -> NCCL -> inverse ordered on it
y = MG.hidden_split_forward(cfg, xd, wd, how="all_reduce", stream=s)
torch.cuda.synchronize()
assert T.max_rel_error(y.cpu().numpy(), ref) < 1e-5, "all_reduce"
yb = MG.hidden_split_forward(cfg, xd, wd, how="reduce_scatter", stream=s)  # [N/world, B, dx, dy]
torch.cuda.synchronize()
nr = cfg.output_dim // world
mine = np.transpose(ref[:, rank * nr:(rank + 1) * nr], (1, 0, 2, 3))
assert T.max_rel_error(yb.cpu().numpy(), mine) < 1e-5, "reduce_scatter"
dist.barrier()
dist.destroy_process_group()
print("ok", rank)
"""


def _run_nccl(world):
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(world):
        e = dict(os.environ, PYTHONPATH=root, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                 MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", _NCCL_WORKER], env=e, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, err) in zip(procs, outs):
        assert p.returncode == 0 and "ok" in o, err[-3000:]


def test_hidden_split_nccl_single_rank():
    """The NCCL data plane of the hidden-dimension split (all_reduce and
    reduce_scatter over a process group on the nccl backend), run as a
    world-1 group on this GPU: exercises the collective calls and their
    ordering after the partial CGEMM on a non-current stream."""
    _run_nccl(1)


def test_hidden_split_nccl_two_gpus():
    """Two ranks on two GPUs over NVLink (skipped on a one-GPU box)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    _run_nccl(2)
