"""CPU, world_size 2 over gloo: the host side of the multi-GPU drivers —
batch shard bounds, max-over-ranks timing and the hidden-split reduction
(partials computed with the oracle on each rank's channel shard, summed with
the same reduce_partials the GPU path uses over NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_11681_b200 import multigpu as MG


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from types import SimpleNamespace

        from oracle import fnofuse_port as O
        res = {}
        # batch sharding: bounds tile the batch, max-over-ranks timing
        b0, b1 = MG.shard_bounds(7, world, rank)
        t = torch.tensor([b0, b1])
        allb = [torch.zeros(2, dtype=torch.long) for _ in range(world)]
        dist.all_gather(allb, t)
        res["bounds"] = [tuple(x.tolist()) for x in allb]
        res["max"] = MG.max_over_ranks(1.0 + rank)
        # hidden split: oracle spectra of this rank's channels, partial mix, reduce
        cfg = SimpleNamespace(batch=2, hidden_dim=6, output_dim=4, dim_x=8, dim_y=16, keep_x=4, keep_y=8, rank=2)
        x, w = O.random_inputs(cfg, 11)
        h0, h1 = MG.shard_bounds(cfg.hidden_dim, world, rank)
        t1 = np.fft.fft(np.fft.fft(x[:, h0:h1].astype(np.complex128), axis=2)[:, :, :4], axis=3)[..., :8]
        part = np.einsum("bhpq,hn->bnpq", t1, w[h0:h1].astype(np.complex128)).astype(np.complex64)
        C = torch.from_numpy(part.copy())
        full = MG.reduce_partials(C.clone(), "all_reduce")
        cm = torch.from_numpy(np.ascontiguousarray(part.transpose(1, 0, 2, 3)))
        blk = MG.reduce_partials(cm, "reduce_scatter")
        spec = np.zeros((2, 4, 8, 16), np.complex128)
        spec[:, :, :4, :8] = full.numpy()
        y = np.fft.ifft2(spec, axes=(2, 3))
        res["err_allreduce"] = O.max_rel_error(y, O.reference_layer(cfg, x, w))
        ref_blk = full.numpy().transpose(1, 0, 2, 3)[rank * 2:(rank + 1) * 2]
        res["err_rs"] = O.max_rel_error(blk.numpy(), ref_blk)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_world2_gloo_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    for r in range(world):
        assert out[r]["bounds"] == [(0, 4), (4, 7)]
        assert out[r]["max"] == 2.0
        assert out[r]["err_allreduce"] < 1e-5
        assert out[r]["err_rs"] < 1e-6


def test_shard_bounds_cover():
    for n in (1, 7, 128):
        for world in (1, 2, 3, 8):
            spans = [MG.shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
