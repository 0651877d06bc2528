"""A captured chain (CUDA graph) owns its workspace: replays stay valid after
other calls regrow or release the shared per-device scratch (regression: the
bench's tf32x3 variants regrew the scratch under the C5 graph)."""

import pytest

pytestmark = pytest.mark.gpu


def test_chain_graph_survives_shared_workspace_regrowth():
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200 import _device
    from paper_2504_11681_b200.chain import FnoChain
    cfg = T.FnoLayerConfig(4, 16, 16, 256, 256, 16, 16, 2)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.view_as_complex(torch.randn((4, 16, 256, 256, 2), generator=g, device="cuda"))
    ws = [torch.view_as_complex(torch.randn((16, 16, 2), generator=g, device="cuda")).contiguous() for _ in range(3)]
    chain = FnoChain(cfg, ws).capture(x)
    y0 = chain.forward(x).clone()
    # regrow and release the shared scratch (tensor-core precision needs the W' image on top)
    T.run_layer_device(cfg, x, ws[0], precision="tf32x3")
    T.run_layer_device(T.FnoLayerConfig(4, 16, 16, 256, 256, 16, 16, 2), x, ws[1], mode="staged")
    _device.release_workspace()
    junk = torch.randn(64 << 20, device="cuda")  # reuse freed memory
    y1 = chain.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    del junk
