"""Accuracy check of the real-field FNO block at realistic widths: ours and torch's CUDA
fp32 (rfft2/irfft2 + einsum + matmul + gelu) against the float64 CPU definition."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2504_11681_b200 as T  # noqa: E402


def block(x, w, wb, bias, cfg):
    B, H, N, dx, dy, kx, ky = (cfg.batch, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y, cfg.keep_x,
                               cfg.keep_y)
    if cfg.rank == 2:
        y = torch.fft.irfft2(torch.einsum('bhpq,hn->bnpq', torch.fft.rfft2(x)[..., :kx, :ky], w), s=(dx, dy))
    else:
        y = torch.fft.irfft(torch.einsum('bhpq,hn->bnpq', torch.fft.rfft(x, dim=-1)[..., :ky], w), n=dy, dim=-1)
    y = y + torch.matmul(wb.t(), x.reshape(B, H, dx * dy)).reshape(B, N, dx, dy) + bias[None, :, None, None]
    return torch.nn.functional.gelu(y)


for case in [(4, 64, 64, 256, 256, 32, 32, 2), (4, 64, 64, 1, 1024, 1, 128, 1), (2, 4, 4, 256, 256, 32, 32, 2)]:
    cfg = T.FnoLayerConfig(*case)
    B, H, N, dx, dy = case[:5]
    g = torch.Generator().manual_seed(1)
    x = torch.randn(B, H, dx, dy, generator=g)
    w = torch.view_as_complex(torch.randn(H, N, 2, generator=g))
    wb = torch.randn(H, N, generator=g)
    bias = torch.randn(N, generator=g)
    ref = block(x.double(), w.to(torch.complex128), wb.double(), bias.double(), cfg)
    ours = T.fno_block(cfg, x.cuda(), w.cuda(), bypass_w=wb.cuda(), bias=bias.cuda(), activation='gelu').cpu()
    tg = block(x.cuda(), w.cuda(), wb.cuda(), bias.cuda(), cfg).cpu()
    print(case, 'ours vs f64 %.2e' % T.max_rel_error(ours.numpy(), ref.numpy()),
          'torch-cuda fp32 vs f64 %.2e' % T.max_rel_error(tg.numpy(), ref.numpy()), flush=True)
