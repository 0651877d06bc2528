"""Time the real-field FNO block (realfield.fno_block: R2C layer + bypass + bias + GELU)
against the same block written with torch.fft.rfft2/irfft2 + einsum + matmul + gelu on the
GPU, and the complex layer of the same shape.  CUDA events, median of 3 x 10 reps."""
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2504_11681_b200 as T  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) / reps)
    return round(statistics.median(out), 4)


for case in [(32, 64, 64, 256, 256, 32, 32, 2), (256, 64, 64, 256, 256, 16, 16, 2), (1024, 64, 64, 1, 1024, 1, 128, 1)]:
    cfg = T.FnoLayerConfig(*case)
    B, H, N, dx, dy, kx, ky = case[:7]
    x = torch.randn(B, H, dx, dy, device='cuda')
    w = torch.randn(H, N, dtype=torch.complex64, device='cuda')
    wb = torch.randn(H, N, device='cuda')
    bias = torch.randn(N, device='cuda')
    out = torch.empty(B, N, dx, dy, device='cuda')

    def ours():
        T.fno_block(cfg, x, w, bypass_w=wb, bias=bias, activation='gelu', out=out)

    def ref():
        if cfg.rank == 2:
            X = torch.fft.rfft2(x)[..., :kx, :ky]
            y = torch.fft.irfft2(torch.einsum('bhpq,hn->bnpq', X, w), s=(dx, dy))
        else:
            X = torch.fft.rfft(x, dim=-1)[..., :ky]
            y = torch.fft.irfft(torch.einsum('bhpq,hn->bnpq', X, w), n=dy, dim=-1)
        y = y + torch.matmul(wb.t(), x.reshape(B, H, dx * dy)).reshape(B, N, dx, dy) + bias[None, :, None, None]
        return torch.nn.functional.gelu(y)

    def block64(x_, w_, wb_, b_):
        if cfg.rank == 2:
            y = torch.fft.irfft2(torch.einsum('bhpq,hn->bnpq', torch.fft.rfft2(x_)[..., :kx, :ky], w_), s=(dx, dy))
        else:
            y = torch.fft.irfft(torch.einsum('bhpq,hn->bnpq', torch.fft.rfft(x_, dim=-1)[..., :ky], w_), n=dy, dim=-1)
        y = y + torch.matmul(wb_.t(), x_.reshape(x_.shape[0], H, dx * dy)).reshape(-1, N, dx, dy)
        return torch.nn.functional.gelu(y + b_[None, :, None, None])

    xc = torch.randn(B, H, dx, dy, dtype=torch.complex64, device='cuda')
    yc = torch.empty(B, N, dx, dy, dtype=torch.complex64, device='cuda')
    t_ours, t_ref = timeit(ours), timeit(ref)
    t_c = timeit(lambda: T.run_layer_device(cfg, xc, w, out=yc, validate=False))
    # accuracy on batch[0:2] against the float64 CPU definition (pocketfft), ours and torch-CUDA fp32
    ours()
    torch.cuda.synchronize()
    f64 = block64(x[:2].double().cpu(), w.cpu().to(torch.complex128), wb.double().cpu(), bias.double().cpu())
    e_ours = T.max_rel_error(out[:2].cpu().numpy(), f64.numpy())
    e_torch = T.max_rel_error(ref()[:2].cpu().numpy(), f64.numpy())
    print(case, 'fno_block ms', t_ours, 'torch rfft2 block ms', t_ref, 'speedup', round(t_ref / t_ours, 2),
          'complex layer ms', t_c, 'err vs f64: ours %.1e torch-cuda %.1e' % (e_ours, e_torch), flush=True)
    del x, xc, yc, out
    torch.cuda.empty_cache()
