"""Per-mode layer timing at the C4 shape (B128 H128 N128 512^2 keep 64^2, FP32):
run_layer_permode (spectrum fwd | tfno_permode_mix | spectrum inverse) vs the
shared-W layer, plus the mix alone vs the round-1 mix (mode-major permute
copies + batched mode CGEMM).  CUDA events, warm-up 3, median of 10."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_11681_b200 as T  # noqa: E402
from paper_2504_11681_b200 import _device
from paper_2504_11681_b200._lib import lib
from paper_2504_11681_b200.permode import prepare_weights, run_layer_permode


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    B, H, N, d, k = (int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (128, 128, 128, 512, 64)))
    cfg = T.FnoLayerConfig(B, H, N, d, d, k, k, rank=2)
    MQ = k * k
    x = torch.randn((B, H, d, d), dtype=torch.complex64, device="cuda")
    w_modes = torch.randn((H, N, k, k), dtype=torch.complex64, device="cuda")
    w = torch.randn((H, N), dtype=torch.complex64, device="cuda")
    wp = prepare_weights(w_modes)
    out = {"shape": [B, H, N, d, k]}
    out["permode_layer_ms"] = timeit(lambda: run_layer_permode(cfg, x, w_prepared=wp))
    out["shared_layer_ms"] = timeit(lambda: T.run_layer_device(cfg, x, w))
    A = torch.randn((B, H, MQ), dtype=torch.complex64, device="cuda")
    C = torch.empty((B, N, MQ), dtype=torch.complex64, device="cuda")
    st = _device.stream_ptr(None)
    out["mix_ms"] = timeit(lambda: lib().tfno_permode_mix(B, H, N, MQ, A.data_ptr(), wp.data_ptr(),
                                                           C.data_ptr(), 1.0, st))
    wq = w_modes.permute(2, 3, 0, 1).reshape(MQ, H, N).contiguous()

    def old_mix():
        Aq = A.permute(2, 1, 0).contiguous()
        Cq = torch.empty((MQ, N, B), dtype=torch.complex64, device="cuda")
        lib().tfno_cgemm(B, N, H, MQ, Aq.data_ptr(), 1, B, H * B, wq.data_ptr(), N, 1, H * N,
                         Cq.data_ptr(), 1, B, N * B, 1.0, st)
        return Cq.permute(2, 1, 0).contiguous()
    out["old_mix_ms"] = timeit(old_mix)
    ref = old_mix()
    lib().tfno_permode_mix(B, H, N, MQ, A.data_ptr(), wp.data_ptr(), C.data_ptr(), 1.0, st)
    torch.cuda.synchronize()
    out["mix_vs_old_max_rel"] = float(((C - ref).abs().max() / ref.abs().max()).item())
    flops = 8.0 * B * H * N * MQ
    out["mix_tflops"] = flops / out["mix_ms"] / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
