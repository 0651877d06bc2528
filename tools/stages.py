"""Per-kernel stage times of the layer schedules (library stage events) for a
list of workloads x modes x precisions, next to the staged cuFFT+cuBLAS
baseline.  One JSON object per line.

    python tools/stages.py --workloads C2-N256-H256-B1024,C1 [--modes fully_fused,fft_optimized]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2504_11681_b200 as T  # noqa: E402
from paper_2504_11681_b200 import _lib  # noqa: E402


def stage_times(cfg, x, w, y, mode, prec, reps=10):
    lib = _lib.lib()
    _, sched = T.layer_schedule(cfg, mode, prec)
    nst = len(sched.split("|")) + 1
    stream = torch.cuda.current_stream()
    for _ in range(3):
        T.run_layer_device(cfg, x, w, out=y, mode=mode, precision=prec, validate=False)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nst)] for _ in range(reps)]
    for row in ev:
        for e_ in row:
            e_.record(stream)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    handles = [bench.ctypes_arr(row) for row in ev]  # the library keeps the pointer during the call
    for i in range(reps):
        lib.tfno_set_stage_events(handles[i], nst)
        T.run_layer_device(cfg, x, w, out=y, mode=mode, precision=prec, validate=False)
    e.record(stream)
    torch.cuda.synchronize()
    lib.tfno_set_stage_events(None, 0)
    st = [round(statistics.median(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(reps)), 4)
          for j in range(nst - 1)]
    return sched, round(s.elapsed_time(e) / reps, 4), st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="C1,C2-N256-H64-B1024,C2-N256-H256-B1024,C2-N1024-H256-B1024,"
                                           "C2-N4096-H64-B1024,C2-N4096-H256-B256")
    ap.add_argument("--modes", default="fully_fused,fft_optimized,fused_fft_gemm,fused_gemm_ifft,staged")
    ap.add_argument("--precs", default="fp32")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for name in args.workloads.split(","):
        B, H, N, dx, dy, kx, ky, rk, desc = bench.WORKLOADS[name]
        cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, rk)
        fl = T.layer_flops(cfg)
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        x = torch.view_as_complex(torch.randn((B, H, dx, dy, 2), generator=g, device=dev))
        w = torch.view_as_complex(torch.randn((H, N, 2), generator=g, device=dev)).contiguous()
        y = torch.empty((B, N, dx, dy), dtype=torch.complex64, device=dev)
        for prec in args.precs.split(","):
            for mode in args.modes.split(","):
                if mode == "staged" and prec != "fp32":
                    continue
                try:
                    sched, ms, st = stage_times(cfg, x, w, y, mode, prec)
                except Exception as ex:  # noqa: BLE001
                    print(json.dumps({"workload": name, "mode": mode, "prec": prec, "error": str(ex)[:100]}))
                    continue
                t_roof = max(fl["bytes"] / 6534.8e9, fl["flops"] / 74.4e12) * 1e3
                print(json.dumps({"workload": name, "mode": mode, "prec": prec, "ms": ms, "sched": sched,
                                  "stages_ms": st, "roof_ms": round(t_roof, 4), "frac_roof": round(t_roof / ms, 3)}),
                      flush=True)
        T._device.release_workspace()
        del x, w, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
