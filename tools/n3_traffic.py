#!/usr/bin/env python
"""N3: kernel-launch and DRAM-traffic reduction of the fused layer vs the
unfused cuFFT + truncate + cuBLAS + pad + cuFFT^-1 pipeline, measured in ONE
process under ncu (the reference's own deliverable is the modeled version of
this comparison: fnofuse.pipeline.traffic_delta, pipeline.py:342-366).

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/n3_raw.csv python tools/n3_traffic.py run C3 C4 C5L
    python tools/n3_traffic.py summarize gpurun_out/n3_raw.csv > profiles/r02/n3_traffic.json

`run` brackets exactly one layer call per (workload, mode) with
cudaProfilerStart/Stop and prints the order of the brackets; `summarize`
attributes every captured kernel to its bracket (launch count, DRAM bytes,
kernel time) and writes the fused/unfused ratios beside the reference's
modeled ledger for the same config.
"""

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {
    "C3": (32, 64, 64, 256, 256, 32, 32, 2),
    "C4": (128, 128, 128, 512, 512, 64, 64, 2),
    "C5L": (256, 64, 64, 256, 256, 16, 16, 2),
    "C1": (16, 64, 64, 1, 128, 1, 32, 1),
    "C2-N1024-H64-B1024": (1024, 64, 64, 1, 1024, 1, 128, 1),
}
MODES = ("staged", "fully_fused")


def run(names):
    import torch

    import paper_2504_11681_b200 as T
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    order = []
    for nm in names:
        B, H, N, dx, dy, kx, ky, rk = SHAPES[nm]
        cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, rk)
        g = torch.Generator(device=dev)
        g.manual_seed(7)
        x = torch.view_as_complex(torch.randn((B, H, dx, dy, 2), generator=g, device=dev))
        w = torch.view_as_complex(torch.randn((H, N, 2), generator=g, device=dev)).contiguous()
        y = torch.empty((B, N, dx, dy), dtype=torch.complex64, device=dev)
        for mode in MODES:
            for _ in range(2):  # warm: plans, workspace, module load
                T.run_layer_device(cfg, x, w, out=y, mode=mode, validate=False)
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
            torch.cuda._sleep(100)  # bracket marker kernel (ATen spin_kernel)
            T.run_layer_device(cfg, x, w, out=y, mode=mode, validate=False)
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
            order.append({"workload": nm, "mode": mode, "schedule": T.layer_schedule(cfg, mode, "fp32")[1]})
        del x, y
        T._device.release_workspace()
        torch.cuda.empty_cache()
    with open(os.path.join(ROOT, "gpurun_out", "n3_order.json"), "w") as f:
        json.dump(order, f)
    print(json.dumps(order))


def summarize(csv_path, order_path=None):
    order_path = order_path or os.path.join(os.path.dirname(csv_path), "n3_order.json")
    order = json.load(open(order_path))
    rows = []
    with open(csv_path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    kern = {}
    for r in rows:
        kid = int(r["ID"])
        k = kern.setdefault(kid, {"name": r["Kernel Name"], "m": {}})
        v = r["Metric Value"].replace(",", "")
        try:
            val = float(v)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                 "ms": 1e-3,
                 "msecond": 1e-3, "second": 1.0}.get(r["Metric Unit"], 1.0)
        k["m"][r["Metric Name"]] = val * scale
    # every bracket starts with the marker kernel: split the launch sequence there
    groups = []
    for i in sorted(kern):
        if "spin_kernel" in kern[i]["name"]:
            groups.append([])
        elif groups:
            groups[-1].append(kern[i])
    assert len(groups) == len(order), (len(groups), len(order))
    out = []
    for o, group in zip(order, groups):
        rd = sum(k["m"].get("dram__bytes_read.sum", 0) for k in group)
        wr = sum(k["m"].get("dram__bytes_write.sum", 0) for k in group)
        t = sum(k["m"].get("gpu__time_duration.sum", 0) for k in group)
        out.append(dict(o, launches=len(group), dram_read=rd, dram_write=wr, dram_bytes=rd + wr,
                        kernel_time_ms=round(t * 1e3, 4), kernels=[k["name"][:90] for k in group]))
    res = {"_source": os.path.basename(csv_path), "_how": __doc__.strip().splitlines()[0], "points": out}
    for nm in sorted({o["workload"] for o in out}):
        pts = {o["mode"]: o for o in out if o["workload"] == nm}
        if "staged" in pts and "fully_fused" in pts:
            s, f = pts["staged"], pts["fully_fused"]
            res[nm] = {"launches_staged": s["launches"], "launches_fused": f["launches"],
                       "dram_GB_staged": round(s["dram_bytes"] / 1e9, 3),
                       "dram_GB_fused": round(f["dram_bytes"] / 1e9, 3),
                       "dram_reduction": round(1 - f["dram_bytes"] / s["dram_bytes"], 4) if s["dram_bytes"] else None,
                       "kernel_ms_staged": s["kernel_time_ms"], "kernel_ms_fused": f["kernel_time_ms"]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2:])
    else:
        summarize(*sys.argv[2:])
