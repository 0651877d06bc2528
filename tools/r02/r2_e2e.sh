#!/bin/bash
# e2e A/B of HostPipeline chunk / copy-stream counts on C4 (pinned host buffers)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "host_pipeline or device_api" > gpurun_out/t17.txt 2>&1; tail -2 gpurun_out/t17.txt
timeout 1200 python - <<'PY' > gpurun_out/e2e_ab.txt 2>&1
import time, torch, paper_2504_11681_b200 as T
cfg = T.FnoLayerConfig(128, 128, 128, 512, 512, 64, 64, 2)
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.view_as_complex(torch.randn((128, 128, 512, 512, 2), generator=g, device="cuda"))
xh = torch.empty(x.shape, dtype=torch.complex64, pin_memory=True); xh.copy_(x); del x
yh = torch.empty(xh.shape, dtype=torch.complex64, pin_memory=True)
w = torch.view_as_complex(torch.randn((128, 128, 2)))
torch.cuda.empty_cache()
import sys; sys.path.insert(0, "tools/r02/ab"); import old_hostpipeline as OLD
for chunk, nbuf, ncopy in [("old", 4, 3), (1, 4, 2), ("old", 2, 3), (4, 4, 2), ("old", 4, 4), (2, 4, 2), ("old", 1, 3)]:
    pipe = (OLD.HostPipeline(cfg, chunk=nbuf, nstreams=ncopy) if chunk == "old" else
            T.pipeline.HostPipeline(cfg, chunk=chunk, nbuf=nbuf, ncopy=ncopy))
    pipe(xh, w, yh); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        pipe(xh, w, yh)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 500
    print(f"chunk {chunk} nbuf {nbuf} ncopy {ncopy}: {ms:.1f} ms/step, {2 * 34.36e9 / (ms * 1e-3) / 1e9:.1f} GB/s both directions", flush=True)
    del pipe; torch.cuda.empty_cache()
PY
cat gpurun_out/e2e_ab.txt
