#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py -q -m gpu > gpurun_out/t15.txt 2>&1; tail -3 gpurun_out/t15.txt
bash tools/sanitize.sh
