#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused1d.py -q -m gpu -x > gpurun_out/t26.txt 2>&1; tail -2 gpurun_out/t26.txt
