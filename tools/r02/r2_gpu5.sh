#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu -x > gpurun_out/gen_tests.txt 2>&1; tail -3 gpurun_out/gen_tests.txt
bash tools/plane_mix.sh gpurun_out/plane_mix.txt
