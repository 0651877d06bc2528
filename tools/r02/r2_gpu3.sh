#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gputests.txt 2>&1; tail -5 gpurun_out/gputests.txt
bash tools/plane_mix.sh gpurun_out/plane_mix.txt
