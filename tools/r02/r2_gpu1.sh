#!/bin/bash
# round-2 GPU pass 1: tests, C4 bench, N3 same-process ncu traffic (staged vs fused), plane_fwd2d full capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gputests.txt 2>&1; tail -3 gpurun_out/gputests.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; tail -c 600 gpurun_out/bench_C4.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/n3_raw.csv python tools/n3_traffic.py run C3 C4 C5L C1 C2-N1024-H64-B1024 > gpurun_out/n3_run.log 2>&1
python tools/n3_traffic.py summarize gpurun_out/n3_raw.csv > gpurun_out/n3_traffic.json 2> gpurun_out/n3_sum.err; head -c 1500 gpurun_out/n3_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_fwd2d -s 1 -c 1 -o gpurun_out/fwd_C4 -f \
  python bench.py --steps 1 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_fwd.log 2>&1; tail -2 gpurun_out/ncu_fwd.log
