#!/bin/bash
# fused1d output-channel cluster (CN): parity + same-box A/B vs the unfused schedule
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused1d.py -q -m gpu -x > gpurun_out/t11.txt 2>&1; tail -3 gpurun_out/t11.txt
out=gpurun_out/ncluster_ab.txt; : > $out
for rep in 1 2; do for wl in C2-N1024-H128-B256 C2-N1024-H128-B1024 C2-N1024-H256-B64 C2-N1024-H256-B256 C2-N1024-H256-B1024; do for cn in 0 -1; do
  TFNO_FUSED1D_NCLUSTER=$cn timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-baselines --no-e2e --no-cpu 2>gpurun_out/b11.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl cn=$cn', d['ms_per_step'], d['schedule'])" >> $out
done; done; done
cat $out; tail -3 gpurun_out/b11.err
