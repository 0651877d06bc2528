#!/bin/bash
# ncu of the C1 fused 1D kernel (PDL default and off: the launch list must see it either way)
mkdir -p gpurun_out
for p in 1 0; do
TFNO_PDL=$p timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused1d" -s 1 -c 1 \
  -o gpurun_out/prof_C1_pdl$p -f python bench.py --workload C1 --steps 2 --warmup 2 --graph off --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_C1_pdl$p.log 2>&1
tail -2 gpurun_out/ncu_C1_pdl$p.log
done
TFNO_PDL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1
grep -c '"' gpurun_out/launches_smoke.csv; grep -o 'tfno::[a-z0-9_]*' gpurun_out/launches_smoke.csv | sort | uniq -c
