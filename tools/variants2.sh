#!/bin/bash
mkdir -p gpurun_out
declare -a V=("DM_GROUP_M=8" "DM_GROUP_M=16" "DM_LOCKSTEP=32" "DM_GROUP_M=16 DM_LOCKSTEP=32" "DM_GROUP_M=32" "DM_GROUP_M=12 DM_LOCKSTEP=32")
for rep in 1 2; do
for v in "${V[@]}"; do
  echo "== rep$rep $v" >> gpurun_out/var2_time.log
  env $v timeout 120 python tools/probe_gemm.py 32768 >> gpurun_out/var2_time.log 2>&1
done
done
for v in "${V[@]}"; do
  echo "== $v" >> gpurun_out/var2_ncu.log
  env $v timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tf32x3 -s 1 -c 1 python tools/probe_gemm.py 32768 2>&1 | grep -E "dram__bytes|gpu__time|hit_rate" >> gpurun_out/var2_ncu.log
done
