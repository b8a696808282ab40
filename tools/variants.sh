#!/bin/bash
# Sweep GEMM tuning knobs: plain timing (N=16384, 32768) then ncu DRAM bytes (N=16384).
mkdir -p gpurun_out
declare -a V=("DM_L2_POLICY=1" "DM_L2_POLICY=0" "DM_L2_POLICY=2" "DM_GROUP_M=16" "DM_GROUP_M=4" "DM_LOCKSTEP=16" "DM_LOCKSTEP=64" "DM_LOCKSTEP=16 DM_L2_POLICY=0" "DM_LOCKSTEP=8 DM_GROUP_M=16")
for v in "${V[@]}"; do
  echo "== $v" >> gpurun_out/var_time.log
  env $v timeout 120 python tools/probe_gemm.py 16384 32768 >> gpurun_out/var_time.log 2>&1
done
for v in "${V[@]}"; do
  echo "== $v" >> gpurun_out/var_ncu.log
  env $v timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tf32x3 -s 1 -c 1 python tools/probe_gemm.py 16384 2>&1 | grep -E "dram__bytes|gpu__time|hit_rate" >> gpurun_out/var_ncu.log
done
