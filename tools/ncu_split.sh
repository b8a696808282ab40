#!/bin/bash
# ncu of the standalone split kernels (first panel of an N=16384 GEMM, 1 GPU).
out=gpurun_out/ncu_split
mkdir -p $out
export TRACE_N=16384
TRACE_DIR=/tmp timeout 300 python tools/trace_gemm.py > $out/plain.log 2>&1 || exit 1
TRACE_DIR=/tmp timeout 900 ncu --set full --clock-control none -k regex:split_ --launch-count 2 \
   -o $out/split python tools/trace_gemm.py > $out/ncu.log 2>&1
ncu -i $out/split.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__grid_size > $out/split_summary.csv
cat $out/plain.log; cat $out/split_summary.csv
