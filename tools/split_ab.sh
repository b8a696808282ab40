#!/bin/bash
# Does the split kernel co-run with the GEMM?  Device timelines at 1 GPU with
# forced K panels, for split blocks of 2/4/8 warps.
tag=${1:-split}
out=gpurun_out/$tag
mkdir -p $out
for w in 2 4 8; do
  DM_PANEL_LOCAL=1 DM_SPLIT_WARPS=$w TRACE_DIR=$out timeout 300 python tools/trace_gemm.py > $out/trace_n1_w$w.log 2>&1
done
tail -n 12 $out/trace_n1_w*.log
