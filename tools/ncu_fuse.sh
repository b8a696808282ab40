#!/bin/bash
# ncu of one panel GEMM with and without the fused split of the next panel (1 GPU).
out=gpurun_out/ncu_fuse
mkdir -p $out
export TRACE_N=16384 DM_PANEL_LOCAL=1
for f in 1 0; do
  DM_FUSE_SPLIT=$f TRACE_DIR=/tmp timeout 300 python tools/trace_gemm.py > $out/plain_$f.log 2>&1 || exit 1
  DM_FUSE_SPLIT=$f TRACE_DIR=/tmp timeout 900 ncu --set full --clock-control none -k regex:tf32x3_gemm_kernel --launch-skip 2 --launch-count 1 \
     -o $out/gemm_fuse$f python tools/trace_gemm.py > $out/ncu_$f.log 2>&1
done
cat $out/plain_1.log $out/plain_0.log
