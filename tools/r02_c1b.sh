#!/bin/bash
# config 1: split-K / CTA group / split scheme of the per-worker 1024x1024x2048 GEMM
out=gpurun_out/r02_c1b; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
for v in "X=1" "DM_KSPLIT=1" "DM_KSPLIT=4" "DM_CTA_GROUP=2" "DM_CTA_GROUP=2 DM_KSPLIT=1" "DM_F16X2_MIN_GFLOP=0" "DM_F16X2_MIN_GFLOP=0 DM_KSPLIT=1"; do
  env $v C1_REPS=300 timeout 300 python tools/config1_diag.py > $out/c1.log 2>&1
  echo "$v: $(grep sync $out/c1.log)"
done
env C1_TRACE=1 C1_REPS=20 DM_KSPLIT=1 timeout 300 python tools/config1_diag.py > $out/c1_trace_k1.log 2>&1; grep ' w0 ' $out/c1_trace_k1.log
