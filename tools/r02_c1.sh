#!/bin/bash
out=gpurun_out/r02_c1; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
for f in 64 0; do
  DM_F16X2_MIN_GFLOP=$f timeout 300 python tools/config1_diag.py > $out/c1_f$f.log 2>&1
  DM_F16X2_MIN_GFLOP=$f C1_TRACE=1 C1_REPS=20 timeout 300 python tools/config1_diag.py > $out/c1_trace_f$f.log 2>&1
  echo "== DM_F16X2_MIN_GFLOP=$f"; cat $out/c1_f$f.log $out/c1_trace_f$f.log | grep -v gemm_mode
done
DM_F16X2_MIN_GFLOP=0 HOST_PROF_REPS=100 timeout 300 python tools/host_prof.py > $out/host_prof_f0.log 2>&1; head -5 $out/host_prof_f0.log
HOST_PROF_REPS=100 timeout 300 python tools/host_prof.py > $out/host_prof_f64.log 2>&1; head -5 $out/host_prof_f64.log
