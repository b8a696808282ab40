#!/bin/bash
# panel cost on one GPU; config-1 timeline / host profile (f16x2)
out=gpurun_out/r02_small; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/beta_probe.py 16384 16384 32768 > $out/beta_16k.log 2>&1; cat $out/beta_16k.log
timeout 600 python tools/beta_probe.py 32768 16384 32768 > $out/beta_32k.log 2>&1; cat $out/beta_32k.log
timeout 300 python tools/config1_diag.py > $out/config1.log 2>&1
C1_TRACE=1 C1_REPS=20 timeout 300 python tools/config1_diag.py > $out/config1_trace.log 2>&1
HOST_PROF_REPS=200 timeout 300 python tools/host_prof.py config1 > $out/host_prof_c1.log 2>&1
cat $out/config1.log $out/config1_trace.log $out/host_prof_c1.log
