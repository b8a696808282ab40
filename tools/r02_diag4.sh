#!/bin/bash
# 4-GPU diagnostics: config-1 wall/trace, host phase profile, ncu of a P=4
# per-rank fused-split GEMM launch (LOCAL session, --devices 0).
out=gpurun_out/r02_diag4; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
nproc > $out/host.txt; nvidia-smi topo -m >> $out/host.txt 2>&1
timeout 300 python tools/config1_diag.py > $out/config1.log 2>&1
C1_TRACE=1 C1_REPS=20 timeout 300 python tools/config1_diag.py > $out/config1_trace.log 2>&1
HOST_PROF_REPS=200 timeout 300 python tools/host_prof.py > $out/host_prof.log 2>&1
C1_REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/config1_launches.csv python tools/config1_diag.py > $out/config1_ncu.log 2>&1
timeout 300 python tools/ncu_p4.py > $out/p4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --devices 0 -k regex:tf32x3_gemm_kernel -s 5 -c 1 \
   -o $out/p4_gemm_fused python tools/ncu_p4.py > $out/p4_ncu.log 2>&1
cat $out/config1.log $out/config1_trace.log; tail -30 $out/host_prof.log; cat $out/p4_plain.log; tail -5 $out/p4_ncu.log
