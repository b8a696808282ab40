#!/bin/bash
# final-code timelines at 2 / 4 GPUs; ncu of one rank's GEMM launch at 2 GPUs (bench roofline.traffic)
out=gpurun_out/r02_trace; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for n in 4 2; do
  mkdir -p $out/n$n
  TRACE_DIR=$out/n$n timeout 600 bash -c "$(declare -f tr); tr $n 2969$n tools/trace_gemm.py" > $out/trace_n$n.log 2>&1
  grep -v "^\*\|OMP\|NCCL\|W1" $out/trace_n$n.log | head -40
done
P4_WORKERS=2 P4_CHECK=1 timeout 900 python tools/ncu_p4_presplit.py > $out/p2_plain.log 2>&1 && \
P4_WORKERS=2 P4_CHECK=0 timeout 1200 ncu --set full --clock-control none --import-source on --devices 0 -k regex:tf32x3_gemm_kernel -s 2 -c 1 \
   -o $out/p2_gemm_presplit python tools/ncu_p4_presplit.py > $out/p2_ncu.log 2>&1
python tools/ncu_summarize.py full $out/p2_gemm_presplit.ncu-rep $out/ncu_gemm_summary_f16x2_p2.json 32768 \
  "P4_WORKERS=2 python tools/ncu_p4_presplit.py (LOCAL session, 2 GPUs, 1x2)" \
  "ncu --set full --clock-control none --import-source on --devices 0 -k regex:tf32x3_gemm_kernel -s 2 -c 1" > $out/p2_summary.log 2>&1
cat $out/p2_plain.log $out/p2_summary.log
