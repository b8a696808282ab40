#!/bin/bash
# Profiles for round $1 (1 GPU): launch list of the bench command and one
# ncu --set full capture of the N=32768 GEMM launch (each only after the same
# command exited 0 without ncu).
r=${1:-r01}
out=gpurun_out/ncu_$r
mkdir -p $out
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$cmd > $out/plain.jsonl 2> $out/plain.err || { tail -n 20 $out/plain.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1
python tools/ncu_summarize.py launches $out/launches.csv $out/launch_shares.txt
ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 1 -c 1 -o $out/gemm_full $cmd > $out/ncu_full.log 2>&1
python tools/ncu_summarize.py full $out/gemm_full.ncu-rep $out/ncu_gemm_summary.json 32768 "$cmd" \
  "ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 1 -c 1"
cat $out/plain.jsonl | head -c 400; echo
