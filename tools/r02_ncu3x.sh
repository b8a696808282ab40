#!/bin/bash
# 1-GPU evidence: ncu of the 3xTF32 N=32768 GEMM (launch list + one --set full
# capture), host topology, compute-sanitizer over tools/sanitize.py.
out=gpurun_out/r02_ncu3x; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
{ nvidia-smi topo -m; lscpu; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c; nvidia-smi -q | grep -i -A2 "bus id\|numa"; free -g; } > $out/topo.txt 2>&1
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-alt --gemm-mode 3xtf32"
timeout 300 $cmd > $out/plain.jsonl 2> $out/plain.err || { tail -n 20 $out/plain.err; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1
python tools/ncu_summarize.py launches $out/launches.csv $out/launch_shares.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 1 -c 1 -o $out/gemm_full $cmd > $out/ncu_full.log 2>&1
python tools/ncu_summarize.py full $out/gemm_full.ncu-rep $out/ncu_gemm_summary.json 32768 "$cmd" \
  "ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 1 -c 1"
head -c 600 $out/plain.jsonl; echo
cat $out/launch_shares.txt | head -20
bash tools/sanitize.sh r02_sanitize
