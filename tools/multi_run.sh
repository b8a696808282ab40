#!/bin/bash
# Multi-GPU check on one box: GPU tests, device timelines at 2/4 ranks, bench at 1/2/4.
# usage (gpurun --gpus 4): bash tools/multi_run.sh <tag>
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for n in 2 4; do
  TRACE_DIR=$out timeout 300 bash -c "$(declare -f tr); tr $n 2950$n tools/trace_gemm.py" > $out/trace_n$n.log 2>&1
done
timeout 300 python bench.py > $out/bench_n1.jsonl 2> $out/bench_n1.err
for n in 2 4; do
  timeout 400 bash -c "$(declare -f tr); tr $n 2960$n bench.py --gpus $n" > $out/bench_n$n.jsonl 2> $out/bench_n$n.err
done
tail -n 3 $out/pytest_gpu.log; cat $out/trace_n4.log | head -40; cat $out/bench_n*.jsonl
