#!/bin/bash
# A/B of copy-engine peer pulls (DM_PULL_CE) at 2 and 4 ranks: timeline + bench.
tag=${1:-ab}
out=gpurun_out/$tag
mkdir -p $out
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
TRACE_DIR=$out timeout 300 bash -c "$(declare -f tr); tr 4 29504 tools/trace_gemm.py" > $out/trace_n4.log 2>&1
for ce in 1 0; do
  for n in 4 2; do
    DM_PULL_CE=$ce timeout 400 bash -c "$(declare -f tr); tr $n 2960$n bench.py --gpus $n" > $out/bench_n${n}_ce$ce.jsonl 2> $out/bench_n${n}_ce$ce.err
  done
done
head -40 $out/trace_n4.log
for f in $out/bench_*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); print(d['value'], d['e2e']['value'], d['roofline']['gemm_share_of_step'])"; done
