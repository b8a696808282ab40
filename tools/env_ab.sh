#!/bin/bash
# A/B of one env knob at several rank counts: timeline (first setting) + bench.
# usage: bash tools/env_ab.sh <tag> <VAR> "<values>" "<rank counts>"
tag=$1; var=$2; vals=$3; ns=$4
out=gpurun_out/$tag
mkdir -p $out
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
first=${vals%% *}
maxn=${ns##* }
if [ "$maxn" -gt 1 ]; then
  env $var=$first TRACE_DIR=$out timeout 300 bash -c "$(declare -f tr); tr $maxn 29504 tools/trace_gemm.py" > $out/trace.log 2>&1
else
  env $var=$first TRACE_DIR=$out timeout 300 python tools/trace_gemm.py > $out/trace.log 2>&1
fi
for v in $vals; do
  for n in $ns; do
    if [ "$n" -gt 1 ]; then
      env $var=$v timeout 400 bash -c "$(declare -f tr); tr $n 2960$n bench.py --gpus $n" > $out/bench_n${n}_$v.jsonl 2> $out/bench_n${n}_$v.err
    else
      env $var=$v timeout 400 python bench.py > $out/bench_n${n}_$v.jsonl 2> $out/bench_n${n}_$v.err
    fi
  done
done
grep -v "^\s*$" $out/trace.log | grep -v OMP | grep -v '\*\*\*' | head -60
for f in $out/bench_*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; print('$f'.split('/')[-1], d['value'], round(d['e2e']['value'],1), r['gemm_share_of_step'], r['frac'], d['clocks']['sm_mhz'])"; done
