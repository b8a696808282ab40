#!/bin/bash
# End-of-milestone measurement on one 4-GPU box: full GPU suite, bench at
# 1/2/4 GPUs, the reference arm, and the secondary BASELINE configs.
tag=${1:-final}
out=gpurun_out/$tag
mkdir -p $out
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 1200 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 400 python bench.py > $out/bench_n1.jsonl 2> $out/bench_n1.err
for n in 2 4; do
  timeout 500 bash -c "$(declare -f tr); tr $n 2970$n bench.py --gpus $n" > $out/bench_n$n.jsonl 2> $out/bench_n$n.err
done
timeout 400 python bench.py --impl reference > $out/bench_reference_n1.jsonl 2> $out/bench_reference_n1.err
timeout 900 python tools/bench_configs.py --ref > $out/configs_4gpu.jsonl 2> $out/configs.err
tail -n 3 $out/pytest_gpu.log
for f in $out/bench_n*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; print('$f'.split('/')[-1], d['value'], round(d['e2e']['value'],1), r['gemm_share_of_step'], r['frac'], d['clocks']['sm_mhz'])"; done
cat $out/bench_reference_n1.jsonl | head -c 600; echo
cat $out/configs_4gpu.jsonl
