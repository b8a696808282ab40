#!/bin/bash
# Round-2 GPU check: build, GPU suite, bench at 1 GPU and at N GPUs through
# bench.py's own launcher (no torchrun wrapper), reference arm.
tag=${1:-r02a}
ngpu=${2:-2}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
free -g > $out/free.txt 2>&1; nproc >> $out/free.txt
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench_n1.jsonl 2> $out/bench_n1.err
if [ "$ngpu" -gt 1 ]; then
  timeout 900 python bench.py --gpus $ngpu --steps 10 --warmup 3 > $out/bench_n$ngpu.jsonl 2> $out/bench_n$ngpu.err
fi
tail -n 5 $out/pytest_gpu.log
for f in $out/bench_n*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; p=d.get('parity_sampled') or {}; a=d.get('alt_split') or {}
    print('$f'.split('/')[-1], d['n_gpus'], d['value'], (d.get('e2e') or {}).get('value'), r['gemm_share_of_step'], r['frac'], r['frac_vs_3xtf32_roofline'], d['clocks']['sm_mhz'], p.get('relfro_vs_reference'), p.get('pass'), a.get('value'), (a.get('parity_sampled') or {}).get('pass'))"; done
