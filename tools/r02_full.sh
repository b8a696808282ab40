#!/bin/bash
# Round-2 milestone check on one box: GPU suite, bench at 1..N GPUs through
# bench.py's own launcher, reference arm, secondary BASELINE configs.
tag=${1:-r02full}
ngpu=${2:-4}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -n 3 $out/pytest_gpu.log
for n in 1 2 4 8; do
  [ "$n" -gt "$ngpu" ] && break
  timeout 900 python bench.py --gpus $n --steps 10 --warmup 3 > $out/bench_n$n.jsonl 2> $out/bench_n$n.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference_n1.jsonl 2> $out/bench_reference.err
[ "$ngpu" -ge 4 ] && timeout 900 python tools/bench_configs.py > $out/configs.jsonl 2> $out/configs.err
for f in $out/bench_n*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; p=d.get('parity_sampled') or {}; a=d.get('alt_split') or {}
    print('$f'.split('/')[-1], d['n_gpus'], d['value'], round((d.get('e2e') or {}).get('value') or 0,1), r['gemm_share_of_step'], r['frac'], r['frac_vs_3xtf32_roofline'], d['clocks']['sm_mhz'], p.get('relfro_vs_reference'), p.get('pass'), a.get('value'), (a.get('parity_sampled') or {}).get('pass'))"; done
head -c 400 $out/bench_reference_n1.jsonl; echo
cut -c1-300 $out/configs.jsonl 2>/dev/null
