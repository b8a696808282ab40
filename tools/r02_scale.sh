#!/bin/bash
# bench.py at 1 / 2 / 4 GPUs through its own launcher (as the driver's
# scaling run) plus the reference arm; one box.
tag=${1:-r02scale}
out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
for n in 1 2 4; do
  timeout 900 python bench.py --gpus $n --steps ${STEPS:-10} --warmup 3 > $out/bench_n$n.jsonl 2> $out/bench_n$n.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference_n1.jsonl 2> $out/bench_reference.err
for f in $out/bench_n*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; p=d.get('parity_sampled') or {}; a=d.get('alt_split') or {}
    print('$f'.split('/')[-1], 'n', d['n_gpus'], 'value', d['value'], 'e2e', round((d.get('e2e') or {}).get('value') or 0,1), 'share', r['gemm_share_of_step'], 'frac', r['frac'], 'mhz', d['clocks']['sm_mhz'], 'parity', p.get('relfro_vs_reference'), p.get('pass'), 'alt', a.get('value'), (a.get('parity_sampled') or {}).get('pass'))"; done
head -c 400 $out/bench_reference_n1.jsonl; echo
