#!/bin/bash
# TMEM chunk (flush) width for f16x2 at N=32768: speed and accuracy (bench parity vs the reference / float64)
out=gpurun_out/r02_flush; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
for f in 256 512 1024 256; do
  DM_FLUSH_K=$f timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-alt > $out/b_f$f.jsonl 2> $out/b_f$f.err
  python -c "
import json
for l in open('$out/b_f$f.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; p=d['parity_sampled']
        print('flush $f', d['value'], 'kernel', r['achieved'], 'clk', d['clocks']['sm_mhz'], 'relfro_ref', p['relfro_vs_reference'], 'vs_fp64', p['relfro_vs_fp64'])"
done
