#!/bin/bash
out=gpurun_out/r02_multi2; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/panel_probe.py - DM_PANEL_LOCAL=4096,DM_PANEL_GROWTH=2,DM_FUSE_SPLIT=2 \
   DM_PANEL_LOCAL=2048,DM_PANEL_GROWTH=3,DM_FUSE_SPLIT=2 DM_PANEL_LOCAL=1024,DM_PANEL_GROWTH=3,DM_FUSE_SPLIT=2 > $out/panel_probe.log 2>&1
cat $out/panel_probe.log
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
TRACE_DIR=$out timeout 600 bash -c "$(declare -f tr); tr 4 29604 tools/trace_gemm.py" > $out/trace_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL" $out/trace_n4.log | head -40
for n in 1 2 4; do
  timeout 900 python bench.py --gpus $n --steps 10 --warmup 3 > $out/bench_n$n.jsonl 2> $out/bench_n$n.err
done
for f in $out/bench_n*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; p=d.get('parity_sampled') or {}; a=d.get('alt_split') or {}
    print('$f'.split('/')[-1], d['n_gpus'], d['value'], round((d.get('e2e') or {}).get('value') or 0,1), r['achieved'], r['gemm_share_of_step'], r['frac'], d['clocks']['sm_mhz'], p.get('relfro_vs_reference'), p.get('pass'), a.get('value'), (a.get('parity_sampled') or {}).get('pass'))"; done
