#!/bin/bash
# 1-GPU check: GPU tests + forced-panel timeline + bench.
tag=${1:-q1}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
DM_PANEL_LOCAL=1 TRACE_DIR=$out timeout 300 python tools/trace_gemm.py > $out/trace_n1_panels.log 2>&1
timeout 300 python bench.py > $out/bench_n1.jsonl 2> $out/bench_n1.err
DM_PANEL_LOCAL=1 timeout 300 python bench.py > $out/bench_n1_panels.jsonl 2> $out/bench_n1_panels.err
tail -n 15 $out/pytest_gpu.log; cat $out/trace_n1_panels.log
for f in $out/bench_*.jsonl; do echo $f; python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['value'], d.get('e2e',{}).get('value'), d['roofline']['gemm_share_of_step'], d['roofline']['frac'])"; done
