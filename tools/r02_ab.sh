#!/bin/bash
# GPU suite + N=1 bench A/B of an environment knob (quick bench: no e2e/alt/cpu)
tag=${1:-r02c}; knob=${2:-DM_MN_MAJOR}
out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for v in 1 0 1 0; do
  env $knob=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-alt --no-cpu >> $out/ab_$v.jsonl 2>> $out/ab.err
done
tail -n 12 $out/pytest_gpu.log
for v in 1 0; do python -c "
import json
for l in open('$out/ab_$v.jsonl'):
    d=json.loads(l); r=d['roofline']; print('$knob=$v', d['value'], r['achieved'], r['gemm_share_of_step'], d['clocks']['sm_mhz'])"; done
