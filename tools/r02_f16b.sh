#!/bin/bash
# f16x2 as the default: GPU suite, bench N=1, ncu of the f16x2 GEMM launch.
out=gpurun_out/r02_f16b; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -n 15 $out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench_n1.jsonl 2> $out/bench_n1.err
python -c "
import json
d=json.loads([l for l in open('$out/bench_n1.jsonl') if l.startswith('{')][0]); r=d['roofline']; p=d['parity_sampled']; a=d['alt_split']
print('n1', d['value'], d['e2e']['value'], r['achieved'], r['frac'], r['gemm_share_of_step'], d['clocks'], p['relfro_vs_reference'], p['relfro_vs_fp64'], a['value'], a['parity_sampled'])"
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-alt"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1
python tools/ncu_summarize.py launches $out/launches.csv $out/launch_shares.txt; cat $out/launch_shares.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 1 -c 1 -o $out/gemm_full $cmd > $out/ncu_full.log 2>&1
python tools/ncu_summarize.py full $out/gemm_full.ncu-rep $out/ncu_gemm_summary.json 32768 "$cmd" \
  "ncu --set full --clock-control none --import-source on -k regex:tf32x3 -s 1 -c 1"
timeout 900 python tools/f16x2_probe.py accuracy > $out/probe_acc.log 2>&1; tail -30 $out/probe_acc.log
