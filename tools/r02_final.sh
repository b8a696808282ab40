#!/bin/bash
# End-of-round evidence on one 4-GPU box: GPU suite, bench 1/2/4 (+reference
# arm), BASELINE configs, launch list + ncu of the N=1 bench GEMM, ncu of one
# rank's presplit GEMM launch at 4 GPUs.
tag=${1:-r02final}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; tail $out/build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -n 4 $out/pytest_gpu.log
for n in 1 2 4; do
  timeout 900 python bench.py --gpus $n --steps 10 --warmup 3 > $out/bench_n$n.jsonl 2> $out/bench_n$n.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference_n1.jsonl 2> $out/bench_reference.err
timeout 900 python tools/bench_configs.py > $out/configs.jsonl 2> $out/configs.err
for f in $out/bench_n*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; p=d.get('parity_sampled') or {}; a=d.get('alt_split') or {}
    print('$f'.split('/')[-1], 'n', d['n_gpus'], 'value', d['value'], 'e2e', round((d.get('e2e') or {}).get('value') or 0,1), 'kern', r['achieved'], 'share', r['gemm_share_of_step'], 'frac', r['frac'], 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'parity', p.get('relfro_vs_reference'), p.get('pass'), 'alt', a.get('value'), (a.get('parity_sampled') or {}).get('pass'))"; done
head -c 300 $out/bench_reference_n1.jsonl; echo
cut -c1-300 $out/configs.jsonl
# profiles (each command ran clean above / here first)
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-alt"
$cmd > $out/plain_n1.jsonl 2> $out/plain_n1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n1.csv $cmd > $out/ncu_launches_n1.log 2>&1
python tools/ncu_summarize.py launches $out/launches_n1.csv $out/launch_shares_n1.txt
P4_CHECK=1 timeout 900 python tools/ncu_p4_presplit.py > $out/p4_plain.log 2>&1 && \
P4_CHECK=0 timeout 1200 ncu --set full --clock-control none --import-source on --devices 0 -k regex:tf32x3_gemm_kernel -s 2 -c 1 \
   -o $out/p4_gemm_presplit python tools/ncu_p4_presplit.py > $out/p4_ncu.log 2>&1
python tools/ncu_summarize.py full $out/p4_gemm_presplit.ncu-rep $out/ncu_gemm_summary_f16x2_p4.json 32768 \
  "python tools/ncu_p4_presplit.py (LOCAL session, 4 GPUs, 2x2)" \
  "ncu --set full --clock-control none --import-source on --devices 0 -k regex:tf32x3_gemm_kernel -s 2 -c 1" > $out/p4_summary.log 2>&1
cat $out/p4_plain.log; tail -3 $out/p4_ncu.log; cat $out/launch_shares_n1.txt | head -8
