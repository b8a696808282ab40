#!/bin/bash
# f16x2 at 2/4 GPUs: fused split (default) vs standalone split kernels (DM_FUSE_SPLIT=0)
out=gpurun_out/r02_fuse; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for fs in 0 1; do
  mkdir -p $out/fs$fs
  DM_FUSE_SPLIT=$fs TRACE_DIR=$out/fs$fs timeout 600 bash -c "$(declare -f tr); tr 4 29604 tools/trace_gemm.py" > $out/trace_n4_fs$fs.log 2>&1
  echo "== fuse=$fs"; grep -v "^\*\|OMP\|NCCL" $out/trace_n4_fs$fs.log | head -40
done
for n in 4 2; do
  DM_FUSE_SPLIT=0 timeout 900 python bench.py --gpus $n --steps 10 --warmup 3 --no-alt --no-e2e > $out/bench_n${n}_fs0.jsonl 2> $out/bench_n${n}_fs0.err
done
for f in $out/bench_n*.jsonl; do python -c "
import json
for l in open('$f'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); r=d['roofline']; p=d.get('parity_sampled') or {}
    print('$f'.split('/')[-1], d['n_gpus'], d['value'], r['achieved'], r['gemm_share_of_step'], r['frac'], d['clocks']['sm_mhz'], p.get('relfro_vs_reference'), p.get('pass'))"; done
