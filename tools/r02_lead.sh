#!/bin/bash
# f16x2, standalone splits (new default): lead-panel ramp and panel width at 2/4 GPUs
out=gpurun_out/r02_lead; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
run() { tag=$1; n=$2; shift 2; env "$@" timeout 600 python bench.py --gpus $n --steps 10 --warmup 3 --no-alt --no-e2e --no-cpu > $out/b_${tag}.jsonl 2> $out/b_${tag}.err;
  python -c "
import json
for l in open('$out/b_${tag}.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('%-28s n=%d %9.1f TFLOP/s  kernel %6.1f share %.3f  clk %s' % ('$tag', d['n_gpus'], d['value'], r['achieved'], r['gemm_share_of_step'], d['clocks']['sm_mhz']))"; }
run n4_base 4 X=1
run n4_lead2048 4 DM_LEAD_PANEL_K=2048
run n4_lead4096 4 DM_LEAD_PANEL_K=4096
run n4_panel16384 4 DM_PANEL_K=16384
run n2_base 2 X=1
run n2_panel8192 2 DM_PANEL_K=8192
run n2_lead2048 2 DM_LEAD_PANEL_K=2048
run n1_base 1 X=1
