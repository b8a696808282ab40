#!/bin/bash
out=gpurun_out/r02_c5; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/bench_configs.py --configs 5 > $out/c5.jsonl 2>&1; cut -c1-200 $out/c5.jsonl
DM_PRESPLIT=0 timeout 600 python tools/bench_configs.py --configs 5 > $out/c5_ps0.jsonl 2>&1; cut -c1-200 $out/c5_ps0.jsonl
timeout 900 python -m pytest tests/test_gpu_presplit.py -q -x > $out/pytest.log 2>&1; tail -2 $out/pytest.log
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
PROBE_N=16384 timeout 900 bash -c "$(declare -f tr); tr 4 29681 tools/spmd_probe.py - DM_PRESPLIT=0" > $out/probe_n4_16k.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n4_16k.log | tail -4
