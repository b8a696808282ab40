#!/bin/bash
# presplit tests + SPMD suite; lead panels at 4 GPUs; small configs after the auto rule
out=gpurun_out/r02_mid; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_presplit.py tests/test_gpu_spmd.py tests/test_gpu_pipeline.py -q > $out/pytest.log 2>&1; tail -4 $out/pytest.log
timeout 300 python tools/config1_diag.py > $out/config1.log 2>&1
C1_TRACE=1 C1_REPS=20 timeout 300 python tools/config1_diag.py > $out/config1_trace.log 2>&1
cat $out/config1.log $out/config1_trace.log
timeout 900 python tools/bench_configs.py > $out/configs.jsonl 2> $out/configs.err; cut -c1-400 $out/configs.jsonl
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 1200 bash -c "$(declare -f tr); tr 4 29641 tools/spmd_probe.py - DM_PRESPLIT_LEAD=2048 DM_PRESPLIT_LEAD=4096 DM_PRESPLIT_PANEL=8192" > $out/probe_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n4.log | tail -8
