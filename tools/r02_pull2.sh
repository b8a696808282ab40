#!/bin/bash
# presplit plane pulls on one vs two copy streams
out=gpurun_out/r02_pull2; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_presplit.py tests/test_gpu_spmd.py -q -x > $out/pytest.log 2>&1; tail -2 $out/pytest.log
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
mkdir -p $out/tr
TRACE_DIR=$out/tr timeout 600 bash -c "$(declare -f tr); tr 4 29701 tools/trace_gemm.py" > $out/trace_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/trace_n4.log | head -30
timeout 900 bash -c "$(declare -f tr); tr 4 29702 tools/spmd_probe.py DM_PULL_STREAMS=2 DM_PULL_STREAMS=1 DM_PULL_STREAMS=2" > $out/probe_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n4.log | grep sync
