#!/bin/bash
# owner-split (presplit) GEMM: GPU tests on 4 GPUs, timelines and benches vs the consumer split
out=gpurun_out/r02_presplit; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_presplit.py tests/test_gpu_spmd.py -x -q > $out/pytest.log 2>&1; tail -5 $out/pytest.log
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
mkdir -p $out/tr
TRACE_DIR=$out/tr timeout 600 bash -c "$(declare -f tr); tr 4 29621 tools/trace_gemm.py" > $out/trace_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/trace_n4.log | head -40
timeout 900 bash -c "$(declare -f tr); tr 4 29622 tools/spmd_probe.py - DM_PRESPLIT_PANEL=16384 DM_PRESPLIT_PANEL=4096 DM_PRESPLIT=0" > $out/probe_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n4.log | tail -8
timeout 600 bash -c "$(declare -f tr); tr 2 29623 tools/spmd_probe.py - DM_PRESPLIT=0" > $out/probe_n2.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n2.log | tail -4
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q > $out/pytest_pipeline.log 2>&1; tail -3 $out/pytest_pipeline.log
