#!/bin/bash
# global row scales (presplit phase 2) tests; e2e breakdown at 4 GPUs with / without presplit
out=gpurun_out/r02_e2e; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_presplit.py tests/test_gpu_spmd.py -q -x > $out/pytest.log 2>&1; tail -3 $out/pytest.log
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 bash -c "$(declare -f tr); tr 4 29651 tools/spmd_probe.py - DM_PRESPLIT_PANEL=8192" > $out/probe_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n4.log | tail -4
for ps in 1 0; do
  DM_PRESPLIT=$ps timeout 900 bash -c "$(declare -f tr); tr 4 2966$ps tools/e2e_probe.py" > $out/e2e_n4_ps$ps.log 2>&1
  grep 'rank 0/' $out/e2e_n4_ps$ps.log
done
