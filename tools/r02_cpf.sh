#!/bin/bash
# C prefetch before beta=1 epilogues (panels after the first) x presplit panel width
out=gpurun_out/r02_cpf; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_presplit.py -x -q > $out/pytest.log 2>&1; tail -2 $out/pytest.log
PROBE_REPS=3 timeout 600 python tools/panel_probe.py - DM_C_PREFETCH=0 > $out/n1.log 2>&1; cat $out/n1.log
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 1200 bash -c "$(declare -f tr); tr 4 29631 tools/spmd_probe.py DM_C_PREFETCH=0 DM_C_PREFETCH=1 DM_C_PREFETCH=2 DM_C_PREFETCH=0,DM_PRESPLIT_PANEL=16384 DM_C_PREFETCH=1,DM_PRESPLIT_PANEL=16384 DM_C_PREFETCH=1,DM_PRESPLIT=0" > $out/probe_n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n4.log | tail -12
timeout 900 bash -c "$(declare -f tr); tr 2 29632 tools/spmd_probe.py DM_C_PREFETCH=0,DM_PRESPLIT_PANEL=16384 DM_C_PREFETCH=1,DM_PRESPLIT_PANEL=16384 DM_C_PREFETCH=1" > $out/probe_n2.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/probe_n2.log | tail -6
