#!/bin/bash
out=gpurun_out/r02_async; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 600 bash -c "$(declare -f tr); tr 4 29611 tools/spmd_probe.py - DM_PANEL_K=16384" > $out/n4.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/n4.log | tail -6
timeout 600 bash -c "$(declare -f tr); tr 2 29612 tools/spmd_probe.py -" > $out/n2.log 2>&1
grep -v "^\*\|OMP\|NCCL\|W1" $out/n2.log | tail -4
