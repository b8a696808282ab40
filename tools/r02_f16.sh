#!/bin/bash
out=gpurun_out/r02_f16; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/f16x2_probe.py transposes session > $out/probe_paths.log 2>&1; echo "rc=$?" >> $out/probe_paths.log
cat $out/probe_paths.log
timeout 600 python tools/f16x2_probe.py throughput > $out/probe_tput.log 2>&1; echo "rc=$?" >> $out/probe_tput.log
cat $out/probe_tput.log
timeout 900 python tools/f16x2_probe.py accuracy > $out/probe_acc.log 2>&1; echo "rc=$?" >> $out/probe_acc.log
cat $out/probe_acc.log
timeout 600 python -m pytest tests/test_gpu_hygiene.py -q -m gpu > $out/hygiene.log 2>&1; tail -3 $out/hygiene.log
