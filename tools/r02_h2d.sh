#!/bin/bash
out=gpurun_out/r02_h2d; mkdir -p $out
timeout 300 python tools/h2d_probe.py 1 > $out/h2d.log 2>&1; cat $out/h2d.log
nproc >> $out/h2d.log; free -g >> $out/h2d.log 2>&1; tail -4 $out/h2d.log
