#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py's
# small GEMM scenarios (one GPU).  Logs go to gpurun_out/<tag>/.
tag=${1:-sanitize}
out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/sanitize.py > $out/plain.log 2>&1; echo "plain rc=$?" >> $out/plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
    --kernel-name regex:'tf32x3|split' python tools/sanitize.py ${SAN_ARGS} > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/$tool.log
  tail -n 4 $out/$tool.log
done
tail -n 3 $out/plain.log
