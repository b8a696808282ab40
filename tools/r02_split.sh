#!/bin/bash
# f16x2 transposing split: swizzled 16-B-store kernel vs the tf32-shaped one (DM_SPLIT_TRANS16=0)
out=gpurun_out/r02_split; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_local_gemm.py -q -k "split_kernels_agree or shapes" > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for t in 1 0; do
  DM_SPLIT_TRANS16=$t PROBE_REPS=3 timeout 600 python tools/panel_probe.py - > $out/n1_t$t.log 2>&1; cat $out/n1_t$t.log
done
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-alt"
for t in 1 0; do
  DM_SPLIT_TRANS16=$t ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:split -c 12 --csv --log-file $out/split_t$t.csv $cmd > $out/ncu_t$t.log 2>&1
  python tools/ncu_summarize.py launches $out/split_t$t.csv $out/split_t$t.txt
done
