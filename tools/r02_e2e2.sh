#!/bin/bash
out=gpurun_out/r02_e2e2; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python tools/h2d_probe.py 1 > $out/h2d.log 2>&1; cat $out/h2d.log
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 bash -c "$(declare -f tr); tr 4 29671 tools/e2e_probe.py" > $out/e2e_n4.log 2>&1
grep -o 'rank 0/4[^r]*' $out/e2e_n4.log
timeout 1200 python -m pytest tests/test_gpu_spmd.py tests/test_gpu_session.py -q -x > $out/pytest.log 2>&1; tail -3 $out/pytest.log
timeout 900 python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --no-alt > $out/bench_n4.jsonl 2> $out/bench_n4.err
python -c "
import json
for l in open('$out/bench_n4.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('n4 value', d['value'], 'e2e', d['e2e'])"
