"""Config 1 (2048^3, 2x2 checkerboard, P=4 over the visible GPUs) diagnostics:
wall time per synchronous / asynchronous call, and with DM_TRACE set (graphs
off) the device timeline of one call per worker."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

n = int(os.environ.get("C1_N", "2048"))
P = 4
ndev = torch.cuda.device_count()
devs = [w % ndev for w in range(P)]
trace = os.environ.get("C1_TRACE", "0") == "1"
path = os.path.join(tempfile.gettempdir(), "dm_c1_trace.jsonl")
if trace:
    if os.path.exists(path):
        os.remove(path)
    os.environ["DM_TRACE"] = path


def wall(s, fn, reps=int(os.environ.get("C1_REPS", "200"))):
    for _ in range(5):
        fn()
    s.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    s.barrier()
    return (time.perf_counter() - t0) / reps * 1e6


with dm.Session(dm.Config(worker_count=P, root_seed=42, devices=devs)) as s:
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    print(f"N={n} devices={devs} gemm_mode={s.gemm_mode()}")
    print(f"sync  : {wall(s, lambda: s.general_gemm(1.0, a, b, 0.0, c)):.1f} us/call", flush=True)
    s.set_async(True)
    print(f"async : {wall(s, lambda: s.general_gemm(1.0, a, b, 0.0, c)):.1f} us/call", flush=True)
    s.set_async(False)
if trace:
    recs = [json.loads(line) for line in open(path)]
    last = max(r["cmd"] for r in recs)
    for r in recs:
        if r["cmd"] == last:
            print(f"  w{r.get('worker', '?')} {r['what']:11s} panel {r['panel']:2d}  {r['t0_ms'] * 1e3:8.1f} -> "
                  f"{r['t1_ms'] * 1e3:8.1f} us  bytes={r['bytes'] / 2**20:7.2f} MiB  flops={r['flops']:.3g}")
