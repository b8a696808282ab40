"""Host-side cost of the command path (DM_HOST_PROF=1 phase timers) for the
small configurations: BASELINE config 1 (2048^3, 2x2, P=4) and the FC
forward / backward / dW (9216->4096, batch 256) -- LOCAL mode over the
visible GPUs; prints wall us per call and the phase breakdown at exit."""
import os
import sys
import time

os.environ.setdefault("DM_HOST_PROF", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402


def wall(s, fn, reps=int(os.environ.get("HOST_PROF_REPS", "50"))):
    for _ in range(5):
        fn()
    s.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    s.barrier()
    return (time.perf_counter() - t0) / reps * 1e6


only = sys.argv[1] if len(sys.argv) > 1 else "all"
ndev = torch.cuda.device_count()
P = 4
devs = [w % ndev for w in range(P)]
with dm.Session(dm.Config(worker_count=P, root_seed=42, devices=devs)) as s:
    n = 2048
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    if only in ("all", "config1"):
        print(f"config1 sync : {wall(s, lambda: s.general_gemm(1.0, a, b, 0.0, c)):.1f} us/call", flush=True)
    if only in ("all", "config1async"):
        s.set_async(True)
        print(f"config1 async: {wall(s, lambda: s.general_gemm(1.0, a, b, 0.0, c)):.1f} us/call", flush=True)
        s.set_async(False)
with dm.Session(dm.Config(worker_count=P, root_seed=3, devices=devs)) as s:
    fin, fout, batch = 9216, 4096, 256
    strip = batch // P
    W = s.create_matrix(dm.make_layout(0, fin, fout, fin // P, fout, P), fill=dm.FillKind.SeededRandom)
    X = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, P), fill=dm.FillKind.SeededRandom)
    Y = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, P))
    dY = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, P), fill=dm.FillKind.SeededRandom)
    dX = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, P))
    dW = s.create_matrix(dm.make_layout(0, fin, fout, fin // P, fout, P))
    if only in ("all", "fwd", "bwd"):
        print(f"fc fwd cached: {wall(s, lambda: s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)):.1f} us/call")
    if only in ("all", "bwd"):
        print(f"fc bwd       : {wall(s, lambda: s.cached_backward_gemm(W, dY, dX)):.1f} us/call")
    if only in ("all", "dw"):
        print(f"fc dW        : {wall(s, lambda: s.general_gemm(1.0, X, dY, 0.0, dW, False, True)):.1f} us/call",
              flush=True)
