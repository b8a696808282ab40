"""Per-call wall time of the FC commands in bench_configs' order (diagnostic):
forward without cache, cache fill, cached forward, cached backward, dW."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

ndev = torch.cuda.device_count()
P = 4
devs = [w % ndev for w in range(P)]
fin, fout, batch = 9216, 4096, 256
strip = batch // P


def calls(s, name, fn, n=8):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    print(f"{name:12s} " + " ".join(f"{t:8.1f}" for t in ts), flush=True)


with dm.Session(dm.Config(worker_count=P, root_seed=3, devices=devs)) as s:
    W = s.create_matrix(dm.make_layout(0, fin, fout, fin // P, fout, P), fill=dm.FillKind.SeededRandom)
    X = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, P), fill=dm.FillKind.SeededRandom)
    Y = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, P))
    dY = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, P), fill=dm.FillKind.SeededRandom)
    dX = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, P))
    dW = s.create_matrix(dm.make_layout(0, fin, fout, fin // P, fout, P))
    if len(sys.argv) > 1 and sys.argv[1] == "pull":
        calls(s, "fwd pull", lambda: s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, False))
    calls(s, "fwd cache", lambda: s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True))
    calls(s, "bwd", lambda: s.cached_backward_gemm(W, dY, dX))
    calls(s, "dW", lambda: s.general_gemm(1.0, X, dY, 0.0, dW, False, True))
    calls(s, "fwd cache", lambda: s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True))
    calls(s, "bwd", lambda: s.cached_backward_gemm(W, dY, dX))
