"""Host overhead per command: wall time of tiny GEMM commands (the device work
is a few microseconds), LOCAL mode on one GPU, and of the local_gemm seam."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

for P in (1, 4):
    with dm.Session(dm.Config(worker_count=P, root_seed=1, devices=[0] * P)) as s:
        lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, 256, 256, 256 // dm.checkerboard_dims(P)[0],
                             256 // dm.checkerboard_dims(P)[1], P)
        a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
        for _ in range(20):
            s.general_gemm(1.0, a, b, 0.0, c)
        t0 = time.perf_counter()
        for _ in range(200):
            s.general_gemm(1.0, a, b, 0.0, c)
        dt = (time.perf_counter() - t0) / 200
        s.set_async(True)
        t0 = time.perf_counter()
        for _ in range(200):
            s.general_gemm(1.0, a, b, 0.0, c)
        s.barrier()
        dta = (time.perf_counter() - t0) / 200
        s.set_async(False)
        print(f"general_gemm 256^3 P={P}: {dt * 1e6:.1f} us/call sync, {dta * 1e6:.1f} us/call async", flush=True)
A = torch.rand(256, 256, device="cuda")
B = torch.rand(256, 256, device="cuda")
C = torch.zeros(256, 256, device="cuda")
for _ in range(20):
    dm.local_gemm(1.0, A, False, B, False, 0.0, C)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    dm.local_gemm(1.0, A, False, B, False, 0.0, C)
torch.cuda.synchronize()
print(f"local_gemm 256^3: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us/call", flush=True)
