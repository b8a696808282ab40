"""Accuracy and speed of the split GEMM vs the TMEM flush chunk (DM_FLUSH_K)
and split mode: relFro vs fp64 at K = 256 / 4096 / 32768 (U[-1,1), 1024^2 C,
CTA-pair tiles) and TFLOP/s at 16384^3 through the local_gemm seam."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1604_01416_b200 import local_gemm  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator().manual_seed(0)
ops = {}
for k in (256, 4096, 32768):
    A = (torch.rand(1024, k, generator=g) * 2 - 1).to(dev)
    B = (torch.rand(k, 1024, generator=g) * 2 - 1).to(dev)
    ops[k] = (A, B, A.double() @ B.double())
N = 16384
A16 = (torch.rand(N, N, generator=g) * 2 - 1).to(dev)
B16 = (torch.rand(N, N, generator=g) * 2 - 1).to(dev)
C16 = torch.empty(N, N, device=dev)
for mode in ("mixed", "3xtf32"):
    for flush in (64, 128, 256, 512):
        os.environ["DM_FLUSH_K"] = str(flush)
        errs = []
        for k, (A, B, want) in ops.items():
            C = torch.empty(1024, 1024, device=dev)
            local_gemm(1.0, A, False, B, False, 0.0, C, cta_group=2, gemm_mode=mode)
            torch.cuda.synchronize()
            errs.append(float((C.double() - want).norm() / want.norm()))
        for _ in range(2):
            local_gemm(1.0, A16, False, B16, False, 0.0, C16, gemm_mode=mode)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        reps = 5
        for _ in range(reps):
            local_gemm(1.0, A16, False, B16, False, 0.0, C16, gemm_mode=mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"mode={mode} flush={flush} relFro K256={errs[0]:.3e} K4096={errs[1]:.3e} K32768={errs[2]:.3e} "
              f"16384^3 {ms:.2f} ms {2 * N**3 / ms / 1e9:.1f} TFLOP/s", flush=True)
