"""Cost of K panels on one GPU: local_gemm (split + tcgen05 GEMM, f16x2) of an
M x N block over K, as one launch or as K/w panel launches accumulating
with beta = 1 -- the per-panel price the distributed pipeline pays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 16384, 32768)))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
A = torch.rand(M, K, device=dev, generator=g) * 2 - 1
B = torch.rand(K, N, device=dev, generator=g) * 2 - 1
Cm = torch.zeros(M, N, device=dev)
st = torch.cuda.current_stream().cuda_stream


def run(width, beta0):
    for p, k0 in enumerate(range(0, K, width)):
        dm.local_gemm(1.0, A[:, k0:k0 + width], False, B[k0:k0 + width], False, beta0 if p == 0 else 1.0, Cm,
                      stream=st, gemm_mode="f16x2")


for width in (K, K // 2, K // 4, K // 8):
    for beta0 in (0.0, 1.0):
        run(width, beta0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run(width, beta0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"M={M} N={N} K={K} panels of {width:6d} first beta={beta0:.0f}: {ms:8.2f} ms "
              f"({2.0 * M * N * K / ms / 1e9:6.1f} TFLOP/s incl. splits)", flush=True)
