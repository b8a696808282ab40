"""Does host->device copy bandwidth drop while the SMs are saturated?  Times
a 4 GiB pinned H2D copy alone and while a long stream of bf16 GEMMs (and,
second, our own f16x2 GEMM through local_gemm) keeps the GPU busy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

dev = torch.device("cuda", 0)
nbytes = 4 << 30
h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
d = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
s_copy = torch.cuda.Stream()
s_work = torch.cuda.Stream()


def h2d_ms():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_copy):
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1)


print(f"H2D 4 GiB alone: {h2d_ms():.1f} ms", flush=True)
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
with torch.cuda.stream(s_work):
    for _ in range(400):
        torch.matmul(a, a)
time.sleep(0.05)
print(f"H2D 4 GiB under bf16 GEMMs: {h2d_ms():.1f} ms", flush=True)
torch.cuda.synchronize()
N = 16384
A = torch.rand(N, N, device=dev) * 2 - 1
B = torch.rand(N, N, device=dev) * 2 - 1
C = torch.zeros(N, N, device=dev)
for _ in range(12):
    dm.local_gemm(1.0, A, False, B, False, 0.0, C, stream=s_work.cuda_stream, gemm_mode="f16x2")
time.sleep(0.05)
print(f"H2D 4 GiB under f16x2 GEMMs: {h2d_ms():.1f} ms", flush=True)
torch.cuda.synchronize()
