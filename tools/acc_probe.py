"""Accuracy vs K and flush chunk (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1604_01416_b200 import local_gemm
dev = torch.device("cuda")
g = torch.Generator().manual_seed(0)
for k in [1024, 4096, 16384, 32768]:
    A = (torch.rand(512, k, generator=g) * 2 - 1).to(dev)
    B = (torch.rand(k, 512, generator=g) * 2 - 1).to(dev)
    want = A.double() @ B.double()
    f32 = (A @ B) if False else None
    row = []
    for cg in (1, 2):
        C = torch.empty(512, 512, device=dev)
        local_gemm(1.0, A, False, B, False, 0.0, C, cta_group=cg)
        torch.cuda.synchronize()
        row.append(float((C.double() - want).norm() / want.norm()))
    # fp32 k-ascending reference arithmetic on a few rows (numpy cumsum in float32)
    a = A[:8].cpu().numpy(); b = B.cpu().numpy()
    import numpy as np
    acc = np.zeros((8, 512), np.float32)
    for kk in range(k):
        acc = (acc + np.outer(a[:, kk], b[kk]).astype(np.float32)).astype(np.float32)
    w8 = want[:8].cpu().numpy()
    ref = float(np.linalg.norm(acc - w8) / np.linalg.norm(w8))
    print(f"mode={os.environ.get('DM_GEMM_MODE','1')} K={k} flush={os.environ.get('DM_FLUSH_K','256')} relFro cg1={row[0]:.3e} cg2={row[1]:.3e} fp32-kasc(8 rows)={ref:.3e}", flush=True)
