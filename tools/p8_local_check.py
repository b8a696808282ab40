"""The 8-GPU headline layout (2x4 checkerboard, N=32768) on the GPUs at hand:
a LOCAL session of 8 workers (two per GPU on a 4-GPU box) runs the presplit
GEMM at full size -- planes split by their 8 owners, whole-row scales from
4-block (A) / 2-block (B) row bands, 16384-wide panels spanning two of A's K
blocks -- and sampled rows / columns are checked against float64.  A
correctness check of the 8-rank schedule at full size, not a timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

N = int(os.environ.get("P8_N", "32768"))
ndev = torch.cuda.device_count()
P = 8
pr, pc = dm.checkerboard_dims(P)
with dm.Session(dm.Config(worker_count=P, root_seed=42, devices=[w % ndev for w in range(P)])) as s:
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N // pr, N // pc, P)
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    s.reset_worker_stats()
    t0 = time.perf_counter()
    s.general_gemm(1.0, a, b, 0.0, c)
    dt = time.perf_counter() - t0
    st = [s.worker_stats(w) for w in range(P)]
    print(f"P=8 ({pr}x{pc}) N={N} on {ndev} GPUs: {dt * 1e3:.1f} ms wall; split launches "
          f"{[x.split_launches for x in st]}, gemm launches {[x.gemm_launches for x in st]}, "
          f"peer MiB {[int(x.peer_bytes_read) >> 20 for x in st]}", flush=True)
    A, B, C = s.gather(a), s.gather(b), s.gather(c)
rows = [(i * 4099 + 17) % N for i in range(8)]
cols = [(j * 4111 + 29) % N for j in range(8)]
Bd = B.astype(np.float64)
want_r = A[rows].astype(np.float64) @ Bd
want_c = A.astype(np.float64) @ Bd[:, cols]
err_r = np.linalg.norm(C[rows] - want_r) / np.linalg.norm(want_r)
err_c = np.linalg.norm(C[:, cols] - want_c) / np.linalg.norm(want_c)
print(f"sampled rows relFro vs fp64 {err_r:.2e}, columns {err_c:.2e}", flush=True)
assert err_r < 1e-5 and err_c < 1e-5
