"""The 4-GPU headline step as one rank sees it, for ncu: a LOCAL session over
4 GPUs (2x2 grid, N=32768 by default), owner-split planes pulled from the
peers' arenas; run under ncu --devices 0 to capture worker 0's GEMM launch
(16384 x 16384 x 16384 K panel).  Without ncu it prints worker 0's stats and
one sampled row against float64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

n = int(os.environ.get("P4_N", "32768"))
P = int(os.environ.get("P4_WORKERS", "4"))  # 2: the 1x2 grid of the 2-GPU bench
pr, pc = dm.checkerboard_dims(P)
with dm.Session(dm.Config(worker_count=P, root_seed=42, devices=list(range(P)))) as s:
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // pr, n // pc, P)
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    s.reset_worker_stats()
    for _ in range(2):
        s.general_gemm(1.0, a, b, 0.0, c)
    st = s.worker_stats(0)
    print(f"worker0: gemm_launches={st.gemm_launches} split_launches={st.split_launches} "
          f"peer_bytes={st.peer_bytes_read / 2**20:.0f} MiB", flush=True)
    if os.environ.get("P4_CHECK", "1") == "1":
        A, B, C = s.gather(a), s.gather(b), s.gather(c)
        i = 12345 % n
        ref = A[i].astype(np.float64) @ B.astype(np.float64)
        err = np.linalg.norm(C[i] - ref) / np.linalg.norm(ref)
        print(f"row {i} relFro vs fp64 {err:.2e}", flush=True)
        assert err < 1e-5
