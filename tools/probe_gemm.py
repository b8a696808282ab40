"""Quick throughput probe of the session GEMM on one GPU (not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_01416_b200 import Config, FillKind, LayoutKind, Session, make_layout  # noqa: E402

sizes = [int(x) for x in (sys.argv[1:] or ["4096", "8192", "16384"])]
for n in sizes:
    with Session(Config(worker_count=1, root_seed=42)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n, n, 1)
        a = s.create_matrix(lay, fill=FillKind.SeededRandom)
        b = s.create_matrix(lay, fill=FillKind.SeededRandom)
        c = s.create_matrix(lay)
        s.set_gemm_timing(True)
        s.general_gemm(1.0, a, b, 0.0, c)
        s.reset_worker_stats()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            s.general_gemm(1.0, a, b, 0.0, c)
        wall = (time.perf_counter() - t0) / reps
        st = s.worker_stats(0)
        kms = st.gemm_ms / reps
        fl = 2.0 * n ** 3
        print(f"mode={os.environ.get('DM_GEMM_MODE', '1')} N={n} cg={os.environ.get('DM_CTA_GROUP', 'auto')} gemm_kernel={kms:.2f} ms "
              f"({fl / kms / 1e9:.1f} TFLOP/s)  command={wall * 1e3:.2f} ms ({fl / wall / 1e12:.1f} TFLOP/s)",
              flush=True)
