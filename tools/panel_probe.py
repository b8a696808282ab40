"""One-worker panel schedules at N (default 32768): command and GEMM-kernel
time per configuration given as ENV=VAL[,ENV=VAL...] arguments ("-" = defaults)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_01416_b200 as dm  # noqa: E402

n = int(os.environ.get("PROBE_N", "32768"))
mode = os.environ.get("PROBE_MODE", "f16x2")
with dm.Session(dm.Config(worker_count=1, root_seed=42, gemm_mode=mode)) as s:
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n, n, 1)
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    for spec in sys.argv[1:] or ["-"]:
        env = dict(kv.split("=") for kv in spec.split(",")) if spec != "-" else {}
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        s.set_gemm_timing(True)
        s.general_gemm(1.0, a, b, 0.0, c)
        s.reset_worker_stats()
        reps = int(os.environ.get("PROBE_REPS", "3"))
        s.barrier()
        s.marker_record(0, 0)
        for _ in range(reps):
            s.general_gemm(1.0, a, b, 0.0, c)
        s.marker_record(0, 1)
        ms = s.marker_elapsed(0, 0, 1) / reps
        st = s.worker_stats(0)
        kms = st.gemm_ms / reps
        fl = 2.0 * n ** 3
        print(f"{spec:60s} command {ms:8.2f} ms ({fl / ms / 1e9:6.1f} TFLOP/s)  gemm {kms:8.2f} ms  "
              f"launches gemm={st.gemm_launches // reps} split={st.split_launches // reps}", flush=True)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
