"""Scaled 2xFP16 split (kModeF16x2) probe: accuracy against float64 on hard
distributions, session paths (single panel, batched split, fused two-phase
split), and throughput beside the other split schemes on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

dev = torch.device("cuda")


def gen(dist, shape, g):
    if dist == "pm1":
        return torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1
    if dist == "u01":
        return torch.rand(shape, generator=g, dtype=torch.float64)
    if dist.startswith("logu"):
        e = float(dist[4:])
        sgn = torch.randint(0, 2, shape, generator=g).double() * 2 - 1
        return sgn * torch.pow(2.0, (torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1) * e)
    if dist == "tiny":
        return (torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1) * 1e-17  # products ~1e-34
    if dist == "huge":
        return (torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1) * 1e15  # products ~1e30
    if dist == "rowscale":  # rows of A spanning 2^-60 .. 2^60
        x = torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1
        return x * torch.pow(2.0, torch.linspace(-60, 60, shape[0], dtype=torch.float64))[:, None]
    raise ValueError(dist)


def accuracy():
    g = torch.Generator().manual_seed(0)
    print("== local_gemm accuracy vs float64 (relFro), reference fp32 k-ascending on 4 rows", flush=True)
    for dist in ["pm1", "u01", "logu20", "logu60", "tiny", "huge", "rowscale"]:
        for k in [256, 4096, 32768]:
            m = n = 512
            A = gen(dist, (m, k), g).float()
            B = gen(dist if dist != "rowscale" else "pm1", (k, n), g).float()
            ex = A.double() @ B.double()
            nrm = ex.norm()
            row = []
            for mode in ["f16x2", "3xtf32", "mixed"]:
                C = torch.zeros(m, n, device=dev)
                dm.local_gemm(1.0, A.to(dev), False, B.to(dev), False, 0.0, C, gemm_mode=mode)
                torch.cuda.synchronize()
                row.append(float((C.double().cpu() - ex).norm() / nrm))
            a4, b = A[:4].numpy(), B.numpy()
            acc = np.zeros((4, n), np.float32)
            for kk in range(0, k, 1):
                acc = (acc + np.outer(a4[:, kk], b[kk]).astype(np.float32)).astype(np.float32)
            ref = float(np.linalg.norm(acc - ex[:4].numpy()) / np.linalg.norm(ex[:4].numpy()))
            print(f"{dist:8s} K={k:6d}  f16x2 {row[0]:.2e}  3xtf32 {row[1]:.2e}  mixed {row[2]:.2e}  "
                  f"ref-fp32 {ref:.2e}", flush=True)


def transposes():
    g = torch.Generator().manual_seed(1)
    print("== transposes / alpha beta / odd shapes (f16x2)", flush=True)
    for (m, n, k) in [(300, 333, 200), (513, 257, 1000), (64, 96, 8192), (1024, 1024, 1024)]:
        for ta in (False, True):
            for tb in (False, True):
                A = gen("pm1", (k, m) if ta else (m, k), g).float().to(dev)
                B = gen("pm1", (n, k) if tb else (k, n), g).float().to(dev)
                C = gen("pm1", (m, n), g).float().to(dev)
                ref = 1.5 * ((A.T if ta else A).double() @ (B.T if tb else B).double()) - 0.5 * C.double()
                for cg in (1, 2):
                    Cw = C.clone()
                    dm.local_gemm(1.5, A, ta, B, tb, -0.5, Cw, cta_group=cg, gemm_mode="f16x2")
                    torch.cuda.synchronize()
                    err = float((Cw.double() - ref).norm() / ref.norm())
                    flag = "ok" if err < 1e-5 else "FAIL"
                    print(f"  {m}x{n}x{k} ta={int(ta)} tb={int(tb)} cg={cg}: {err:.2e} {flag}", flush=True)


def session_paths():
    print("== session paths (f16x2)", flush=True)
    cases = [("P1 single panel", 1, {}, 4096),
             ("P1 geometric panels, fused 2-phase split", 1, {"DM_PANEL_LOCAL": "1024"}, 8192),
             ("P2 one GPU, forced pipeline (separate splits)", 2,
              {"DM_PIPELINE_MIN_GFLOP": "0", "DM_PANEL_K": "1024"}, 4096),
             ("P4 one GPU, batched split", 4, {}, 1024)]
    for name, P, env, n in cases:
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            with dm.Session(dm.Config(worker_count=P, root_seed=5, devices=[0] * P, gemm_mode="f16x2")) as s:
                pr, pc = dm.checkerboard_dims(P)
                lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // pr, n // pc, P)
                a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
                s.reset_worker_stats()
                s.general_gemm(1.0, a, b, 0.0, c)
                st = s.worker_stats(0)
                A, B, C = s.gather(a), s.gather(b), s.gather(c)
                idx = np.arange(0, n, max(1, n // 64))
                ex = A[idx].astype(np.float64) @ B.astype(np.float64)
                err = np.linalg.norm(C[idx] - ex) / np.linalg.norm(ex)
                print(f"  {name:48s} N={n} launches gemm={st.gemm_launches} split={st.split_launches} "
                      f"relFro(64 rows)={err:.2e} {'ok' if err < 1e-5 else 'FAIL'}", flush=True)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


def throughput():
    print("== throughput, P=1 session general_gemm (kernel / command)", flush=True)
    for n in [int(x) for x in os.environ.get("PROBE_N", "16384 32768").split()]:
        for mode in ["f16x2", "mixed", "3xtf32"]:
            with dm.Session(dm.Config(worker_count=1, root_seed=42, gemm_mode=mode)) as s:
                lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n, n, 1)
                a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
                s.set_gemm_timing(True)
                s.general_gemm(1.0, a, b, 0.0, c)
                s.reset_worker_stats()
                reps = 3
                t0 = time.perf_counter()
                for _ in range(reps):
                    s.general_gemm(1.0, a, b, 0.0, c)
                wall = (time.perf_counter() - t0) / reps
                kms = s.worker_stats(0).gemm_ms / reps
                fl = 2.0 * n ** 3
                print(f"  N={n} {mode:7s} kernel {kms:8.2f} ms ({fl / kms / 1e9:6.1f} TFLOP/s)  command "
                      f"{wall * 1e3:8.2f} ms ({fl / wall / 1e12:6.1f} TFLOP/s)", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["accuracy", "transposes", "session", "throughput"]
    if "accuracy" in what:
        accuracy()
    if "transposes" in what:
        transposes()
    if "session" in what:
        session_paths()
    if "throughput" in what:
        throughput()
