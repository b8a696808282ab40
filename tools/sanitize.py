"""Small GEMM scenarios for compute-sanitizer (memcheck / racecheck / synccheck).

Covers the tcgen05 GEMM's schedules at sizes the sanitizer finishes quickly:
CTA group 1 / 2 x split mode mixed / 3xTF32, split-K (tall-skinny strips),
producer lockstep (one worker per device), fused split warps (K-panel pipeline
with remote pieces: 2 LOCAL workers on one GPU, DM_PIPELINE_MIN_GFLOP=0,
DM_PANEL_K=256), the four transposes, beta != 0, Half16 C and the
stream-ordered local_gemm seam.  Each scenario checks its result against a
float64 numpy product (relFro <= 1e-5), so a sanitizer run also proves the
instrumented launches computed the right thing.

  compute-sanitizer --tool racecheck python tools/sanitize.py [--quick]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402
from paper_1604_01416_b200 import Config, LayoutKind, Precision, Session, make_layout  # noqa: E402


def relfro(x, ref):
    return float(np.linalg.norm((x.astype(np.float64) - ref).ravel()) / max(np.linalg.norm(ref.ravel()), 1e-300))


def run(name, workers, mode, m, n, k, ta=False, tb=False, alpha=1.0, beta=0.0, prec=Precision.Single32, env=None,
        kind=LayoutKind.Checkerboard2D):
    for key, v in (env or {}).items():
        os.environ[key] = str(v)
    try:
        rng = np.random.default_rng(m * 7 + n * 13 + k)
        A = rng.uniform(-1, 1, (k, m) if ta else (m, k)).astype(np.float32)
        B = rng.uniform(-1, 1, (n, k) if tb else (k, n)).astype(np.float32)
        C0 = rng.uniform(-1, 1, (m, n)).astype(np.float32)
        if prec == Precision.Half16:
            A, B, C0 = (x.astype(np.float16).astype(np.float32) for x in (A, B, C0))
        with Session(Config(worker_count=workers, root_seed=7, gemm_mode=mode, devices=[0] * workers)) as s:
            def mat(h):
                r, c = h.shape
                br, bc = (r + 1) // 2 if workers > 1 else r, (c + 1) // 2 if workers > 1 else c
                lay = make_layout(kind, r, c, br, bc, workers)
                mid = s.create_matrix(lay, precision=prec)
                s.scatter(mid, h.astype(np.float16) if prec == Precision.Half16 else h)
                return mid
            a, b, c = mat(A), mat(B), mat(C0)
            s.general_gemm(alpha, a, b, beta, c, trans_a=ta, trans_b=tb)
            out = s.gather(c).astype(np.float32)
        opA = A.T if ta else A
        opB = B.T if tb else B
        ref = alpha * (opA.astype(np.float64) @ opB.astype(np.float64)) + beta * C0.astype(np.float64)
        err = relfro(out, ref)
        tol = 1e-3 if prec == Precision.Half16 else 1e-5
        ok = err <= tol
        print(f"{name:40s} relFro {err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
        return ok
    finally:
        for key in (env or {}):
            os.environ.pop(key, None)


def run_local_gemm(m, n, k, cg):
    import torch
    a = torch.rand(m, k, device="cuda") - 0.5
    b = torch.rand(k, n, device="cuda") - 0.5
    c = torch.rand(m, n, device="cuda") - 0.5
    ref = 1.5 * (a.double() @ b.double()) - 0.5 * c.double()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dm.local_gemm(1.5, a, False, b, False, -0.5, c, cta_group=cg, stream=st.cuda_stream)
    st.synchronize()
    err = float((c.double() - ref).norm() / ref.norm())
    ok = err <= 1e-5
    print(f"{'local_gemm cg' + str(cg) + f' {m}x{n}x{k}':40s} relFro {err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="one shape per schedule")
    ap.add_argument("--only", default="", help="substring filter on scenario names")
    args = ap.parse_args()
    cases = []
    for cg in (1, 2):
        for mode in ("mixed", "3xtf32"):
            cases.append((f"square cg{cg} {mode}", 1, mode, 512, 512, 512, False, False, 1.0, 0.0,
                          Precision.Single32, {"DM_CTA_GROUP": cg}))
            cases.append((f"splitK strip cg{cg} {mode}", 1, mode, 256, 256, 4096, False, False, 1.0, 0.0,
                          Precision.Single32, {"DM_CTA_GROUP": cg, "DM_LOCKSTEP": 0}))
            cases.append((f"lockstep 2 waves cg{cg} {mode}", 1, mode, 1024, 2560 if cg == 2 else 1280, 1024,
                          False, False, 1.0, 0.0, Precision.Single32, {"DM_CTA_GROUP": cg, "DM_LOCKSTEP": 2}))
            cases.append((f"fused split P2 cg{cg} {mode}", 2, mode, 512, 512, 1024, False, True, 1.5, -0.5,
                          Precision.Single32, {"DM_CTA_GROUP": cg, "DM_PIPELINE_MIN_GFLOP": 0, "DM_PANEL_K": 256,
                                                "DM_FUSE_SPLIT": 1}))
    for ta in (False, True):
        for tb in (False, True):
            cases.append((f"transposes ta={int(ta)} tb={int(tb)} beta", 1, "auto", 384, 320, 448, ta, tb, 1.5, -0.5,
                          Precision.Single32, {}))
    cases.append(("half16 C P2 pipeline", 2, "auto", 256, 256, 1024, False, False, 1.0, 1.0, Precision.Half16,
                  {"DM_PIPELINE_MIN_GFLOP": 0, "DM_PANEL_K": 256}))
    if args.quick:
        cases = [c for c in cases if "cg2" in c[0] or "transposes ta=1 tb=1" in c[0]]
    if args.only:
        cases = [c for c in cases if args.only in c[0]]
    ok = True
    for c in cases:
        ok &= run(*c)
    if not args.only or "local_gemm" in args.only:
        for cg in (1, 2):
            ok &= run_local_gemm(256, 384, 512, cg)
    print("ALL OK" if ok else "FAILURES", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
