"""Measure the non-headline BASELINE.json configs (bench.py measures config 3).

  1  2048^3, 2x2 checkerboard, P=4 (+ the reference CPU general_gemm, --ref)
  2  N=16384 square on 1 GPU, persistent device operands
  4  FC layers, batch 256: 9216->4096 and 4096->4096, reference convention
     fwd Y = W^T X (cyclic_gemm TN, cache W), bwd dX = W dY (cached_backward_gemm NN),
     dW = X dY^T (general_gemm NT), over min(8, #GPUs) GPUs (+ reference CPU, --ref)
  5  chained C = A*B; D = C*E on device-resident checkerboard matrices, pool reuse

Workers are one per GPU in a LOCAL session (peer access); timings are device
events around each call (markers on worker 0's GEMM stream, max over the call
since every call ends with a full sync).  Prints one JSON line per config.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402


def timed(s, fn, reps):
    for _ in range(3):  # warm-up: allocations, first pulls, graph captures (steady state after)
        fn()
    s.barrier()
    t0 = time.perf_counter()
    s.marker_record(0, 4)
    for _ in range(reps):
        fn()
    s.marker_record(0, 5)
    wall = (time.perf_counter() - t0) / reps
    return s.marker_elapsed(0, 4, 5) / reps, wall * 1e3


def peaks():
    """Measured per-GPU peaks (MEASURED_PEAKS.json): HBM GB/s and the split
    schemes' useful fp32 TFLOP/s (bf16 dense / 4 mixed, / 6 3xTF32)."""
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return p["hbm_gbs"], p["bf16_tflops_sustained"]
    except Exception:
        return 6500.0, 1400.0


NVLINK_GBS = 750.0  # per-GPU peer read bandwidth used for the link bound (NVLink 5, one direction, measured ~700-800)


def roofline(ms, flops_w, hbm_bytes_w, link_bytes_w, k):
    """Per-op roofline of one worker's share (the workers run in parallel):
    the slowest of tensor time (the split scheme auto picks at this K), HBM
    bytes (raw fp32 operands read + C written) and NVLink bytes (pulled pieces)."""
    hbm, bf16 = peaks()
    tensor = bf16 / {"mixed": 4.0, "3xtf32": 6.0, "f16x2": 3.0}[dm.split_mode_for("auto", k)]
    t = {"tensor": flops_w / (tensor * 1e12) * 1e3, "hbm": hbm_bytes_w / (hbm * 1e9) * 1e3,
         "nvlink": link_bytes_w / (NVLINK_GBS * 1e9) * 1e3}
    kind = max(t, key=t.get)
    return {"bound": kind, "bound_ms": round(t[kind], 5), "frac": round(t[kind] / ms, 4),
            "tensor_ms": round(t["tensor"], 5), "hbm_ms": round(t["hbm"], 5), "nvlink_ms": round(t["nvlink"], 5)}


def cfg1(args, ndev):
    n, P = 2048, 4
    devs = [w % ndev for w in range(P)]
    with dm.Session(dm.Config(worker_count=P, root_seed=42, devices=devs)) as s:
        lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
        a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
        ms, wall = timed(s, lambda: s.general_gemm(1.0, a, b, 0.0, c), 20)
        h = n // 2  # per worker: C block h x h over K = n; A row panel + B column panel, half of each remote
        out = {"config": 1, "workload": "general_gemm 2048^3, 2x2 checkerboard, P=4", "devices": devs,
               "ms": round(ms, 4), "tflops": 2 * n ** 3 / ms / 1e9, "wall_ms": round(wall, 4),
               "roofline": roofline(ms, 2.0 * h * h * n, 4.0 * (2 * h * n + h * h), 4.0 * 2 * h * (n - h), n)}
        if args.ref:
            from oracle import RefOracle
            ro = RefOracle()
            with ro.session(4, 42, deterministic=False) as rs:
                ra, rb, rc = (rs.create(3, n, n, n // 2, n // 2, 4) for _ in range(3))
                t0 = time.perf_counter()
                rs.general_gemm(1.0, ra, rb, 0.0, rc)
                dt = time.perf_counter() - t0
                refC = rs.gather(rc)
            from oracle import COracle
            out["reference_cpu_s"] = round(dt, 2)
            out["reference_cpu_gflops"] = 2 * n ** 3 / dt / 1e9
            out["relfro_vs_reference"] = COracle().rel_frobenius(s.gather(c), refC)
            out["speedup_vs_reference"] = dt * 1e3 / ms
    print(json.dumps(out), flush=True)


def cfg2(args):
    n = 16384
    with dm.Session(dm.Config(worker_count=1, root_seed=42, devices=[0])) as s:
        lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n, n, 1)
        a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
        ms, wall = timed(s, lambda: s.general_gemm(1.0, a, b, 0.0, c), 5)
    print(json.dumps({"config": 2, "workload": "general_gemm 16384^3 on 1 GPU", "ms": round(ms, 3),
                      "tflops": 2 * n ** 3 / ms / 1e9}), flush=True)


def cfg4(args, ndev):
    P = min(8, ndev) if args.fc_workers is None else args.fc_workers
    devs = [w % ndev for w in range(P)]
    batch, fout = 256, 4096
    for fin in (9216, 4096):
        strip = batch // P
        with dm.Session(dm.Config(worker_count=P, root_seed=3, devices=devs)) as s:
            W = s.create_matrix(dm.make_layout(0, fin, fout, fin // P, fout, P), fill=dm.FillKind.SeededRandom)
            X = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, P), fill=dm.FillKind.SeededRandom)
            Y = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, P))
            dY = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, P), fill=dm.FillKind.SeededRandom)
            dX = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, P))
            dW = s.create_matrix(dm.make_layout(0, fin, fout, fin // P, fout, P))
            # forward without the block cache: every call pulls the foreign W blocks
            s.reset_worker_stats()
            fwd_pull_ms, _ = timed(s, lambda: s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, False), 10)
            pulled = sum(s.worker_stats(w).peer_bytes_read for w in range(P)) // 13
            # forward with cache_a: W pulled once, later calls read the fresh cache
            s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
            s.reset_worker_stats()
            fwd_ms, _ = timed(s, lambda: s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True), 20)
            fwd_cached_peer = sum(s.worker_stats(w).peer_bytes_read for w in range(P))
            s.reset_worker_stats()
            bwd_ms, _ = timed(s, lambda: s.cached_backward_gemm(W, dY, dX), 20)
            bwd_peer = sum(s.worker_stats(w).peer_bytes_read for w in range(P))
            dw_ms, _ = timed(s, lambda: s.general_gemm(1.0, X, dY, 0.0, dW, False, True), 20)
            # W-stationary forward: W split by output features,
            # X replicated (one all-gather per batch), Y row-blocked: 0 W bytes move
            Wc = s.create_matrix(dm.make_layout(1, fin, fout, fin, fout // P, P), fill=dm.FillKind.SeededRandom)
            Xr = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, P), fill=dm.FillKind.SeededRandom)
            Yr = s.create_matrix(dm.make_layout(0, fout, batch, fout // P, batch, P))
            s.barrier()
            s.marker_record(0, 4)
            s.replicate(Xr, True)  # the per-batch all-gather of X
            s.marker_record(0, 5)
            rep_ms = s.marker_elapsed(0, 4, 5)
            s.reset_worker_stats()
            ws_ms, _ = timed(s, lambda: s.general_gemm(1.0, Wc, Xr, 0.0, Yr, True, False), 20)
            ws_peer = sum(s.worker_stats(w).peer_bytes_read for w in range(P))
            fl = 2.0 * fin * fout * batch
            fl_pull = fl
            b = batch // P
            # per worker: fwd / bwd read all of W + the X / dY strip, write the Y / dX strip;
            # dW reads its X rows (all batch columns, 3/4 remote) and all of dY (3/4 remote)
            rl = {"fwd_TN_pull": roofline(fwd_pull_ms, fl / P, 4.0 * (fin * fout + fin * b + fout * b),
                                          4.0 * fin * fout * (P - 1) / P, fin),
                  "fwd_TN_cached": roofline(fwd_ms, fl / P, 4.0 * (fin * fout + fin * b + fout * b), 0, fin),
                  "bwd_NN_cached": roofline(bwd_ms, fl / P, 4.0 * (fin * fout + fout * b + fin * b), 0, fout),
                  "dW_NT": roofline(dw_ms, fl / P, 4.0 * (fin // P * batch + fout * batch + fin // P * fout),
                                    4.0 * (fin // P * batch + fout * batch) * (P - 1) / P, batch),
                  "fwd_wstationary": roofline(ws_ms, fl / P, 4.0 * (fin * fout // P + fin * batch + fout // P * batch),
                                              0, fin)}
            out = {"config": 4, "workload": f"FC {fin}->{fout}, batch {batch}, P={P}", "devices": devs,
                   "fwd_TN_pull_ms": round(fwd_pull_ms, 4), "fwd_pull_peer_bytes_per_call": int(pulled),
                   "fwd_TN_cached_ms": round(fwd_ms, 4), "fwd_cached_peer_bytes": int(fwd_cached_peer), "bwd_NN_cached_ms": round(bwd_ms, 4),
                   "bwd_peer_bytes": int(bwd_peer), "dW_NT_ms": round(dw_ms, 4),
                   "fwd_wstationary_ms": round(ws_ms, 4), "fwd_wstationary_peer_bytes": int(ws_peer),
                   "replicate_X_ms": round(rep_ms, 4),
                   "fwd_pull_tflops": fl_pull / fwd_pull_ms / 1e9, "fwd_tflops": fl / fwd_ms / 1e9, "bwd_tflops": fl / bwd_ms / 1e9, "dW_tflops": fl / dw_ms / 1e9,
                   "roofline": rl}
            if args.ref:
                from oracle import RefOracle
                ro = RefOracle()
                with ro.session(P, 3, deterministic=False) as rs:
                    rW = rs.create(0, fin, fout, fin // P, fout, P)
                    rX = rs.create(1, fin, batch, fin, strip, P)
                    rY = rs.create(1, fout, batch, fout, strip, P, fill=0)
                    rdY = rs.create(1, fout, batch, fout, strip, P)
                    rdX = rs.create(1, fin, batch, fin, strip, P, fill=0)
                    rdW = rs.create(0, fin, fout, fin // P, fout, P, fill=0)
                    t = time.perf_counter(); rs.cyclic_gemm(1.0, rW, rX, 0.0, rY, True, False, True); f = time.perf_counter() - t
                    t = time.perf_counter(); rs.cached_backward_gemm(rW, rdY, rdX); bw = time.perf_counter() - t
                    t = time.perf_counter(); rs.general_gemm(1.0, rX, rdY, 0.0, rdW, False, True); d = time.perf_counter() - t
                    from oracle import COracle
                    orc = COracle()
                    out["reference_cpu_s"] = {"fwd": round(f, 2), "bwd": round(bw, 2), "dW": round(d, 2)}
                    out["relfro_vs_reference"] = {"Y": orc.rel_frobenius(s.gather(Y), rs.gather(rY)),
                                                  "dX": orc.rel_frobenius(s.gather(dX), rs.gather(rdX)),
                                                  "dW": orc.rel_frobenius(s.gather(dW), rs.gather(rdW))}
            print(json.dumps(out), flush=True)


def cfg5(args, ndev):
    P = min(4, ndev) if ndev >= 4 else (2 if ndev >= 2 else 1)
    n = args.chain_n
    pr, pc = dm.checkerboard_dims(P)
    devs = list(range(P))
    with dm.Session(dm.Config(worker_count=P, root_seed=5, devices=devs)) as s:
        lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // pr, n // pc, P)
        A, B, E = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
        Cm, D = s.create_matrix(lay), s.create_matrix(lay)

        def chain():
            s.general_gemm(1.0, A, B, 0.0, Cm)
            s.general_gemm(1.0, Cm, E, 0.0, D)
        chain()
        fresh = [s.worker_pool_stats(w).fresh_allocations for w in range(P)]
        ms, _ = timed(s, chain, 3)
        fresh2 = [s.worker_pool_stats(w).fresh_allocations for w in range(P)]
        reuses = [s.worker_pool_stats(w).reuses for w in range(P)]
    print(json.dumps({"config": 5, "workload": f"chained C=A*B; D=C*E, N={n}, {pr}x{pc} grid, P={P}",
                      "ms_per_chain": round(ms, 2), "tflops": 4.0 * n ** 3 / ms / 1e9,
                      "pool_fresh_after_iter1": fresh, "pool_fresh_after_timed": fresh2,
                      "pool_steady": fresh == fresh2, "pool_reuses": reuses}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--ref", action="store_true", help="also time the reference CPU path (configs 1, 4)")
    ap.add_argument("--fc-workers", type=int, default=None)
    ap.add_argument("--chain-n", type=int, default=16384)
    args = ap.parse_args()
    ndev = torch.cuda.device_count()
    want = {int(x) for x in args.configs.split(",")}
    if 1 in want:
        cfg1(args, ndev)
    if 2 in want:
        cfg2(args)
    if 4 in want:
        cfg4(args, ndev)
    if 5 in want:
        cfg5(args, ndev)


if __name__ == "__main__":
    main()
