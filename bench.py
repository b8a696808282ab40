#!/usr/bin/env python
"""Distributed SGEMM benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 32768]

One step = one fp32 general_gemm C = A*B at N x N x N (default N=32768) on a
Checkerboard2D layout over the pr x pc process grid of the N GPUs (the
reference's checkerboard_dims, layout.hpp:100-105), operands resident in HBM,
synthetic inputs from the reference's seeded fill (root seed 42).  Total work
is fixed as N grows ("strong" scaling).  Rank 0 prints one JSON line.

--impl reference times the reference's own CPU implementation
(oracle/_ref = /root/reference compiled unmodified) on the host cores: each
step is a bounded sample -- whole rows of the same N^3 GEMM through the
reference's local_gemm on the reference's panel geometry (full K, stride N),
which are bit-identical to the rows its distributed general_gemm produces.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "distributed SGEMM TFLOP/s at N=32768 on 1/2/4/8 B200; % of roofline; vs CPU ref"


# ------------------------------------------------------------------ helpers
def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def gemm_mode() -> int:
    return 0 if os.environ.get("DM_GEMM_MODE", "1") == "0" else 1


def measured_peaks():
    """Useful-fp32-flop peak of the MMA mix actually executed, from the measured
    dense bf16 rate: TF32 runs at bf16/2, so per useful k16 step
      3xTF32: 6 TF32 k8 MMAs            = 6 bf16-k16 slots -> peak = bf16 / 6
      mixed : 2 TF32 k8 + 2 BF16 k16    = 4 bf16-k16 slots -> peak = bf16 / 4"""
    div = 6.0 if gemm_mode() == 0 else 4.0
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return (p["bf16_tflops"] / div, p["bf16_tflops_sustained"] / div,
                f"measured (MEASURED_PEAKS.json bf16 / {div:.0f})", p["bf16_tflops_sustained"] / 6.0)
    except Exception:
        return 1590.0 / div, 1400.0 / div, f"fallback (B200_PROFILING.md bf16 / {div:.0f})", 1400.0 / 6.0


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 200 ms from before the
    warm-up; stop() keeps the samples whose host timestamp falls inside the
    timed window [mark_start, mark_end] (the nearest one if the window is
    shorter than the sampling period)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                gpu = int(vis.split(",")[gpu])
            except (ValueError, IndexError):
                pass
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)  # let the sample after the window land
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        t0 = self.t0 or 0.0
        t1 = self.t1 or time.time()
        inside = [(t, ln) for t, ln in self.lines if t0 <= t <= t1 + 0.2]
        if not inside and self.lines:
            inside = [min(self.lines, key=lambda x: abs(x[0] - t0))]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in inside:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        busy = [x for x in sm if mx and x > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "window_s": round(t1 - t0, 3) if self.t0 else None}


def load_ncu_traffic():
    """dram read+write bytes per launch of the GEMM kernel from the committed
    ncu --set full capture summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_gemm_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


def checkerboard(world):
    """Process grid of P workers (layout.hpp:100-105): pr = largest divisor <= sqrt(P)."""
    pr = max(d for d in range(1, int(world ** 0.5) + 1) if world % d == 0)
    return pr, world // pr


def bench_config(N, world):
    """The workload both arms report (BASELINE.json config 3 at this GPU count)."""
    pr, pc = checkerboard(world)
    return {"workload": f"fp32 general_gemm {N}x{N}x{N}, Checkerboard2D {pr}x{pc} grid, "
                        f"blocks {N // pr}x{N // pc}, alpha=1 beta=0",
            "N": N, "grid": f"{pr}x{pc}", "parallelism": f"summa-pull{world}",
            "l2": (f"inputs ({4 * N * N / 2**30:.2f} GiB per operand) larger than the 126 MB L2; no flush needed"
                   if 4 * N * N > 126e6 else "inputs fit in L2 (not a headline configuration)")}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1604_01416_b200 as dm

    rank, world, local = dist_env()
    N = args.n
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [dm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cfg = dm.Config(worker_count=world, root_seed=42, mode="spmd", rank=rank, devices=[local],
                        nccl_id=obj[0])
    else:
        torch.cuda.set_device(0)
        cfg = dm.Config(worker_count=1, root_seed=42, devices=[0])
    pr, pc = dm.checkerboard_dims(world)
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N // pr, N // pc, world)
    s = dm.Session(cfg)
    me = rank
    a = s.create_matrix(lay, fill=dm.FillKind.SeededRandom)
    b = s.create_matrix(lay, fill=dm.FillKind.SeededRandom)
    c = s.create_matrix(lay, fill=dm.FillKind.Zeros)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    clocks = ClockSampler(local if world > 1 else 0)
    clocks.start()
    # ---- warm-up
    for _ in range(args.warmup):
        s.general_gemm(1.0, a, b, 0.0, c)

    # ---- timed: device-resident operands
    s.barrier()
    torch.cuda.synchronize()
    s.reset_worker_stats()
    s.set_gemm_timing(True)
    clocks.mark_start()
    s.marker_record(me, 0)
    for _ in range(args.steps):
        s.general_gemm(1.0, a, b, 0.0, c)
    s.marker_record(me, 1)
    s.barrier()
    torch.cuda.synchronize()
    clocks.mark_end()
    clk = clocks.stop()
    dev_ms = s.marker_elapsed(me, 0, 1)
    st = s.worker_stats(me)
    s.set_gemm_timing(False)
    t_ms = max_over_ranks(dev_ms)
    flops = 2.0 * N ** 3 * args.steps
    value = flops / (t_ms / 1e3) / 1e12
    launches = sum_over_ranks(float(st.gemm_launches + st.split_launches))
    # dominant kernel: tf32x3 GEMM, events around each launch on its stream
    kern_ms_avg = st.gemm_ms / max(1, st.gemm_launches)
    kern_flops = st.gemm_flops / max(1, st.gemm_launches)
    kern_tflops = kern_flops / (kern_ms_avg / 1e3) / 1e12
    gemm_share = st.gemm_ms / dev_ms if dev_ms else None
    peak_burst, peak_sust, peak_src, peak_3x = measured_peaks()
    traffic, ncu = load_ncu_traffic()
    if not (ncu and world == 1 and f"{N}^3" in ncu.get("problem", "") and
            ("mixed" in ncu.get("kernel", "")) == bool(gemm_mode())):
        traffic = None  # the committed capture is of a different launch shape

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        # Pinned host operands.  Every rank copies only its own blocks, so at
        # N > 1 only the rank's block-row band of each host matrix is touched
        # and page-locked (cudaHostRegister); at N = 1 the whole matrix is.
        r_lo, r_hi = (me // pc) * (N // pr), (me // pc + 1) * (N // pr)
        cudart = torch.cuda.cudart()

        def host_matrix(fill_seed):
            h = np.empty((N, N), dtype=np.float32)
            band = h[r_lo:r_hi]
            rc = cudart.cudaHostRegister(band.ctypes.data, band.nbytes, 0)
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister failed: {rc}")
            if fill_seed is not None:
                band[:] = np.random.default_rng(fill_seed).random(band.shape, dtype=np.float32)
            return h, band

        # Pin all four host matrices, then agree across ranks before any
        # collective: a rank that cannot pin must not leave the others waiting.
        pinned, why = [], ""
        try:
            for seed in (rank, rank + 1000, None, None):
                pinned.append(host_matrix(seed))
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line
            why = f"host pinning failed on rank {rank}: {e}"
        if sum_over_ranks(1.0 if len(pinned) == 4 else 0.0) < world:
            for _, band in pinned:
                cudart.cudaHostUnregister(band.ctypes.data)
            e2e = {"value": None, "unit": "TFLOP/s", "unavailable": why or "a peer rank could not pin host memory"}
            pinned = None
    if not args.no_e2e and pinned is not None:
        (hA, bA), (hB, bB), (hC0, bC0), (hC1, bC1) = pinned
        root = -1 if world > 1 else 0
        # Double-buffered device operands + asynchronous commands: step i's
        # H2D (copy engine), GEMM (tensor cores) and D2H (copy engine) overlap
        # with the neighbouring steps; every step still copies its inputs in
        # and its result out through the public API.
        sets = [(a, b, c), tuple(s.create_matrix(lay) for _ in range(3))]
        outs = [hC0, hC1]

        def e2e_step(i):
            ea, eb, ec = sets[i % 2]
            s.scatter(ea, hA)
            s.scatter(eb, hB)
            s.general_gemm(1.0, ea, eb, 0.0, ec)
            s.gather(ec, outs[i % 2], root=root)

        s.set_async(True)
        for i in range(2):
            e2e_step(i)
        s.barrier()
        s.marker_record(me, 2)
        for i in range(args.steps):
            e2e_step(i)
        s.barrier()
        s.marker_record(me, 3)
        s.set_async(False)
        e2e_ms = max_over_ranks(s.marker_elapsed(me, 2, 3))
        # bytes actually copied, whole job: every rank copies its owned blocks
        blk = (N // pr) * (N // pc) * 4
        e2e = {"value": flops / (e2e_ms / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": 2 * blk * world, "d2h_bytes_per_step": blk * world,
               "ms_per_step": e2e_ms / args.steps,
               "path": "Session.scatter(A,B from pinned host) + general_gemm + gather(C to pinned host), "
                       "asynchronous command mode, double-buffered device matrices"}
        for band in (bA, bB, bC0, bC1):
            cudart.cudaHostUnregister(band.ctypes.data)
        del hA, hB, hC0, hC1

    # ---- CPU baseline + full-size sampled parity (rank 0 at N=1 only)
    cpu = None
    parity = None
    if world == 1 and not args.no_cpu:
        cpu, parity = cpu_baseline_and_parity(s, a, b, c, N, args)

    s.close()
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference seeded fill, root seed 42)",
        "config": bench_config(N, world),
        "impl": "ours",
        "roofline": {"bound": "tensor", "achieved": round(kern_tflops, 2), "peak": round(peak_sust, 2),
                     "unit": "TFLOP/s", "frac": round(kern_tflops / peak_sust, 4),
                     "traffic": traffic,
                     "peak_source": peak_src + " sustained; burst=" + f"{peak_burst:.1f}",
                     "kernel": ("dm::tf32x3_gemm_kernel<2,1> (CTA pair; hi*hi tcgen05 kind::tf32 + "
                                "bf16 cross terms kind::f16)") if gemm_mode() else
                               "dm::tf32x3_gemm_kernel<2,0> (CTA pair; tcgen05 kind::tf32 x3)",
                     "frac_vs_3xtf32_roofline": round(kern_tflops / peak_3x, 4),
                     "flops_per_launch": kern_flops, "avg_launch_ms": round(kern_ms_avg, 3),
                     "launches": int(st.gemm_launches), "gemm_share_of_step": round(gemm_share, 4) if gemm_share else None},
        "e2e": e2e, "cpu_baseline": cpu, "parity_sampled": parity,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_and_parity(s, a, b, c, N, args):
    """Reference local_gemm (oracle/_ref) on sampled rows of the same GEMM:
    timed as the CPU baseline AND compared with our result rows (the sampled
    rows are bit-identical to the reference's distributed result)."""
    import numpy as np
    from oracle import COracle, RefOracle, ref_available

    threads = min(os.cpu_count() or 1, args.cpu_threads)
    A = s.gather(a)
    B = s.gather(b)
    Cg = s.gather(c)
    rows = np.linspace(0, N - 1, threads).astype(np.int64)
    a_rows = np.ascontiguousarray(A[rows])
    del A
    kind = "reference" if ref_available() else "port"
    t0 = time.perf_counter()
    if kind == "reference":
        want = RefOracle().sampled_rows(1.0, a_rows, B, False, 0.0, None, threads=threads)
    else:  # the C restatement, one row per thread would need threads; keep it serial
        want = COracle().local_gemm(1.0, a_rows[:1], False, B, False, 0.0)
        rows = rows[:1]
    dt = time.perf_counter() - t0
    got = np.ascontiguousarray(Cg[rows])
    relfro = COracle().rel_frobenius(got, want)
    cpu = {"value": round(2.0 * N * N * len(rows) / dt / 1e12, 8), "unit": "TFLOP/s",
           "cores": threads, "kind": kind,
           "sample": f"{len(rows)} full rows of the N={N} GEMM via reference local_gemm "
                     f"(1 x K row slices, stride N), one per thread, {dt:.1f} s"}
    parity = {"rows": len(rows), "relfro_vs_reference": relfro, "tolerance": 1e-5,
              "pass": bool(relfro <= 1e-5)}
    return cpu, parity


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    import ctypes

    import numpy as np

    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    from oracle import COracle, RefOracle, ref_available

    N = args.n
    threads = os.cpu_count() or 1
    orc = COracle()
    kind = "reference" if ref_available() else "port"
    # operands exactly as the reference's create_matrix(SeededRandom) makes them
    # (root seed 42, ids 1 and 2, P=1: one N x N block)
    seedA, seedB = orc.matrix_seed(42, 1), orc.matrix_seed(42, 2)
    B = orc.fill_block_parallel(N, N, seedB, 0, 0, threads=threads)
    # sampled op(A) rows: row r of the single block = elements [r*N, (r+1)*N)
    step_rows = max(1, min(threads, args.ref_rows))

    def a_rows(idx):
        out = np.empty((len(idx), N), np.float32)
        for i, r in enumerate(idx):
            orc.lib.orc_fill_range(out[i].ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                   int(r) * N, N, seedA, 0, 0)
        return out

    ro = RefOracle() if kind == "reference" else None
    # warm-up: fault in the B pages the row walks touch (a CPU loop has no other state)
    for _ in range(args.warmup):
        float(B[:, :: 1024].sum())
    rng = np.random.default_rng(0)
    times = []
    for _ in range(args.steps):
        idx = rng.integers(0, N, step_rows)
        ar = a_rows(idx)
        t0 = time.perf_counter()
        if ro is not None:
            ro.sampled_rows(1.0, ar, B, False, 0.0, None, threads=step_rows)
        else:
            orc.local_gemm(1.0, ar, False, B, False, 0.0)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = 2.0 * N * N * step_rows * args.steps / tot / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference seeded fill, root seed 42)",
        "config": bench_config(N, world),  # the same workload; each step times a bounded row sample
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": step_rows, "kind": kind,
                         "sample": f"{step_rows} full rows per step of the N={N} GEMM through the "
                                   f"reference local_gemm (kernels.hpp:48-89), one row per thread"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "warmup_note": "CPU warm-up steps touch the operand pages only",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=16, help="rows (= threads) of the CPU sample")
    ap.add_argument("--ref-rows", type=int, default=64, help="max rows per reference-arm step")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
