#!/usr/bin/env python
"""Distributed SGEMM benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 32768]

One step = one fp32 general_gemm C = A*B at N x N x N (default N=32768) on a
Checkerboard2D layout over the pr x pc process grid of the N GPUs (the
reference's checkerboard_dims, layout.hpp:100-105), operands resident in HBM,
synthetic inputs from the reference's seeded fill (root seed 42).  Total work
is fixed as N grows ("strong" scaling).  Rank 0 prints one JSON line.

--gpus N > 1 without torchrun: bench.py launches its own N ranks through
torch.distributed.run (one process per GPU, NCCL, 127.0.0.1); under torchrun
WORLD_SIZE must equal --gpus.  At every N the line carries sampled parity of
the timed result against the reference (16 full rows + 16 full columns spread
over every C block and tile), the reference CPU baseline, and a second timed
run of the north star's own 3xTF32 split beside the default f16x2 split
(3xTF32's 11+11-bit pair and three products, executed on fp16 MMAs).

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


# Useful-fp32-flop peak of each split-product scheme from the measured dense
# bf16 rate (TF32 runs at bf16/2); per useful k16 step:
#   3xTF32: 6 TF32 k8 MMAs           = 6 bf16-k16 slots -> peak = bf16 / 6
#   mixed : 2 TF32 k8 + 2 BF16 k16   = 4 bf16-k16 slots -> peak = bf16 / 4
#   f16x2 : 3 FP16 k16               = 3 bf16-k16 slots -> peak = bf16 / 3
SLOTS = {"mixed": 4.0, "3xtf32": 6.0, "f16x2": 3.0}
KERNELS = {
    "f16x2": "dm::tf32x3_gemm_kernel<2,3> (CTA pair; scaled 2xFP16 split, h1*h0 + h0*h1 + h0*h0 as tcgen05 "
             "kind::f16, power-of-two row scales undone in the epilogue)",
    "mixed": "dm::tf32x3_gemm_kernel<2,1> (CTA pair; hi*hi tcgen05 kind::tf32 + bf16 cross terms kind::f16)",
    "3xtf32": "dm::tf32x3_gemm_kernel<2,0> (CTA pair; tcgen05 kind::tf32 x3)",
}


def measured_peaks(mode: str):
    """(burst, sustained, source) useful-flop peak of `mode` in TFLOP/s."""
    div = SLOTS[mode]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"] / div, p["bf16_tflops_sustained"] / div, \
            f"measured bf16 dense (MEASURED_PEAKS.json) / {div:.0f}"
    except Exception:
        return 1590.0 / div, 1400.0 / div, f"fallback bf16 dense (B200_PROFILING.md) / {div:.0f}"


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


def load_ncu_traffic(N: int, world: int, mode: str):
    """DRAM read+write bytes per launch of the GEMM kernel from the committed
    ncu --set full capture of the same launch shape (profiles/ncu_gemm_summary*.json:
    N, grid size -- a P>1 capture is one rank's launch -- and split mode), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_gemm_summary*.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except Exception:
            continue
        if (d.get("N") == N and d.get("world", 1) == world and d.get("mode", "mixed") == mode
                and d.get("dram_bytes_per_launch")):
            return d["dram_bytes_per_launch"], os.path.relpath(path, ROOT)
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


def sample_indices(N: int, count: int, salt: int):
    """`count` indices spread over [0, N): one per equal slice, at a varying
    offset inside it, so the samples touch every block row/column of every
    grid up to 2x4 and different 256-wide tiles and lanes."""
    step = max(1, N // count)
    return [min(N - 1, i * step + (i * 131 + salt * 977 + 17) % step) for i in range(count)]


def spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: launch this script as N ranks (one per
    GPU) through torch.distributed.run; rank 0's JSON line passes through."""
    import socket
    try:
        import torch
        n_dev = torch.cuda.device_count()
    except Exception:
        n_dev = 0
    if n_dev < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {n_dev} CUDA devices are visible", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


# ------------------------------------------------------------------ our arm
class Timed:
    """One timed region of `steps` general_gemm commands on resident operands."""

    def __init__(self, s, me, world, max_over_ranks, sum_over_ranks):
        self.s, self.me, self.world = s, me, world
        self.max_over_ranks, self.sum_over_ranks = max_over_ranks, sum_over_ranks

    def run(self, a, b, c, N, steps, warmup, clocks=None):
        import torch
        s, me = self.s, self.me
        for _ in range(warmup):
            s.general_gemm(1.0, a, b, 0.0, c)
        s.barrier()
        torch.cuda.synchronize()
        s.reset_worker_stats()
        s.set_gemm_timing(True)
        if clocks:
            clocks.mark_start()
        s.marker_record(me, 0)
        for _ in range(steps):
            s.general_gemm(1.0, a, b, 0.0, c)
        s.marker_record(me, 1)
        s.barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.mark_end()
        dev_ms = s.marker_elapsed(me, 0, 1)
        st = s.worker_stats(me)
        s.set_gemm_timing(False)
        t_ms = self.max_over_ranks(dev_ms)
        flops = 2.0 * N ** 3 * steps
        kern_ms = st.gemm_ms / max(1, st.gemm_launches)
        kern_flops = st.gemm_flops / max(1, st.gemm_launches)
        return {"t_ms": t_ms, "value": flops / (t_ms / 1e3) / 1e12, "flops": flops,
                "kern_ms": kern_ms, "kern_flops": kern_flops,
                "kern_tflops": kern_flops / (kern_ms / 1e3) / 1e12 if kern_ms > 0 else 0.0,
                "gemm_share": st.gemm_ms / dev_ms if dev_ms else None,
                "gemm_launches": int(st.gemm_launches),
                "launches": int(self.sum_over_ranks(float(st.gemm_launches + st.split_launches)))}


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
    else:
        torch.cuda.set_device(0)

    def make_session(mode):
        if world > 1:
            obj = [dm.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            cfg = dm.Config(worker_count=world, root_seed=42, mode="spmd", rank=rank, devices=[local],
                            nccl_id=obj[0], gemm_mode=mode)
        else:
            cfg = dm.Config(worker_count=1, root_seed=42, devices=[0], gemm_mode=mode)
        return dm.Session(cfg)

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

    pr, pc = dm.checkerboard_dims(world)
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N // pr, N // pc, world)
    s = make_session(args.gemm_mode)
    session_mode = s.gemm_mode()
    mode = dm.split_mode_for(session_mode, N)  # the scheme this K runs in (auto: f16x2)
    me = rank
    a = s.create_matrix(lay, fill=dm.FillKind.SeededRandom)
    b = s.create_matrix(lay, fill=dm.FillKind.SeededRandom)
    c = s.create_matrix(lay, fill=dm.FillKind.Zeros)
    timer = Timed(s, me, world, max_over_ranks, sum_over_ranks)

    clocks = ClockSampler(local if world > 1 else 0)
    clocks.start()
    main = timer.run(a, b, c, N, args.steps, args.warmup, clocks)
    clk = clocks.stop()

    # ---- the timed result, collected on rank 0 for the sampled parity check
    held = None
    if not args.no_cpu:
        held = tuple(s.gather(m) for m in (a, b, c))  # root 0 assembles; other ranks take part
        if rank != 0:
            held = None

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(s, dm, np, torch, lay, (a, b, c), N, args, rank, world, me, pr, pc, sum_over_ranks,
                      max_over_ranks, main["flops"])
    s.close()

    # ---- the north star's own scheme beside it: the same workload in 3xTF32
    alt = None
    if not args.no_alt:
        alt_mode = "3xtf32" if mode != "3xtf32" else "f16x2"
        s2 = make_session(alt_mode)
        a2, b2 = (s2.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(2))
        c2 = s2.create_matrix(lay, fill=dm.FillKind.Zeros)
        steps2 = max(1, min(args.steps, args.alt_steps))
        r2 = Timed(s2, me, world, max_over_ranks, sum_over_ranks).run(a2, b2, c2, N, steps2, min(args.warmup, 3))
        held2 = s2.gather(c2) if not args.no_cpu else None  # collective: every rank takes part
        s2.close()
        b2_burst, b2_sust, b2_src = measured_peaks(alt_mode)
        alt = {"gemm_mode": alt_mode, "value": round(r2["value"], 3), "unit": "TFLOP/s", "steps": steps2,
               "ms_per_step": round(r2["t_ms"] / steps2, 3),
               "kernel_tflops": round(r2["kern_tflops"], 2),
               "frac_of_its_roofline": round(r2["kern_tflops"] / b2_sust, 4),
               "roofline_peak": round(b2_sust, 2), "peak_source": b2_src + " sustained",
               "frac_vs_3xtf32_roofline": round(r2["kern_tflops"] / measured_peaks("3xtf32")[1], 4),
               "gemm_share_of_step": round(r2["gemm_share"], 4) if r2["gemm_share"] else None}
        if rank == 0 and held2 is not None:
            alt["_c"] = held2
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return

    # ---- rank 0: sampled parity (rows + columns) and the CPU reference baseline
    cpu, parity = None, None
    if held is not None:
        A, B, Cg = held
        cpu, parity = cpu_baseline_and_parity(A, B, Cg, N, args, alt.pop("_c", None) if alt else None,
                                              alt["gemm_mode"] if alt else None)
        if alt is not None and parity is not None and "alt" in parity:
            alt["parity_sampled"] = parity.pop("alt")
        del A, B, Cg, held
    if alt is not None:
        alt.pop("_c", None)

    peak_burst, peak_sust, peak_src = measured_peaks(mode)
    peak_3x = measured_peaks("3xtf32")[1]
    traffic, traffic_src = load_ncu_traffic(N, world, mode)
    kernel = KERNELS[mode]
    line = {
        "metric": METRIC, "value": round(main["value"], 3), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(main["t_ms"] / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference seeded fill, root seed 42)",
        "config": dict(bench_config(N, world), gemm_mode=mode, session_gemm_mode=session_mode),
        "impl": "ours",
        "roofline": {"bound": "tensor", "achieved": round(main["kern_tflops"], 2), "peak": round(peak_sust, 2),
                     "unit": "TFLOP/s", "frac": round(main["kern_tflops"] / peak_sust, 4),
                     "frac_basis": (f"executed-mix roofline: the {mode} split's own useful-flop peak "
                                    f"(bf16 dense / {SLOTS[mode]:.0f}), per GPU, on that GPU's GEMM launches"),
                     "frac_vs_3xtf32_roofline": round(main["kern_tflops"] / peak_3x, 4),
                     "roofline_3xtf32_peak": round(peak_3x, 2),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src + f" sustained; burst={peak_burst:.1f}",
                     "kernel": kernel, "flops_per_launch": main["kern_flops"],
                     "avg_launch_ms": round(main["kern_ms"], 3), "launches": main["gemm_launches"],
                     "gemm_share_of_step": round(main["gemm_share"], 4) if main["gemm_share"] else None},
        "e2e": e2e, "cpu_baseline": cpu, "parity_sampled": parity,
        "alt_split": alt,
        "gpu_launches": main["launches"],
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def run_e2e(s, dm, np, torch, lay, mats, N, args, rank, world, me, pr, pc, sum_over_ranks, max_over_ranks,
            flops):
    """The same metric through the public API with host buffers: every step
    scatters A and B from pinned host memory, multiplies, and gathers C back."""
    a, b, c = mats
    # Every rank copies only its own blocks, so at N > 1 only the rank's
    # block-row band of each host matrix is touched and page-locked
    # (cudaHostRegister); at N = 1 the whole matrix is.
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
        return {"value": None, "unit": "TFLOP/s", "unavailable": why or "a peer rank could not pin host memory"}
    (hA, bA), (hB, bB), (hC0, bC0), (hC1, bC1) = pinned
    root = -1 if world > 1 else 0
    # Double-buffered device operands + asynchronous commands: step i's H2D
    # (copy engine), GEMM (tensor cores) and D2H (copy engine) overlap with the
    # neighbouring steps; every step still copies its inputs in and its result
    # out through the public API.
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
    blk = (N // pr) * (N // pc) * 4  # bytes actually copied, whole job: every rank its owned blocks
    for band in (bA, bB, bC0, bC1):
        cudart.cudaHostUnregister(band.ctypes.data)
    return {"value": flops / (e2e_ms / 1e3) / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": 2 * blk * world, "d2h_bytes_per_step": blk * world,
            "ms_per_step": e2e_ms / args.steps,
            "path": "Session.scatter(A,B from pinned host) + general_gemm + gather(C to pinned host), "
                    "asynchronous command mode, double-buffered device matrices"}


def cpu_baseline_and_parity(A, B, Cg, N, args, C_alt=None, alt_mode=None):
    """The reference's local_gemm (oracle/_ref) on 16 full rows and 16 full
    columns of the same GEMM: the rows are timed as the CPU baseline, and both
    are compared with the timed GPU result.  A sampled row (column) of the
    reference's distributed result equals its local_gemm on that 1 x K row
    (K x 1 column) bit for bit (k ascending over the full K in every
    executor, ops.hpp:274, 485), so this is parity against the reference's
    own output for those elements.  Also reports both sides' error against an
    fp64 product of the same inputs."""
    import numpy as np
    from oracle import COracle, RefOracle, ref_available

    threads = min(os.cpu_count() or 1, args.cpu_threads)
    rows = sample_indices(N, args.sample_rows, 1)
    cols = sample_indices(N, args.sample_cols, 2)
    a_rows = np.ascontiguousarray(A[rows])
    b_cols = np.ascontiguousarray(B[:, cols].T)
    kind = "reference" if ref_available() else "port"
    t0 = time.perf_counter()
    if kind == "reference":
        ro = RefOracle()
        want_r = ro.sampled_rows(1.0, a_rows, B, False, 0.0, None, threads=threads)
        dt_rows = time.perf_counter() - t0
        t1 = time.perf_counter()
        want_c = ro.sampled_cols(1.0, A, False, b_cols, 0.0, None, threads=threads)
        dt_cols = time.perf_counter() - t1
    else:  # the C restatement (serial): one row, no columns
        rows = rows[:1]
        want_r = COracle().local_gemm(1.0, a_rows[:1], False, B, False, 0.0)
        dt_rows = time.perf_counter() - t0
        cols, want_c, dt_cols = [], np.zeros((0, N), np.float32), 0.0
    got_r = np.ascontiguousarray(Cg[rows])
    got_c = np.ascontiguousarray(Cg[:, cols].T)
    orc = COracle()
    rel_r = orc.rel_frobenius(got_r, want_r)
    rel_c = orc.rel_frobenius(got_c, want_c) if len(cols) else 0.0
    got_all = np.concatenate([got_r.ravel(), got_c.ravel()])
    want_all = np.concatenate([want_r.ravel(), want_c.ravel()])
    rel = orc.rel_frobenius(got_all, want_all)
    # fp64 products of the same samples: how far each side is from exact
    exact = np.concatenate([(a_rows[:len(rows)].astype(np.float64) @ B.astype(np.float64)).ravel(),
                            (A.astype(np.float64) @ b_cols.T.astype(np.float64)).T.ravel()]) \
        if len(cols) else (a_rows[:1].astype(np.float64) @ B.astype(np.float64)).ravel()

    def rel64(x):
        return float(np.linalg.norm(x.astype(np.float64) - exact) / np.linalg.norm(exact))
    cpu = {"value": round(2.0 * N * N * len(rows) / dt_rows / 1e12, 8), "unit": "TFLOP/s",
           "cores": threads, "kind": kind,
           "sample": f"{len(rows)} full rows of the N={N} GEMM via reference local_gemm (1 x K row slices, "
                     f"stride N), one per thread: {dt_rows:.1f} s; plus {len(cols)} full columns for parity "
                     f"({dt_cols:.1f} s, not timed into the value)"}
    parity = {"rows": len(rows), "cols": len(cols), "row_indices": rows, "col_indices": cols,
              "relfro_vs_reference": rel, "relfro_rows": rel_r, "relfro_cols": rel_c, "tolerance": 1e-5,
              "pass": bool(rel <= 1e-5),
              "relfro_vs_fp64": {"gpu": rel64(got_all), "reference": rel64(want_all)}}
    if C_alt is not None:
        alt_all = np.concatenate([np.ascontiguousarray(C_alt[rows]).ravel(),
                                  np.ascontiguousarray(C_alt[:, cols].T).ravel()])
        ra = orc.rel_frobenius(alt_all, want_all)
        parity["alt"] = {"gemm_mode": alt_mode, "relfro_vs_reference": ra, "pass": bool(ra <= 1e-5),
                         "relfro_vs_fp64": rel64(alt_all), "rows": len(rows), "cols": len(cols)}
    return cpu, parity


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    import ctypes

    import numpy as np

    rank, _, _ = dist_env()
    world = args.gpus  # the arm reports the workload of the N-GPU run it stands beside
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
    ap.add_argument("--gemm-mode", choices=["default", "auto", "f16x2", "mixed", "3xtf32"], default="default",
                    help="split-product scheme of the headline run (default: DM_GEMM_MODE, else auto = "
                         "f16x2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline and sampled parity")
    ap.add_argument("--no-alt", action="store_true", help="skip the second (3xTF32) timed run")
    ap.add_argument("--alt-steps", type=int, default=10, help="max timed steps of the second run")
    ap.add_argument("--cpu-threads", type=int, default=16, help="host threads of the CPU reference")
    ap.add_argument("--sample-rows", type=int, default=16)
    ap.add_argument("--sample-cols", type=int, default=16)
    ap.add_argument("--ref-rows", type=int, default=64, help="max rows per reference-arm step")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    launched = "WORLD_SIZE" in os.environ
    if launched and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but torchrun started WORLD_SIZE={os.environ['WORLD_SIZE']} ranks",
              file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    elif not launched and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
