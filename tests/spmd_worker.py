"""One rank of an SPMD (one process per GPU) parity run; launched by
tests/test_gpu_spmd.py through torch.distributed.run.  Every rank issues the
same calls in the same order (the reference's single global command order,
session.hpp:585-605); rank 0 checks results against the pinned oracle.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402
from oracle import COracle  # noqa: E402

GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    orc = COracle()
    results = {}

    def session(seed):
        # an NCCL unique id initialises exactly one communicator: fresh id per session
        obj = [dm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return dm.Session(dm.Config(worker_count=world, root_seed=seed, mode="spmd", rank=rank,
                                    devices=[local], nccl_id=obj[0]))

    # 1. checkerboard SUMMA-pull general_gemm, alpha/beta, all transposes
    s = session(42)
    pr, pc = dm.checkerboard_dims(world)
    n = 1536
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // pr, n // pc, world)
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    A, B, C0 = s.gather(a), s.gather(b), s.gather(c)   # root 0 assembles (others untouched)
    # default schedule, then the K-panel pipeline forced on at this small size:
    # copy-engine landing + stream flags + split warps fused into the GEMM
    forced = {"DM_PIPELINE_MIN_GFLOP": "0", "DM_PANEL_K": "512", "DM_FUSE_SPLIT": "2", "DM_PULL_CHUNK_MB": "1",
              "DM_PRESPLIT": "0"}
    # ... and the owner-split schedule: plane rectangles pulled from the owners'
    # IPC-mapped plane arenas (session_presplit.cpp), narrow panels
    presplit = {"DM_PIPELINE_MIN_GFLOP": "0", "DM_PRESPLIT": "1", "DM_PRESPLIT_PANEL": "256",
                "DM_F16X2_MIN_GFLOP": "0"}
    for tag, env in (("", {}), ("ce_", forced), ("ps_", presplit)):
        os.environ.update(env)
        for trans in range(4):
            ta, tb = bool(trans & 1), bool(trans & 2)
            s.general_gemm(1.5, a, b, -0.5, c, ta, tb)
            got = s.gather(c)
            if rank == 0:
                want = orc.local_gemm(1.5, A, ta, B, tb, -0.5, C0)
                results[f"general_{tag}t{trans}"] = orc.rel_frobenius(got, want)
                C0 = got  # next GEMM reads this C
            else:
                C0 = None
            st = s.worker_stats(rank)
            results[f"peer_bytes_{tag}r{rank}_t{trans}"] = int(st.peer_bytes_read)
            s.reset_worker_stats()
        for k in env:
            del os.environ[k]
    # inputs bit-exact with the reference's seeded fill (same layout, same ids)
    if rank == 0:
        results["A_bitexact"] = bool(A.tobytes() == orc.seeded_matrix(42, 1, 3, n, n, n // pr, n // pc).tobytes())
    # root=-1: every rank writes its own blocks
    own = np.zeros((n, n), np.float32)
    s.gather(a, own, root=-1)
    full = orc.seeded_matrix(42, 1, 3, n, n, n // pr, n // pc)
    mask = np.zeros((n, n), bool)
    for r in range(pr):
        for cc in range(pc):
            if lay.owner(r, cc) == rank:
                mask[r * (n // pr):(r + 1) * (n // pr), cc * (n // pc):(cc + 1) * (n // pc)] = True
    results[f"own_blocks_r{rank}"] = bool(np.array_equal(own[mask], full[mask]))
    s.close()

    # 2. golden sweep cases with this worker count (general + cyclic)
    cases = [g for g in GOLDEN["sweep"] if g["workers"] == world][:12]
    worst = 0.0
    for case in cases:
        s = session(case["root_seed"])
        ma = s.create_matrix(dm.make_layout(*case["la"]), fill=dm.FillKind.SeededRandom)
        mb = s.create_matrix(dm.make_layout(*case["lb"]), fill=dm.FillKind.SeededRandom)
        mc = s.create_matrix(dm.make_layout(*case["lc"]), fill=dm.FillKind.SeededRandom)
        A, B, C0 = s.gather(ma), s.gather(mb), s.gather(mc)
        if case["op"] == "general":
            s.general_gemm(case["alpha"], ma, mb, case["beta"], mc, case["ta"], case["tb"])
        else:
            s.cyclic_gemm(case["alpha"], ma, mb, case["beta"], mc, case["ta"], case["tb"], False)
        got = s.gather(mc)
        if rank == 0:
            assert f"{orc.fnv1a(A):016x}" == case["A"]
            want = orc.local_gemm(case["alpha"], A, case["ta"], B, case["tb"], case["beta"], C0)
            assert f"{orc.fnv1a(want):016x}" == case["C"]
            worst = max(worst, orc.rel_frobenius(got, want))
        s.close()
    results["sweep_cases"] = len(cases)
    results["sweep_worst"] = worst

    # 3. FC: cyclic fwd with cache, cached backward (zero peer bytes)
    s = session(3)
    fin, fout, batch = 96 * world, 64, 16 * world
    strip = batch // world
    W = s.create_matrix(dm.make_layout(0, fin, fout, fin // world, fout, world), fill=dm.FillKind.SeededRandom)
    X = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, world), fill=dm.FillKind.SeededRandom)
    Y = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, world))
    dY = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, world), fill=dm.FillKind.SeededRandom)
    dX = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, world))
    Wh, Xh, dYh = s.gather(W), s.gather(X), s.gather(dY)
    s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
    Yh = s.gather(Y)
    s.reset_worker_stats()
    s.cached_backward_gemm(W, dY, dX)
    results[f"bwd_peer_bytes_r{rank}"] = int(s.worker_stats(rank).peer_bytes_read)
    dXh = s.gather(dX)
    if rank == 0:
        results["fc_fwd"] = orc.rel_frobenius(Yh, orc.local_gemm(1.0, Wh, True, Xh, False, 0.0))
        results["fc_bwd"] = orc.rel_frobenius(dXh, orc.local_gemm(1.0, Wh, False, dYh, False, 0.0))
    s.close()

    # 4. SURVEY 8(f) ops over IPC: reshape (narrowing via exchange arenas),
    #    row/col sums, replication, checkpoint -- digests must equal the
    #    reference's (golden cases with this worker count)
    ok = True
    for c in [g for g in GOLDEN["reshape"] if g["workers"] == world][:6]:
        s = session(c["root_seed"])
        a = s.create_matrix(dm.make_layout(*c["src"], world), dm.Precision(c["src_prec"]), dm.FillKind.SeededRandom)
        b = s.reshape(a, dm.make_layout(*c["dst"], world), dm.Precision(c["dst_prec"]))
        got = s.gather(b)
        if rank == 0:
            ok &= f"{orc.fnv1a(got):016x}" == c["dst_fnv"]
        s.close()
    results["reshape_ok"] = ok
    ok = True
    for c in [g for g in GOLDEN["sums"] if g["workers"] == world][::5]:
        s = session(c["root_seed"])
        m = s.create_matrix(dm.make_layout(*c["layout"]), dm.Precision(c["precision"]), dm.FillKind.SeededRandom)
        o = s.add_row_col_sum(m, c["axis"], c["det"])
        got = s.gather(o)
        if rank == 0:
            ok &= f"{orc.fnv1a(got):016x}" == c["out_fnv"]
        s.close()
    results["sums_ok"] = ok
    s = session(71)
    m = s.create_matrix(dm.make_layout(3, 30, 22, 7, 6, world), fill=dm.FillKind.SeededRandom)
    s.replicate(m, True)
    full = s.gather(m)
    rd = s.replica_read(m, world - 1)
    at_reader = s.gather(m, root=world - 1)  # collective: every rank calls it
    results[f"replica_ok_r{rank}"] = bool(rank != world - 1 or rd.tobytes() == at_reader.tobytes())
    ck = os.path.join(ROOT, "gpurun_out", f"spmd_ck_{world}.dmth")
    os.makedirs(os.path.dirname(ck), exist_ok=True)
    s.checkpoint(ck)
    s.close()
    dist.barrier()
    obj = [dm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    r = dm.Session.restore(ck, dm.Config(mode="spmd", rank=rank, devices=[local], nccl_id=obj[0]))
    back = r.gather(m)
    if rank == 0:
        results["checkpoint_roundtrip"] = bool(back.tobytes() == full.tobytes())
    r.close()

    # 5. asynchronous command mode, K-panel pipeline forced: a GEMM output
    #    feeds the next GEMM as a peer operand, then is overwritten while
    #    peers may still be pulling its panels (write-after-read across ranks);
    #    owner-split: the next command's owner splits overwrite the plane
    #    arenas peers pulled from
    for tag, env in (("", forced), ("ps_", presplit)):
        os.environ.update(env)
        s = session(55)
        n = 1024
        lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // pr, n // pc, world)
        a, b, c, d, e = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(5))
        A, B, D = s.gather(a), s.gather(b), s.gather(d)
        s.set_async(True)
        for _ in range(2):
            s.general_gemm(1.0, a, b, 0.0, c)      # C1 = A B
            s.general_gemm(1.0, c, d, 0.0, e)      # E = C1 D: every rank pulls C1 panels
            s.general_gemm(-1.0, a, b, 0.0, c)     # overwrite C while those pulls may run
        s.barrier()
        s.set_async(False)
        Eg, Cg = s.gather(e), s.gather(c)
        if rank == 0:
            c1 = A.astype(np.float64) @ B.astype(np.float64)
            want_e = c1 @ D.astype(np.float64)
            results[f"async_chain_{tag}e"] = float(np.linalg.norm(Eg - want_e) / np.linalg.norm(want_e))
            results[f"async_chain_{tag}c"] = float(np.linalg.norm(Cg + c1) / np.linalg.norm(c1))
        # scatter right after a GEMM that read the operand: the overwrite must
        # not reach a peer still pulling the old blocks (consumer split) -- and
        # needs no cross-rank barrier when only the owner read them (presplit)
        rng = np.random.default_rng(7)
        A2 = (rng.random((n, n), dtype=np.float32) * 2 - 1).astype(np.float32)
        s.set_async(True)
        s.general_gemm(1.0, a, b, 0.0, c)      # reads A
        s.scatter(a, A2)                       # overwrites A
        s.general_gemm(1.0, a, b, 0.0, e)      # reads the new A
        s.barrier()
        s.set_async(False)
        Cg, Eg = s.gather(c), s.gather(e)
        if rank == 0:
            c1 = A.astype(np.float64) @ B.astype(np.float64)
            e1 = A2.astype(np.float64) @ B.astype(np.float64)
            results[f"async_scatter_{tag}c"] = float(np.linalg.norm(Cg - c1) / np.linalg.norm(c1))
            results[f"async_scatter_{tag}e"] = float(np.linalg.norm(Eg - e1) / np.linalg.norm(e1))
        s.close()
        for k in env:
            del os.environ[k]

    allres = [None] * world
    dist.all_gather_object(allres, results)
    if rank == 0:
        merged = {}
        for r in allres:
            merged.update(r)
        print("SPMD_RESULTS " + json.dumps(merged), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
