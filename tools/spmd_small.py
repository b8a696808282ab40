"""BASELINE config 1 (2048^3, 2x2 checkerboard) and the FC 9216->4096 batch-256
commands in SPMD mode (one process per GPU, torchrun): wall time per
synchronous command on rank 0 (every rank issues its own launches; the
command ends with the coherence-digest all-gather)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

torch.cuda.set_device(local)
dist.init_process_group("gloo")


def session(**kw):
    obj = [dm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return dm.Session(dm.Config(worker_count=world, mode="spmd", rank=rank, devices=[local], nccl_id=obj[0],
                                root_seed=42, **kw))


def wall(s, fn, reps=int(os.environ.get("SMALL_REPS", "200"))):
    for _ in range(10):
        fn()
    s.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    s.barrier()
    return (time.perf_counter() - t0) / reps * 1e6


for coh in (True, False):
    s = session(coherence_checks=coh)
    n = 2048
    pr, pc = dm.checkerboard_dims(world)
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, n, n, n // pr, n // pc, world)
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    us = wall(s, lambda: s.general_gemm(1.0, a, b, 0.0, c))
    fin, fout, batch = 9216, 4096, 256
    strip = batch // world
    W = s.create_matrix(dm.make_layout(0, fin, fout, fin // world, fout, world), fill=dm.FillKind.SeededRandom)
    X = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, world), fill=dm.FillKind.SeededRandom)
    Y = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, world))
    dY = s.create_matrix(dm.make_layout(1, fout, batch, fout, strip, world), fill=dm.FillKind.SeededRandom)
    dX = s.create_matrix(dm.make_layout(1, fin, batch, fin, strip, world))
    dW = s.create_matrix(dm.make_layout(0, fin, fout, fin // world, fout, world))
    fwd = wall(s, lambda: s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True))
    bwd = wall(s, lambda: s.cached_backward_gemm(W, dY, dX))
    dw = wall(s, lambda: s.general_gemm(1.0, X, dY, 0.0, dW, False, True))
    if rank == 0:
        print(f"SPMD {world} ranks, coherence_checks={coh}: config1 {us:.1f} us/call; FC 9216->4096 fwd {fwd:.1f} "
              f"bwd {bwd:.1f} dW {dw:.1f} us/call", flush=True)
    s.close()
dist.destroy_process_group()
