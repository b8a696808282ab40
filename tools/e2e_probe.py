"""Where does an e2e step go at N GPUs?  Times (per rank, device markers) the
synchronous scatter, GEMM and gather separately, then the asynchronous
double-buffered loop.  Run under torch.distributed.run (or plain for N=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
N = int(os.environ.get("E2E_N", "32768"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")
    obj = [dm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = dm.Config(worker_count=world, mode="spmd", rank=rank, devices=[local], nccl_id=obj[0])
else:
    cfg = dm.Config(worker_count=1, devices=[0])
pr, pc = dm.checkerboard_dims(world)
lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N // pr, N // pc, world)
s = dm.Session(cfg)
sets = [[s.create_matrix(lay) for _ in range(3)] for _ in range(2)]
r_lo, r_hi = (rank // pc) * (N // pr), (rank // pc + 1) * (N // pr)
cudart = torch.cuda.cudart()
hosts = []
for _ in range(4):
    h = np.empty((N, N), np.float32)
    band = h[r_lo:r_hi]
    assert int(cudart.cudaHostRegister(band.ctypes.data, band.nbytes, 0)) == 0
    band[:] = np.random.default_rng(len(hosts)).random(band.shape, dtype=np.float32)
    hosts.append(h)
hA, hB, hC0, hC1 = hosts
root = -1 if world > 1 else 0


def timed(fn, reps=3):
    fn()
    s.barrier()
    s.marker_record(rank, 0)
    for _ in range(reps):
        fn()
    s.barrier()
    s.marker_record(rank, 1)
    return s.marker_elapsed(rank, 0, 1) / reps


a, b, c = sets[0]
t_h2d = timed(lambda: (s.scatter(a, hA), s.scatter(b, hB)))
t_gemm = timed(lambda: s.general_gemm(1.0, a, b, 0.0, c))
t_d2h = timed(lambda: s.gather(c, hC0, root=root))
t_sync = timed(lambda: (s.scatter(a, hA), s.scatter(b, hB), s.general_gemm(1.0, a, b, 0.0, c),
                        s.gather(c, hC0, root=root)))
outs = [hC0, hC1]
it = [0]


def astep():
    i = it[0]
    it[0] += 1
    ea, eb, ec = sets[i % 2]
    s.scatter(ea, hA)
    s.scatter(eb, hB)
    s.general_gemm(1.0, ea, eb, 0.0, ec)
    s.gather(ec, outs[i % 2], root=root)


s.set_async(True)
t_async = timed(astep, reps=4)
extra = ""
if os.environ.get("E2E_VARIANTS", "0") == "1":
    def step_no_gather():
        i = it[0]
        it[0] += 1
        ea, eb, ec = sets[i % 2]
        s.scatter(ea, hA)
        s.scatter(eb, hB)
        s.general_gemm(1.0, ea, eb, 0.0, ec)

    def step_no_scatter():
        i = it[0]
        it[0] += 1
        ea, eb, ec = sets[i % 2]
        s.general_gemm(1.0, ea, eb, 0.0, ec)
        s.gather(ec, outs[i % 2], root=root)

    def step_copies_only():
        i = it[0]
        it[0] += 1
        ea, eb, ec = sets[i % 2]
        s.scatter(ea, hA)
        s.scatter(eb, hB)
        s.gather(ec, outs[i % 2], root=root)
    extra = (f" async(no gather)={timed(step_no_gather, reps=4):.1f} async(no scatter)={timed(step_no_scatter, reps=4):.1f}"
             f" async(copies only)={timed(step_copies_only, reps=4):.1f}")
s.set_async(False)
print(f"rank {rank}/{world} N={N}: h2d(A,B)={t_h2d:.1f} gemm={t_gemm:.1f} d2h(C)={t_d2h:.1f} "
      f"sync_step={t_sync:.1f} async_step={t_async:.1f}{extra} ms", flush=True)
s.close()
