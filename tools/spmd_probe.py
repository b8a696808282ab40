"""SPMD step probe (torchrun, one rank per GPU): device-timed ms per
N=32768 general_gemm on the checkerboard grid, synchronous commands vs the
asynchronous command mode, for configurations given as ENV=VAL[,ENV=VAL...]
arguments ("-" = defaults).  Rank 0 prints one line per configuration (max
over ranks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

N = int(os.environ.get("PROBE_N", "32768"))
steps = int(os.environ.get("PROBE_STEPS", "6"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def session():
    obj = [dm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = dm.Config(worker_count=world, mode="spmd", rank=rank, devices=[local], nccl_id=obj[0], root_seed=42)
    return dm.Session(cfg)


def vmax(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


pr, pc = dm.checkerboard_dims(world)
lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N // pr, N // pc, world)
for spec in sys.argv[1:] or ["-"]:
    env = dict(kv.split("=") for kv in spec.split(",")) if spec != "-" else {}
    os.environ.update(env)
    s = session()
    a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
    for asy in (False, True):
        s.set_async(asy)
        for _ in range(2):
            s.general_gemm(1.0, a, b, 0.0, c)
        s.barrier()
        torch.cuda.synchronize()
        s.set_gemm_timing(True)
        s.reset_worker_stats()
        s.marker_record(rank, 0)
        for _ in range(steps):
            s.general_gemm(1.0, a, b, 0.0, c)
        s.marker_record(rank, 1)
        s.barrier()
        torch.cuda.synchronize()
        ms = vmax(s.marker_elapsed(rank, 0, 1) / steps)
        st = s.worker_stats(rank)
        gms = vmax(st.gemm_ms / steps)
        s.set_gemm_timing(False)
        s.set_async(False)
        if rank == 0:
            tf = 2.0 * N ** 3 / ms / 1e9
            print(f"{spec:44s} {'async' if asy else 'sync ':5s} {ms:8.2f} ms/step ({tf:7.1f} TFLOP/s)  "
                  f"gemm {gms:7.2f} ms (max rank)", flush=True)
    s.close()
    for k in env:
        os.environ.pop(k, None)
dist.destroy_process_group()
