"""Device timeline of one distributed GEMM (DM_TRACE): per rank, when each K
panel's pull/split and GEMM ran, relative to the command start."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
path = os.path.join(os.environ.get("TRACE_DIR", tempfile.gettempdir()), f"dm_trace_{world}_{rank}.jsonl")
if os.path.exists(path):
    os.remove(path)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1604_01416_b200 as dm  # noqa: E402

N = int(os.environ.get("TRACE_N", "32768"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")
    obj = [dm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = dm.Config(worker_count=world, mode="spmd", rank=rank, devices=[local], nccl_id=obj[0], root_seed=42)
else:
    cfg = dm.Config(worker_count=1, devices=[0], root_seed=42)
pr, pc = dm.checkerboard_dims(world)
lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N // pr, N // pc, world)
s = dm.Session(cfg)
a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
s.general_gemm(1.0, a, b, 0.0, c)
os.environ["DM_TRACE"] = path
s.close()
s = dm.Session(cfg) if world == 1 else None
if world > 1:
    obj = [dm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg.nccl_id = obj[0]
    s = dm.Session(cfg)
a, b, c = (s.create_matrix(lay, fill=dm.FillKind.SeededRandom) for _ in range(3))
s.general_gemm(1.0, a, b, 0.0, c)
s.general_gemm(1.0, a, b, 0.0, c)
s.close()
recs = [json.loads(l) for l in open(path)]
last = max(r["cmd"] for r in recs)
lines = [f"rank {rank}/{world} N={N} (cmd {last}):"]
for r in recs:
    if r["cmd"] == last:
        lines.append(f"  {r['what']:11s} panel {r['panel']:2d}  {r['t0_ms']:8.3f} -> {r['t1_ms']:8.3f} ms"
                     f"  bytes={r['bytes'] / 2**20:8.1f} MiB  flops={r['flops']:.3g}")
print("\n".join(lines), flush=True)
