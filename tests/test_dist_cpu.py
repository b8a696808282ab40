"""World-size-2 gloo tests of the SPMD host logic (CPU only).

* NCCL unique-id bootstrap: rank 0's id reaches every rank intact;
* the GEMM data-movement plan is a pure function of the replicated layouts:
  every rank computes its own share, and the shares sum to the reference's
  transfer trace (tests/golden/golden.json 'plans');
* the SUMMA ingress of each rank is 2N^2 bytes on the 1x2 grid.
"""
import json
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import paper_1604_01416_b200 as dm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        obj = [dm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        out["id_ok"] = len(set(ids)) == 1 and len(ids[0]) == 128
    except dm.Error as e:  # NCCL bootstrap may need a network interface
        out["id_ok"] = f"skip: {e}"
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    mine = []
    for p in g["plans"]:
        la, lb, lc = (dm.make_layout(*x) for x in (p["la"], p["lb"], p["lc"]))
        P = p["la"][5]
        cnt = byt = 0
        for w in range(rank, P, world):  # this rank's share of the workers
            nb, by = dm.plan_general_gemm(la, p["ta"], lb, p["tb"], lc, w)
            cnt += nb
            byt += by
        mine.append((cnt, byt))
    shares = [None] * world
    dist.all_gather_object(shares, mine)
    totals = [(sum(s[i][0] for s in shares), sum(s[i][1] for s in shares)) for i in range(len(mine))]
    out["plans_ok"] = all(t == (p["transfers"], p["payload_bytes"]) for t, p in zip(totals, g["plans"]))
    N = 32768
    lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N, N // 2, 2)
    out["ingress"] = dm.plan_general_gemm(lay, False, lay, False, lay, rank)[1]
    q.put((rank, out))
    dist.destroy_process_group()


def test_gloo_world2():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r]["plans_ok"]
        assert res[r]["ingress"] == 2 * 32768 * 32768
        assert res[r]["id_ok"] is True or str(res[r]["id_ok"]).startswith("skip")
