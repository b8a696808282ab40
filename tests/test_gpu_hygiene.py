"""Kernel hygiene without compute-sanitizer (closed on this GPU pool, see
profiles/r02/hygiene/README.md):

* races   -- every schedule of the tcgen05 GEMM (CTA group 1 / 2, split mode
             f16x2 / mixed / 3xTF32, split-K, producer lockstep over several
             waves, fused split warps reading flag-gated landing buffers, the
             f16x2 two-phase fused split with its grid handoff) is
             deterministic by construction (fixed MMA order, fixed-order
             split-K sums), so a smem / TMEM / mbarrier race shows up as run-
             to-run differences: each schedule is repeated and must be
             bitwise identical, and within 1e-5 of float64;
* bounds  -- the local_gemm seam writes C through a caller pitch: odd shapes
             inside a sentinel-filled frame must leave the frame, A and B
             untouched (epilogue, split-K reduce, edge tiles).
"""
import os

import numpy as np
import pytest

from paper_1604_01416_b200 import Config, LayoutKind, Session, make_layout

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SCHEDULES = [
    # name, workers, m, n, k, trans_b, env
    ("square", 1, 512, 512, 512, False, {}),
    ("splitK", 1, 256, 256, 4096, False, {"DM_LOCKSTEP": "0"}),
    ("lockstep", 1, 1024, 2560, 1024, False, {"DM_LOCKSTEP": "2"}),
    ("fused_split_P2", 2, 512, 512, 1024, True, {"DM_PIPELINE_MIN_GFLOP": "0", "DM_PANEL_K": "256",
                                                  "DM_FUSE_SPLIT": "1"}),
    # one worker, geometric local panels: f16x2's fused two-phase split (row
    # maxima, grid handoff, split) runs in the GEMM's split warps
    ("fused_local_P1", 1, 1024, 1024, 4096, False, {"DM_PANEL_LOCAL": "512", "DM_FUSE_SPLIT": "2"}),
]


@pytest.fixture
def env(monkeypatch):
    def set_env(d):
        for k, v in d.items():
            monkeypatch.setenv(k, v)
    return set_env


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("mode", ["mixed", "3xtf32", "f16x2"])
@pytest.mark.parametrize("sched", SCHEDULES, ids=[s[0] for s in SCHEDULES])
def test_schedule_repeats_bitwise(sched, mode, cg, env):
    name, workers, m, n, k, tb, extra = sched
    env({"DM_CTA_GROUP": str(cg), **extra})
    rng = np.random.default_rng(m + n + k + cg)
    A = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, k) if tb else (k, n)).astype(np.float32)
    C0 = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    ref = 1.5 * (A.astype(np.float64) @ (B.T if tb else B).astype(np.float64)) - 0.5 * C0.astype(np.float64)
    with Session(Config(worker_count=workers, root_seed=1, gemm_mode=mode, devices=[0] * workers)) as s:
        def mat(h):
            r, c = h.shape
            div = 2 if workers > 1 else 1
            mid = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, r, c, (r + div - 1) // div,
                                              (c + div - 1) // div, workers))
            s.scatter(mid, h)
            return mid
        a, b, c = mat(A), mat(B), mat(C0)
        outs = []
        for _ in range(6):
            s.scatter(c, C0)
            s.general_gemm(1.5, a, b, -0.5, c, trans_b=tb)
            outs.append(s.gather(c))
    first = outs[0]
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), first.view(np.uint32)), f"{name}: run-to-run difference"
    err = np.linalg.norm(first - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, err


SENTINEL = -7.25e30


@pytest.mark.parametrize("mode", ["f16x2", "3xtf32"])
@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("shape", [(300, 333, 200, 5), (64, 96, 8192, 3), (513, 257, 1000, 4)],
                         ids=["odd", "splitK_strip", "edge_tiles"])
def test_local_gemm_stays_inside_c(shape, cg, mode):
    import paper_1604_01416_b200 as dm
    m, n, k, pad = shape
    g = torch.Generator(device="cuda").manual_seed(m * n + k)
    a = torch.rand(m, k, device="cuda", generator=g) - 0.5
    b = torch.rand(k, n, device="cuda", generator=g) - 0.5
    a0, b0 = a.clone(), b.clone()
    ldc = n + 4 * pad  # pitch a multiple of 4 (vector epilogue) with a right margin
    frame = torch.full((m + pad, ldc), SENTINEL, device="cuda")
    c = frame[:m, :n]
    c.copy_(torch.rand(m, n, device="cuda", generator=g) - 0.5)
    c0 = c.clone()
    dm.local_gemm(1.25, a, False, b, False, 0.75, c, cta_group=cg, gemm_mode=mode)
    torch.cuda.synchronize()
    assert torch.all(frame[:m, n:] == SENTINEL), "wrote right of C"
    assert torch.all(frame[m:, :] == SENTINEL), "wrote below C"
    assert torch.equal(a, a0) and torch.equal(b, b0), "modified an operand"
    ref = 1.25 * (a0.double() @ b0.double()) + 0.75 * c0.double()
    err = float((c.double() - ref).norm() / ref.norm())
    assert err <= 1e-5, err
