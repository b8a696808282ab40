"""The K-panel pipeline of general_gemm under every schedule it can take.

The distributed GEMM streams op(A)/op(B) in K panels (session.cpp run_gemm):
the first panel is split by its own kernels, later panels either by the
previous panel's GEMM launch (two fused split warps, DM_FUSE_SPLIT=1) or by
separate split kernels; pieces on another GPU land through copy engines first.
Whatever the schedule, the result must match the oracle within the
reference's fp32 bound (tests/acceptance.cpp:66-72: relFro <= 1e-5), with the
reference's transposes and alpha/beta (tests/test_dist_ops.cpp:136-147, 267-282).
"""
import numpy as np
import pytest

from paper_1604_01416_b200 import Config, FillKind, LayoutKind, Session, make_layout

pytestmark = pytest.mark.gpu
TOL = 1e-5


def relfro(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))


def ref_gemm(alpha, A, ta, B, tb, beta, C0):
    a, b = A.astype(np.float64), B.astype(np.float64)
    return alpha * ((a.T if ta else a) @ (b.T if tb else b)) + beta * C0.astype(np.float64)


@pytest.fixture(autouse=True)
def _pipeline_on(monkeypatch):
    # these sizes are below the work threshold that turns the K pipeline on
    monkeypatch.setenv("DM_PIPELINE_MIN_GFLOP", "0")
    # the consumer-split schedules (the owner-split one: test_gpu_presplit.py)
    monkeypatch.setenv("DM_PRESPLIT", "0")


def run_case(P, n, blk, trans, alpha=1.5, beta=-0.5, seed=77, devices=None, gemm_mode="default"):
    ta, tb = bool(trans & 1), bool(trans & 2)
    with Session(Config(worker_count=P, root_seed=seed + trans, devices=devices or [0] * P,
                        gemm_mode=gemm_mode)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, blk[0], blk[1], P)
        a, b, c = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        s.reset_worker_stats()
        s.general_gemm(alpha, a, b, beta, c, ta, tb)
        got = s.gather(c)
        splits = sum(s.worker_stats(w).split_launches for w in range(P))
        return relfro(got, ref_gemm(alpha, A, ta, B, tb, beta, C0)), splits


@pytest.mark.parametrize("gemm_mode", ["f16x2", "mixed", "3xtf32"])
@pytest.mark.parametrize("trans", [0, 1, 2, 3])
@pytest.mark.parametrize("lead", [0, 128])
def test_panels_fused_vs_separate(cuda, monkeypatch, trans, lead, gemm_mode):
    monkeypatch.setenv("DM_PANEL_K", "512")
    monkeypatch.setenv("DM_LEAD_PANEL_K", str(lead))
    res = {}
    for fuse in (2, 0):  # 2: fuse even where the GEMM is too short to hide it
        monkeypatch.setenv("DM_FUSE_SPLIT", str(fuse))
        res[fuse] = run_case(4, 1536, (768, 768), trans, gemm_mode=gemm_mode)
        assert res[fuse][0] <= TOL, (fuse, res[fuse])
    if gemm_mode == "f16x2":
        # the two-phase fused split (row maxima, grid handoff, split) needs all
        # CTAs of its launch co-resident: never fused while 4 workers share the GPU
        assert res[2][1] == res[0][1]
    else:
        # fused panels are split inside the GEMM launches: fewer split kernels
        assert res[2][1] < res[0][1]


@pytest.mark.parametrize("trans", [0, 1, 2, 3])
def test_f16x2_fused_two_phase_split(cuda, monkeypatch, trans):
    # one worker owning its GPU, geometric local panels: panels after the first
    # are split by the GEMM's split warps in two phases (fewer split kernels)
    monkeypatch.setenv("DM_PANEL_LOCAL", "256")
    res = {}
    for fuse in (2, 0):
        monkeypatch.setenv("DM_FUSE_SPLIT", str(fuse))
        res[fuse] = run_case(1, 1280, (1280, 1280), trans, gemm_mode="f16x2")
        assert res[fuse][0] <= TOL, (fuse, res[fuse])
    assert res[2][1] < res[0][1]


@pytest.mark.parametrize("trans", [0, 3])
def test_unaligned_pieces_fall_back(cuda, monkeypatch, trans):
    # odd block pitches (233 / 175 columns) are not 16-B aligned: the fused
    # split refuses them and the panel is split by its own kernels
    monkeypatch.setenv("DM_PANEL_K", "256")
    monkeypatch.setenv("DM_FUSE_SPLIT", "2")
    err, _ = run_case(3, 700, (233, 175), trans)
    assert err <= TOL


@pytest.mark.parametrize("trans", [0, 1, 2, 3])
def test_geometric_local_panels(cuda, monkeypatch, trans):
    # one worker, all operands local: geometric panels (lead 256, x3)
    monkeypatch.setenv("DM_PANEL_LOCAL", "256")
    monkeypatch.setenv("DM_FUSE_SPLIT", "2")
    err, _ = run_case(1, 1280, (1280, 1280), trans)
    assert err <= TOL


def test_beta_zero_ignores_garbage_c_across_panels(cuda, monkeypatch):
    # beta == 0 never reads C on the first panel (kernels.hpp:69-71); later
    # panels accumulate into the C the first one wrote
    monkeypatch.setenv("DM_PANEL_K", "512")
    n = 1024
    with Session(Config(worker_count=4, root_seed=3, devices=[0] * 4)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, 512, 512, 4)
        a, b = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(2))
        garbage = np.full((n, n), np.nan, np.float32)
        c = s.create_matrix(lay, fill=FillKind.FromHost, host=garbage)
        A, B = s.gather(a), s.gather(b)
        s.general_gemm(1.0, a, b, 0.0, c)
        got = s.gather(c)
        assert np.isfinite(got).all()
        assert relfro(got, A.astype(np.float64) @ B.astype(np.float64)) <= TOL


@pytest.mark.parametrize("trans", [0, 3])
def test_local_mode_across_gpus(cuda, monkeypatch, trans):
    """One process driving workers on different GPUs: remote pieces cross NVLink
    on copy engines into landing buffers, the split warps wait on the flag."""
    import torch
    ndev = torch.cuda.device_count()
    if ndev < 2:
        pytest.skip("needs >= 2 GPUs")
    P = 4
    monkeypatch.setenv("DM_PANEL_K", "512")
    for fuse, chunk in (("2", "0"), ("0", "0"), ("2", "1")):  # chunk 1 MiB: chunked first-panel pull
        monkeypatch.setenv("DM_FUSE_SPLIT", fuse)
        monkeypatch.setenv("DM_PULL_CHUNK_MB", chunk)
        err, _ = run_case(P, 1536, (768, 768), trans, devices=[w % ndev for w in range(P)])
        assert err <= TOL, (fuse, chunk)


def test_eight_workers_2x4_across_gpus(cuda, monkeypatch):
    """The 8-GPU grid (2x4 checkerboard) driven in LOCAL mode over the visible
    GPUs (two workers per GPU on a 4-GPU box): its pull plans, copy-engine
    landing and fused splits against the oracle."""
    import torch
    ndev = torch.cuda.device_count()
    if ndev < 2:
        pytest.skip("needs >= 2 GPUs")
    monkeypatch.setenv("DM_PANEL_K", "512")
    P, n = 8, 2048
    for trans in (0, 3):
        err, _ = run_case(P, n, (n // 2, n // 4), trans, devices=[w % ndev for w in range(P)])
        assert err <= TOL, trans


@pytest.mark.parametrize("devices", [[0] * 4, "all"])
def test_async_chain_write_after_read(cuda, monkeypatch, devices):
    """Asynchronous mode with the pipeline forced: C feeds the next GEMM as a
    peer operand and is then overwritten by a third GEMM.  The overwrite must
    wait for every worker's reads of the old C (pulls, fused splits) -- the
    reference's synchronous command order (session.hpp:585-605) as events."""
    import torch
    if devices == "all":
        n_dev = torch.cuda.device_count()
        if n_dev < 2:
            pytest.skip("needs >= 2 GPUs")
        devices = [w % n_dev for w in range(4)]
    monkeypatch.setenv("DM_PANEL_K", "512")
    monkeypatch.setenv("DM_FUSE_SPLIT", "2")
    monkeypatch.setenv("DM_PULL_CHUNK_MB", "1")
    n = 1024
    with Session(Config(worker_count=4, root_seed=55, devices=devices)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, 4)
        a, b, c, d, e = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(5))
        A, B, D = s.gather(a), s.gather(b), s.gather(d)
        s.set_async(True)
        s.general_gemm(1.0, a, b, 0.0, c)
        s.general_gemm(1.0, c, d, 0.0, e)
        s.general_gemm(-1.0, a, b, 0.0, c)
        s.barrier()
        s.set_async(False)
        c1 = A.astype(np.float64) @ B.astype(np.float64)
        assert relfro(s.gather(e), c1 @ D.astype(np.float64)) <= TOL
        assert relfro(s.gather(c), -c1) <= TOL
