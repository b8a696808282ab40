"""Presplit GEMM commands (session_presplit.cpp): with the scaled fp16 pair,
a pipelined general_gemm has every OWNER split its own A / B blocks once into
its plane arena; consumers pull plane rectangles (the same bytes as the fp32
pieces of the reference's pull plan, ops.hpp:406-503) and never split.

Checked against the oracle within the reference's fp32 bound (relFro <= 1e-5,
tests/acceptance.cpp:66-72) with the reference's transposes and alpha/beta
(tests/test_dist_ops.cpp:136-147, 267-282), on the checkerboard grids of 2, 4
and 8 workers, ragged edge blocks, narrow panels (copies into panel buffers)
and wide ones (planes read in place from the owner's arena), plus the
schedule evidence: owner split launches only, and peer bytes equal to the
consumer-split schedule's (= the reference plan's).
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


def run_case(P, m, n, k, blk_a, blk_b, blk_c, trans, alpha=1.5, beta=-0.5, seed=91, devices=None,
             gemm_mode="f16x2"):
    ta, tb = bool(trans & 1), bool(trans & 2)
    with Session(Config(worker_count=P, root_seed=seed + trans, devices=devices or [0] * P,
                        gemm_mode=gemm_mode)) as s:
        ar, ac = (k, m) if ta else (m, k)
        br, bc = (n, k) if tb else (k, n)
        a = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, ar, ac, *blk_a, P), fill=FillKind.SeededRandom)
        b = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, br, bc, *blk_b, P), fill=FillKind.SeededRandom)
        c = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, m, n, *blk_c, P), fill=FillKind.SeededRandom)
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        s.reset_worker_stats()
        s.general_gemm(alpha, a, b, beta, c, ta, tb)
        got = s.gather(c)
        st = [s.worker_stats(w) for w in range(P)]
        return relfro(got, ref_gemm(alpha, A, ta, B, tb, beta, C0)), st


@pytest.mark.parametrize("trans", [0, 1, 2, 3])
@pytest.mark.parametrize("panel", [256, 8192])
def test_presplit_2x2_transposes(cuda, monkeypatch, trans, panel):
    monkeypatch.setenv("DM_PRESPLIT_PANEL", str(panel))
    n = 1536
    err, st = run_case(4, n, n, n, (768, 768), (768, 768), (768, 768), trans)
    assert err <= TOL, err
    # owner split only: partial maxima, whole-row maxima + split per owned A block and B block
    assert all(x.split_launches == 6 for x in st), [x.split_launches for x in st]


@pytest.mark.parametrize("trans", [0, 3])
def test_presplit_peer_bytes_match_consumer_split(cuda, monkeypatch, trans):
    n = 1536
    res = {}
    for ps in ("1", "0"):
        monkeypatch.setenv("DM_PRESPLIT", ps)
        monkeypatch.setenv("DM_PANEL_K", "512")
        err, st = run_case(4, n, n, n, (768, 768), (768, 768), (768, 768), trans)
        assert err <= TOL, (ps, err)
        res[ps] = [int(x.peer_bytes_read) for x in st]
    assert res["1"] == res["0"]
    if trans == 0:
        # 2x2 grid: each worker pulls the off-owner half of its A row band and B column band
        want = 4 * 768 * (n - 768) * 2
        assert res["1"] == [want] * 4


@pytest.mark.parametrize("trans", [0, 1, 2, 3])
def test_presplit_ragged_rectangular(cuda, monkeypatch, trans):
    # M x N x K = 1000 x 872 x 1304 with trimmed edge blocks; A, B, C blockings differ
    monkeypatch.setenv("DM_PRESPLIT_PANEL", "512")
    m, n, k = 1000, 872, 1304
    ba = (344, 448) if not (trans & 1) else (448, 344)
    bb = (448, 296) if not (trans & 2) else (296, 448)
    err, st = run_case(4, m, n, k, ba, bb, (504, 440), trans)
    assert err <= TOL, err


def test_presplit_eight_workers_2x4(cuda, monkeypatch):
    # the 8-GPU grid (2x4): A's K blocks (512) are narrower than B's (1024)
    for panel in ("8192", "256"):
        monkeypatch.setenv("DM_PRESPLIT_PANEL", panel)
        n = 2048
        for trans in (0, 3):
            err, st = run_case(8, n, n, n, (n // 2, n // 4), (n // 2, n // 4), (n // 2, n // 4), trans)
            assert err <= TOL, (panel, trans, err)
            assert all(x.split_launches == 6 for x in st)


def test_presplit_unaligned_blocks_fall_back(cuda, monkeypatch):
    # K blocks of 233 columns: plane rows would not start 16-B aligned, so the
    # command keeps the consumer split -- the same schedule as DM_PRESPLIT=0
    launches = {}
    for ps in ("1", "0"):
        monkeypatch.setenv("DM_PRESPLIT", ps)
        err, st = run_case(3, 700, 700, 700, (233, 233), (233, 233), (233, 233), 0)
        assert err <= TOL
        launches[ps] = [(x.split_launches, x.gemm_launches) for x in st]
    assert launches["1"] == launches["0"]


def test_presplit_not_for_other_split_modes(cuda, monkeypatch):
    n = 1024
    for mode in ("mixed", "3xtf32"):
        launches = {}
        for ps in ("1", "0"):
            monkeypatch.setenv("DM_PRESPLIT", ps)
            err, st = run_case(4, n, n, n, (512, 512), (512, 512), (512, 512), 0, gemm_mode=mode)
            assert err <= TOL
            launches[ps] = [(x.split_launches, x.gemm_launches) for x in st]
        assert launches["1"] == launches["0"], mode


def test_presplit_across_gpus(cuda, monkeypatch):
    """LOCAL mode over the visible GPUs: plane rectangles cross NVLink on the
    copy engines from the owners' arenas (2x2 and the 2x4 grid)."""
    import torch
    ndev = torch.cuda.device_count()
    if ndev < 2:
        pytest.skip("needs >= 2 GPUs")
    for P, n, blk in ((4, 1536, (768, 768)), (8, 2048, (1024, 512))):
        for panel in ("256", "8192"):
            monkeypatch.setenv("DM_PRESPLIT_PANEL", panel)
            for trans in (0, 3):
                err, st = run_case(P, n, n, n, blk, blk, blk, trans, devices=[w % ndev for w in range(P)])
                assert err <= TOL, (P, panel, trans, err)
                assert all(x.split_launches == 6 for x in st)


@pytest.mark.parametrize("devices", [[0] * 4, "all"])
def test_presplit_async_chain(cuda, monkeypatch, devices):
    """Asynchronous commands: the second GEMM's owner splits overwrite the
    plane arenas the first GEMM's pulls read, and C of the first feeds the
    second as an operand while the third overwrites it -- ordered by the
    plane-read events and the command barrier."""
    import torch
    if devices == "all":
        n_dev = torch.cuda.device_count()
        if n_dev < 2:
            pytest.skip("needs >= 2 GPUs")
        devices = [w % n_dev for w in range(4)]
    monkeypatch.setenv("DM_PRESPLIT_PANEL", "256")
    n = 1024
    with Session(Config(worker_count=4, root_seed=57, devices=devices, gemm_mode="f16x2")) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, 4)
        a, b, c, d, e = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(5))
        A, B, D = s.gather(a), s.gather(b), s.gather(d)
        s.set_async(True)
        for _ in range(2):
            s.general_gemm(1.0, a, b, 0.0, c)
            s.general_gemm(1.0, c, d, 0.0, e)
            s.general_gemm(-1.0, a, b, 0.0, c)
        s.barrier()
        s.set_async(False)
        c1 = A.astype(np.float64) @ B.astype(np.float64)
        assert relfro(s.gather(e), c1 @ D.astype(np.float64)) <= TOL
        assert relfro(s.gather(c), -c1) <= TOL


def test_presplit_matches_consumer_split(cuda, monkeypatch):
    """The owner splits scale every plane row by its WHOLE op row's maximum
    (partial maxima combined across the row band's owners), as a one-panel
    consumer split does: the two schedules differ only in how the K panels'
    sums are added into C (two launches vs one), so they agree far inside
    the fp32 bound."""
    n = 1024
    out = {}
    for ps in ("1", "0"):
        monkeypatch.setenv("DM_PRESPLIT", ps)
        monkeypatch.setenv("DM_PANEL_K", "0")  # consumer split: one panel
        with Session(Config(worker_count=4, root_seed=5, devices=[0] * 4, gemm_mode="f16x2")) as s:
            lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, 4)
            a, b, c = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
            A, B = s.gather(a), s.gather(b)
            s.reset_worker_stats()
            s.general_gemm(1.0, a, b, 0.0, c)
            out[ps] = (s.gather(c), [s.worker_stats(w).split_launches for w in range(4)])
    assert out["1"][1] == [6] * 4  # the presplit schedule ran
    want = A.astype(np.float64) @ B.astype(np.float64)
    assert relfro(out["1"][0], want) <= TOL and relfro(out["0"][0], want) <= TOL
    assert relfro(out["1"][0], out["0"][0]) <= 1e-6


def test_presplit_panels_span_blocks(cuda, monkeypatch):
    """K blocks of 256 (A) and 512 (B) under 1024-wide panels: every panel
    assembles its planes from several owners' blocks, whose rows share the
    whole-row scale."""
    monkeypatch.setenv("DM_PRESPLIT_PANEL", "1024")
    m = n = 1024
    k = 2048
    for trans in (0, 3):
        ba = (512, 256) if not (trans & 1) else (256, 512)
        bb = (512, 512)
        err, st = run_case(4, m, n, k, ba, bb, (512, 512), trans)
        assert err <= TOL, (trans, err)


@pytest.mark.parametrize("tb", [False, True])
def test_presplit_same_matrix_both_operands(cuda, monkeypatch, tb):
    """A * A^T (and A * A): one matrix is both operands, split once per role
    and orientation into the owners' arenas."""
    monkeypatch.setenv("DM_PRESPLIT_PANEL", "512")
    n = 1024
    with Session(Config(worker_count=4, root_seed=13, devices=[0] * 4, gemm_mode="f16x2")) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, 4)
        a = s.create_matrix(lay, fill=FillKind.SeededRandom)
        c = s.create_matrix(lay, fill=FillKind.SeededRandom)
        A, C0 = s.gather(a), s.gather(c)
        s.reset_worker_stats()
        s.general_gemm(0.75, a, a, 0.25, c, False, tb)
        got = s.gather(c)
        assert all(s.worker_stats(w).split_launches == 6 for w in range(4))
    assert relfro(got, ref_gemm(0.75, A, False, A, tb, 0.25, C0)) <= TOL


def test_presplit_panels_and_lead(cuda, monkeypatch):
    """The K panels the workers run (dm_presplit_panels: block edges, at least
    two) and the lead panel cut off the first panel of a worker whose every
    panel needs a pull (2x2: the off-diagonal workers) -- GEMM launch counts."""
    import paper_1604_01416_b200 as dm
    n = 4096
    assert dm.presplit_panels(n, n // 2, n // 2) == [0, 2048, 4096]
    monkeypatch.setenv("DM_PRESPLIT_LEAD", "512")
    err, st = run_case(4, n, n, n, (n // 2, n // 2), (n // 2, n // 2), (n // 2, n // 2), 0)
    assert err <= TOL
    # workers 0 and 3 own a whole local panel; 1 and 2 pull for every panel
    assert [x.gemm_launches for x in st] == [2, 3, 3, 2], [x.gemm_launches for x in st]
    monkeypatch.setenv("DM_PRESPLIT_LEAD", "0")
    err, st = run_case(4, n, n, n, (n // 2, n // 2), (n // 2, n // 2), (n // 2, n // 2), 0)
    assert err <= TOL
    assert [x.gemm_launches for x in st] == [2, 2, 2, 2]
