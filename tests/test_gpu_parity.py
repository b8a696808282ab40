"""GPU parity against the reference's own outputs (tests/golden/golden.json).

For every golden case: the device seeded fill + distribute/collect must be
BIT-EXACT with the reference (FNV digest of the gathered inputs), and the
tcgen05 3xTF32 result must sit within relFro <= 1e-5 of the reference's fp32
result (harness.hpp:114-125 tolerance).  The reference result is recomputed by
the pinned C restatement, whose digest must equal the golden one -- so the
chain GPU -> oracle -> reference is closed on every case.
"""
import json
import os

import numpy as np
import pytest

from oracle import COracle
from paper_1604_01416_b200 import (CacheMissError, Config, FillKind, PlanError, Session,
                                   ShapeError, UsageError, make_layout)

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
TOL = 1e-5


@pytest.fixture(scope="module")
def orc():
    return COracle()


def hx(v):
    return f"{v:016x}"


def run_case(orc, case):
    P = case["workers"]
    with Session(Config(worker_count=P, root_seed=case["root_seed"], devices=[0] * P)) as s:
        a = s.create_matrix(make_layout(*case["la"]), fill=FillKind.SeededRandom)
        b = s.create_matrix(make_layout(*case["lb"]), fill=FillKind.SeededRandom)
        c = s.create_matrix(make_layout(*case["lc"]), fill=FillKind.SeededRandom)
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        assert (hx(orc.fnv1a(A)), hx(orc.fnv1a(B)), hx(orc.fnv1a(C0))) == \
            (case["A"], case["B"], case["C0"]), "device fill / gather not bit-exact"
        if case["op"] == "general":
            s.general_gemm(case["alpha"], a, b, case["beta"], c, case["ta"], case["tb"])
        else:
            s.cyclic_gemm(case["alpha"], a, b, case["beta"], c, case["ta"], case["tb"], False)
        got = s.gather(c)
        assert s.descriptor(c).version == 1
    want = orc.local_gemm(case["alpha"], A, case["ta"], B, case["tb"], case["beta"], C0)
    assert hx(orc.fnv1a(want)) == case["C"]
    return orc.rel_frobenius(got, want)


@pytest.mark.parametrize("i", range(len(GOLDEN["sweep"])))
def test_sweep(cuda, orc, i):
    assert run_case(orc, GOLDEN["sweep"][i]) <= TOL


@pytest.mark.parametrize("idx", [0, 1])
def test_kat_256(cuda, orc, idx):
    k = GOLDEN["kat"][idx]
    with Session(Config(worker_count=4, root_seed=42, devices=[0] * 4)) as s:
        lay = make_layout(*k["layout"])
        a, b, c = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        assert hx(orc.fnv1a(A)) == k["A"]["fnv"]
        assert hx(orc.fnv1a(B)) == k["B"]["fnv"]
        assert hx(orc.fnv1a(C0)) == k["C0"]["fnv"]
        s.general_gemm(k["alpha"], a, b, k["beta"], c)
        got = s.gather(c)
    want = orc.local_gemm(k["alpha"], A, False, B, False, k["beta"], C0)
    assert hx(orc.fnv1a(want)) == k["C"]["fnv"]
    assert orc.rel_frobenius(got, want) <= TOL


def test_kat_2048_sampled(cuda, orc):
    """Config 1 (2048^3, 2x2): inputs bit-exact; 32 sampled rows of C against the
    reference arithmetic (row slices are bit-identical to the reference's
    distributed result); global sum against the reference's."""
    k = GOLDEN["kat"][2]
    with Session(Config(worker_count=4, root_seed=42, devices=[0] * 4)) as s:
        lay = make_layout(*k["layout"])
        a, b, c = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        assert hx(orc.fnv1a(A)) == k["A"]["fnv"] and hx(orc.fnv1a(B)) == k["B"]["fnv"]
        assert hx(orc.fnv1a(C0)) == k["C0"]["fnv"]
        s.general_gemm(1.0, a, b, 0.0, c)
        got = s.gather(c)
    rows = np.linspace(0, 2047, 32).astype(int)
    want = orc.local_gemm(1.0, A[rows], False, B, False, 0.0)
    assert orc.rel_frobenius(np.ascontiguousarray(got[rows]), want) <= TOL
    assert abs(got.astype(np.float64).sum() - k["C"]["sum"]) <= 1e-5 * np.abs(got).sum()


def test_fc_scenario(cuda, orc):
    fc = GOLDEN["fc"]
    P, fin, fout, batch = fc["workers"], fc["fin"], fc["fout"], fc["batch"]
    strip = batch // P
    with Session(Config(worker_count=P, root_seed=3, devices=[0] * P)) as s:
        W = s.create_matrix(make_layout(0, fin, fout, fin // P, fout, P), fill=FillKind.SeededRandom)
        X = s.create_matrix(make_layout(1, fin, batch, fin, strip, P), fill=FillKind.SeededRandom)
        Y = s.create_matrix(make_layout(1, fout, batch, fout, strip, P))
        dY = s.create_matrix(make_layout(1, fout, batch, fout, strip, P), fill=FillKind.SeededRandom)
        dX = s.create_matrix(make_layout(1, fin, batch, fin, strip, P))
        dW = s.create_matrix(make_layout(0, fin, fout, fin // P, fout, P))
        Wh, Xh, dYh = s.gather(W), s.gather(X), s.gather(dY)
        assert (hx(orc.fnv1a(Wh)), hx(orc.fnv1a(Xh)), hx(orc.fnv1a(dYh))) == (fc["W"], fc["X"], fc["dY"])
        with pytest.raises(CacheMissError):
            s.cached_backward_gemm(W, dY, dX)
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        s.reset_worker_stats()
        s.cached_backward_gemm(W, dY, dX)
        assert sum(s.worker_stats(w).peer_bytes_read for w in range(P)) == 0  # zero transfers
        s.general_gemm(1.0, X, dY, 0.0, dW, False, True)
        for mid, key, ref in ((Y, "Y", orc.local_gemm(1.0, Wh, True, Xh, False, 0.0)),
                              (dX, "dX", orc.local_gemm(1.0, Wh, False, dYh, False, 0.0)),
                              (dW, "dW", orc.local_gemm(1.0, Xh, False, dYh, True, 0.0))):
            assert hx(orc.fnv1a(ref)) == fc[key]
            assert orc.rel_frobenius(s.gather(mid), ref) <= TOL
        s.scatter(W, np.zeros((fin, fout), np.float32))
        with pytest.raises(CacheMissError):
            s.cached_backward_gemm(W, dY, dX)


def test_error_codes(cuda):
    """Same calls, same error classes as the reference (golden 'errors')."""
    with Session(Config(worker_count=2, root_seed=1, devices=[0, 0])) as s:
        lay = make_layout(3, 8, 8, 4, 4, 2)
        a, b = s.create_matrix(lay, fill=FillKind.SeededRandom), s.create_matrix(lay, fill=FillKind.SeededRandom)
        c = s.create_matrix(make_layout(3, 8, 9, 4, 4, 2), fill=FillKind.SeededRandom)
        with pytest.raises(UsageError):
            s.general_gemm(1.0, a, b, 0.0, a)
        with pytest.raises(ShapeError):
            s.general_gemm(1.0, a, b, 0.0, c)
        with pytest.raises(PlanError):
            s.cyclic_gemm(1.0, a, b, 0.0, s.create_matrix(lay, fill=FillKind.SeededRandom))
        with pytest.raises(UsageError):
            s.general_gemm(1.0, a, b, 0.0, 999)


def test_scatter_gather_roundtrip_bitwise(cuda):
    rng = np.random.default_rng(0)
    host = rng.standard_normal((300, 260)).astype(np.float32)
    host.view(np.uint32)[0, :4] = [0x7fc00001, 0x80000000, 0x00000001, 0x7f800000]  # NaN payload, -0, denormal, inf
    for P, kind in ((1, 3), (3, 0), (4, 2), (8, 3)):
        with Session(Config(worker_count=P, devices=[0] * P)) as s:
            m = s.create_matrix(make_layout(kind, 300, 260, 64, 96, P), fill=FillKind.FromHost, host=host)
            assert s.gather(m).tobytes() == host.tobytes()
