"""GPU parity of the SURVEY 8(f) operations against the reference's own outputs
(tests/golden/golden.json, tests/golden/ref_checkpoint.dmth):

* seeded fills at Half16 / Single32 / Double64: bit-exact;
* reshape with narrowing before the link / widening at the receiver: bit-exact;
* add_row_col_sum, deterministic and salted fast mode: bit-exact (same fold order);
* replicate + lazy version-checked replica_read: bit-exact, same descriptor effects;
* update_block: bit-exact, version bump;
* Half16 GEMM (fp32 compute, one rounding on store): within 1 half ulp;
* DMTH checkpoint: the reference's file restores bit-exactly, and the same
  session state checkpoints to a byte-identical file.
"""
import json
import os

import numpy as np
import pytest

from paper_1604_01416_b200 import (Config, FillKind, IntegrityError, Precision, Session,
                                   make_layout)

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def fnv(arr):
    from oracle import COracle
    return f"{COracle().fnv1a(np.ascontiguousarray(arr)):016x}"


def session(P, seed):
    return Session(Config(worker_count=P, root_seed=seed, devices=[0] * P))


@pytest.mark.parametrize("i", range(len(GOLDEN["fills_p"])))
def test_fill_precisions(cuda, i):
    f = GOLDEN["fills_p"][i]
    with session(f["layout"][5], f["root_seed"]) as s:
        m = s.create_matrix(make_layout(*f["layout"]), Precision(f["precision"]), FillKind.SeededRandom)
        assert fnv(s.gather(m)) == f["fnv"]


@pytest.mark.parametrize("i", range(len(GOLDEN["reshape"])))
def test_reshape(cuda, i):
    c = GOLDEN["reshape"][i]
    P = c["workers"]
    with session(P, c["root_seed"]) as s:
        a = s.create_matrix(make_layout(*c["src"], P), Precision(c["src_prec"]), FillKind.SeededRandom)
        assert fnv(s.gather(a)) == c["src_fnv"]
        b = s.reshape(a, make_layout(*c["dst"], P), Precision(c["dst_prec"]))
        assert b == c["dst_id"]
        assert fnv(s.gather(b)) == c["dst_fnv"]


@pytest.mark.parametrize("i", range(0, len(GOLDEN["sums"]), 3))
def test_row_col_sums(cuda, i):
    c = GOLDEN["sums"][i]
    with session(c["workers"], c["root_seed"]) as s:
        m = s.create_matrix(make_layout(*c["layout"]), Precision(c["precision"]), FillKind.SeededRandom)
        assert fnv(s.gather(m)) == c["in_fnv"]
        o = s.add_row_col_sum(m, c["axis"], c["det"])
        o2 = s.add_row_col_sum(m, c["axis"], c["det"])
        assert o == c["out_id"]
        assert s.descriptor(o).layout.to_string() == c["out_layout"]
        assert fnv(s.gather(o)) == c["out_fnv"]
        assert fnv(s.gather(o2)) == c["out2_fnv"]


@pytest.mark.parametrize("i", range(len(GOLDEN["replication"])))
def test_replication(cuda, i):
    c = GOLDEN["replication"][i]
    P = c["workers"]
    with session(P, c["root_seed"]) as s:
        m = s.create_matrix(make_layout(*c["layout"]), fill=FillKind.SeededRandom)
        s.replicate(m, True)
        d = s.descriptor(m)
        assert [d.version, d.replica_version, d.replicated] == c["desc_after_enable"]
        assert fnv(s.replica_read(m, P - 1)) == c["read0_fnv"]
        s.scatter(m, (np.arange(30 * 22, dtype=np.float32).reshape(30, 22) / 7.0).astype(np.float32))
        d = s.descriptor(m)
        assert [d.version, d.replica_version, d.replicated] == c["desc_after_scatter"]
        assert fnv(s.replica_read(m, 0)) == c["read1_fnv"]
        d = s.descriptor(m)
        assert [d.version, d.replica_version, d.replicated] == c["desc_after_read"]


def test_fresh_replicas_feed_gemm(cuda):
    """A replicated operand is read from local replicas: zero peer bytes."""
    P = 4
    with session(P, 5) as s:
        lay = make_layout(3, 64, 64, 32, 32, P)
        a, b, c = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
        s.replicate(a, True)
        s.replicate(b, True)
        s.reset_worker_stats()
        s.general_gemm(1.0, a, b, 0.0, c)
        assert sum(s.worker_stats(w).peer_bytes_read for w in range(P)) == 0


def test_update_block(cuda):
    c = GOLDEN["update_block"][0]
    with session(c["workers"], c["root_seed"]) as s:
        m = s.create_matrix(make_layout(*c["layout"]), fill=FillKind.SeededRandom)
        s.update_block(m, *c["block"], np.linspace(-3, 3, 20 * 7, dtype=np.float32).reshape(20, 7))
        assert s.descriptor(m).version == c["version"]
        assert fnv(s.gather(m)) == c["fnv"]


@pytest.mark.parametrize("i", range(len(GOLDEN["half_gemm"])))
def test_half_gemm(cuda, i):
    from oracle import RefOracle, ref_available
    c = GOLDEN["half_gemm"][i]
    P = c["workers"]
    with session(P, c["root_seed"]) as s:
        a = s.create_matrix(make_layout(3, 40, 40, 16, 12, P), Precision.Half16, FillKind.SeededRandom)
        b = s.create_matrix(make_layout(0, 40, 40, 10, 40, P), Precision.Half16, FillKind.SeededRandom)
        cm = s.create_matrix(make_layout(2, 40, 40, 9, 40, P), Precision.Half16, FillKind.SeededRandom)
        A, B, C0 = s.gather(a), s.gather(b), s.gather(cm)
        assert (fnv(A), fnv(B), fnv(C0)) == (c["A"], c["B"], c["C0"])
        s.general_gemm(1.5, a, b, -0.5, cm, c["ta"], c["tb"])
        got = s.gather(cm)
    if not ref_available():
        pytest.skip("oracle/_ref not shipped")
    ro = RefOracle()
    with ro.session(P, c["root_seed"]) as rs:
        ra = rs.create_p(3, 40, 40, 16, 12, P, 0)
        rb = rs.create_p(0, 40, 40, 10, 40, P, 0)
        rc = rs.create_p(2, 40, 40, 9, 40, P, 0)
        rs.general_gemm(1.5, ra, rb, -0.5, rc, c["ta"], c["tb"])
        want = rs.gather_p(rc)
    assert fnv(want) == c["C"]
    ulp = np.abs(got.view(np.int16).astype(np.int32) - want.view(np.int16).astype(np.int32))
    assert ulp.max() <= 1 and (ulp == 0).mean() > 0.9


@pytest.mark.parametrize("P", [1, 2])
def test_half_gemm_long_k(cuda, P):
    """Half16 GEMM with few C tiles and a long K: split-K work items whose fp32
    partials are summed in fixed order and rounded to half once (AccumOf<Half>,
    kernels.hpp:29-35) -- within one half ulp of the reference."""
    from oracle import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not shipped")
    m, n, k = 128, 96, 4096
    with session(P, 77) as s:
        a = s.create_matrix(make_layout(0, m, k, m // P, k, P), Precision.Half16, FillKind.SeededRandom)
        b = s.create_matrix(make_layout(1, k, n, k, n // P, P), Precision.Half16, FillKind.SeededRandom)
        cm = s.create_matrix(make_layout(0, m, n, m // P, n, P), Precision.Half16, FillKind.SeededRandom)
        s.general_gemm(1.5, a, b, -0.5, cm, False, False)
        got = s.gather(cm)
    with RefOracle().session(P, 77) as rs:
        ra = rs.create_p(0, m, k, m // P, k, P, 0)
        rb = rs.create_p(1, k, n, k, n // P, P, 0)
        rc = rs.create_p(0, m, n, m // P, n, P, 0)
        A, B, C0 = rs.gather_p(ra), rs.gather_p(rb), rs.gather_p(rc)
        rs.general_gemm(1.5, ra, rb, -0.5, rc, False, False)
        want = rs.gather_p(rc)
    exact = 1.5 * (A.astype(np.float64) @ B.astype(np.float64)) - 0.5 * C0.astype(np.float64)

    def rel(x):
        return np.linalg.norm(x.astype(np.float64) - exact) / np.linalg.norm(exact)
    # near-zero outputs differ by many half ulps between any two fp32 summation
    # orders over K=4096; the bar is "no less accurate than the reference"
    assert rel(got) <= 1.5 * rel(want) + 1e-6
    assert (got.view(np.int16) == want.view(np.int16)).mean() > 0.8


@pytest.mark.parametrize("P", [1, 3])
@pytest.mark.parametrize("trans", [0, 1, 2, 3])
def test_double_gemm_bitexact(cuda, P, trans):
    """Double64 GEMMs reproduce the reference bit for bit: same k-ascending,
    unfused accumulation per output (kernels.hpp:48-75; the reference's fp64
    bar, tests/acceptance.cpp:61-65, tests/test_dist_ops.cpp:63-70)."""
    from oracle import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not shipped")
    ta, tb = bool(trans & 1), bool(trans & 2)
    la, lb, lc = (3, 72, 72, 24, 20), (0, 72, 72, 17, 72), (2, 72, 72, 9, 72)
    for alpha, beta in ((1.0, 0.0), (1.5, -0.5)):
        with session(P, 31 + trans) as s:
            a = s.create_matrix(make_layout(*la, P), Precision.Double64, FillKind.SeededRandom)
            b = s.create_matrix(make_layout(*lb, P), Precision.Double64, FillKind.SeededRandom)
            c = s.create_matrix(make_layout(*lc, P), Precision.Double64, FillKind.SeededRandom)
            s.general_gemm(alpha, a, b, beta, c, ta, tb)
            got = s.gather(c)
        with RefOracle().session(P, 31 + trans) as rs:
            ra, rb, rc = (rs.create_p(*l, P, 2) for l in (la, lb, lc))
            rs.general_gemm(alpha, ra, rb, beta, rc, ta, tb)
            want = rs.gather_p(rc)
        assert got.tobytes() == want.tobytes(), (alpha, beta)


def test_double_cyclic_and_cached_backward_bitexact(cuda):
    from oracle import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not shipped")
    P, fin, fout, batch = 3, 48, 40, 24
    lw, lx, ly, ldy, ldx = ((0, fin, fout, fin // P, fout), (1, fin, batch, fin, batch // P),
                            (1, fout, batch, fout, batch // P), (1, fout, batch, fout, batch // P),
                            (1, fin, batch, fin, batch // P))
    with session(P, 8) as s:
        W, X, Y, dY, dX = (s.create_matrix(make_layout(*l, P), Precision.Double64, FillKind.SeededRandom)
                           for l in (lw, lx, ly, ldy, ldx))
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        s.cached_backward_gemm(W, dY, dX)
        got_y, got_dx = s.gather(Y), s.gather(dX)
    with RefOracle().session(P, 8) as rs:
        rW, rX, rY, rdY, rdX = (rs.create_p(*l, P, 2) for l in (lw, lx, ly, ldy, ldx))
        rs.cyclic_gemm(1.0, rW, rX, 0.0, rY, True, False, True)
        rs.cached_backward_gemm(rW, rdY, rdX)
        want_y, want_dx = rs.gather_p(rY), rs.gather_p(rdX)
    assert got_y.tobytes() == want_y.tobytes()
    assert got_dx.tobytes() == want_dx.tobytes()


def test_restore_reference_checkpoint(cuda, tmp_path):
    ck = GOLDEN["checkpoint"]
    path = os.path.join(HERE, "golden", ck["file"])
    s = Session.restore(path, Config(devices=[0] * ck["workers"]))
    try:
        assert s.worker_count() == ck["workers"]
        for mid, want in ck["matrices"].items():
            assert fnv(s.gather(int(mid))) == want
        assert s.descriptor(1).version == 1 and s.descriptor(2).replicated
        # the same session state checkpoints to a byte-identical file
        out = str(tmp_path / "ours.dmth")
        s.checkpoint(out)
        assert fnv(np.frombuffer(open(out, "rb").read(), np.uint8)) == ck["file_fnv"]
    finally:
        s.close()


def test_checkpoint_rebuilt_state_matches_reference_file(cuda, tmp_path):
    ck = GOLDEN["checkpoint"]
    with session(3, ck["root_seed"]) as s:
        a = s.create_matrix(make_layout(3, 20, 18, 7, 5, 3), Precision.Single32, FillKind.SeededRandom)
        b = s.create_matrix(make_layout(0, 12, 10, 4, 10, 3), Precision.Half16, FillKind.SeededRandom)
        s.create_matrix(make_layout(2, 9, 14, 2, 14, 3), Precision.Double64, FillKind.SeededRandom)
        s.replicate(b, True)
        s.scatter(a, (np.arange(20 * 18, dtype=np.float32).reshape(20, 18) * 0.25 - 7).astype(np.float32))
        out = str(tmp_path / "rebuilt.dmth")
        s.checkpoint(out)
    assert fnv(np.frombuffer(open(out, "rb").read(), np.uint8)) == ck["file_fnv"]


def test_checkpoint_corruption_detected(cuda, tmp_path):
    ck = GOLDEN["checkpoint"]
    data = bytearray(open(os.path.join(HERE, "golden", ck["file"]), "rb").read())
    data[100] ^= 0x01
    bad = tmp_path / "bad.dmth"
    bad.write_bytes(bytes(data))
    with pytest.raises(IntegrityError):
        Session.restore(str(bad), Config(devices=[0] * 3))


def test_half_gemm_forced_pipeline_rounds_once(cuda, monkeypatch):
    """Half16 C is rounded once from the fp32 sum over the whole K (AccumOf<Half>
    + narrow_store, kernels.hpp:29-35, 72) even when the K-panel pipeline is
    forced on (remote pieces, tiny panels): the result is bit-identical to the
    single-panel schedule, and no less accurate than the reference."""
    from oracle import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not shipped")
    P, m, n, k = 2, 128, 128, 2048

    def run():
        with session(P, 91) as s:
            a = s.create_matrix(make_layout(1, m, k, m, k // P, P), Precision.Half16, FillKind.SeededRandom)
            b = s.create_matrix(make_layout(0, k, n, k // P, n, P), Precision.Half16, FillKind.SeededRandom)
            cm = s.create_matrix(make_layout(1, m, n, m, n // P, P), Precision.Half16, FillKind.SeededRandom)
            A, B, C0 = s.gather(a), s.gather(b), s.gather(cm)
            s.general_gemm(1.5, a, b, -0.5, cm, False, False)
            return s.gather(cm), A, B, C0
    plain, A, B, C0 = run()
    monkeypatch.setenv("DM_PIPELINE_MIN_GFLOP", "0")
    monkeypatch.setenv("DM_PANEL_K", "512")
    forced, _, _, _ = run()
    assert forced.tobytes() == plain.tobytes()
    with RefOracle().session(P, 91) as rs:
        ra = rs.create_p(1, m, k, m, k // P, P, 0)
        rb = rs.create_p(0, k, n, k // P, n, P, 0)
        rc = rs.create_p(1, m, n, m, n // P, P, 0)
        rs.general_gemm(1.5, ra, rb, -0.5, rc, False, False)
        want = rs.gather_p(rc)
    exact = 1.5 * (A.astype(np.float64) @ B.astype(np.float64)) - 0.5 * C0.astype(np.float64)

    def rel(x):
        return np.linalg.norm(x.astype(np.float64) - exact) / np.linalg.norm(exact)
    assert rel(forced) <= 1.5 * rel(want) + 1e-6
    assert (forced.view(np.int16) == want.view(np.int16)).mean() > 0.8
