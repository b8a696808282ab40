"""Distributed-matrix session on the GPU: distribute/collect bit-exactness and
general/cyclic/cached-backward GEMM parity, LOCAL mode (all workers driven by
this process; P workers may share one GPU).

Mirrors tests/test_runtime.cpp:106-141 (scatter/gather bitwise, 4 layouts)
and tests/test_dist_ops.cpp:149-155, 206-249, 267-306 of the reference.
"""
import numpy as np
import pytest

from paper_1604_01416_b200 import (CacheMissError, Config, FillKind, LayoutKind, PlanError,
                                   Session, ShapeError, UsageError, make_layout)

pytestmark = pytest.mark.gpu
TOL = 1e-5

KINDS = [LayoutKind.RowBlocks1D, LayoutKind.ColBlocks1D, LayoutKind.RowCyclic1D,
         LayoutKind.Checkerboard2D]


def relfro(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / den) if den else float(np.linalg.norm(got - want))


def ref_gemm(alpha, A, ta, B, tb, beta, C0):
    a = A.astype(np.float64)
    b = B.astype(np.float64)
    out = alpha * ((a.T if ta else a) @ (b.T if tb else b))
    if beta != 0.0:
        out = out + beta * C0.astype(np.float64)
    return out


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("kind", KINDS)
def test_scatter_gather_bitwise(cuda, P, kind):
    rng = np.random.default_rng(P * 10 + int(kind))
    host = rng.standard_normal((37, 53)).astype(np.float32)
    with Session(Config(worker_count=P, root_seed=5, devices=[0] * P)) as s:
        lay = make_layout(kind, 37, 53, 8, 16, P)
        m = s.create_matrix(lay, fill=FillKind.FromHost, host=host)
        assert s.descriptor(m).version == 1
        back = s.gather(m)
        assert back.tobytes() == host.tobytes()


@pytest.mark.parametrize("P", [1, 3, 4])
@pytest.mark.parametrize("trans", [0, 1, 2, 3])
def test_general_gemm_mixed_layouts(cuda, P, trans):
    ta, tb = bool(trans & 1), bool(trans & 2)
    n = 96
    with Session(Config(worker_count=P, root_seed=9000 + trans, devices=[0] * P)) as s:
        la = make_layout(KINDS[trans % 4], n, n, 20, 24, P)
        lb = make_layout(KINDS[(trans + 1) % 4], n, n, 24, 20, P)
        lc = make_layout(KINDS[(trans + 2) % 4], n, n, 32, 16, P)
        a = s.create_matrix(la, fill=FillKind.SeededRandom)
        b = s.create_matrix(lb, fill=FillKind.SeededRandom)
        c = s.create_matrix(lc, fill=FillKind.SeededRandom)
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        s.general_gemm(1.5, a, b, -0.5, c, ta, tb)
        got = s.gather(c)
        assert relfro(got, ref_gemm(1.5, A, ta, B, tb, -0.5, C0)) <= TOL
        assert s.descriptor(c).version == 1


def test_general_gemm_checkerboard_2048(cuda):
    """BASELINE config 1: 2048^3 on a 2x2 checkerboard of 1024^2 blocks, P=4."""
    n, P = 2048, 4
    with Session(Config(worker_count=P, root_seed=42, devices=[0] * P)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
        a = s.create_matrix(lay, fill=FillKind.SeededRandom)
        b = s.create_matrix(lay, fill=FillKind.SeededRandom)
        c = s.create_matrix(lay, fill=FillKind.SeededRandom)
        A, B = s.gather(a), s.gather(b)
        s.general_gemm(1.0, a, b, 0.0, c, False, False)
        got = s.gather(c)
        assert relfro(got, ref_gemm(1.0, A, False, B, False, 0.0, None)) <= TOL
        st = [s.worker_stats(w) for w in range(P)]
        # every worker pulls one A block and one B block of 4 MiB (2N^2 bytes ingress)
        assert all(x.peer_bytes_read == 2 * 1024 * 1024 * 4 for x in st)


def test_cyclic_and_cached_backward(cuda):
    """FC pattern: fwd Y=W^T X (TN, cache W), bwd dX=W dY (NN, cached)."""
    P, fin, fout, batch = 4, 96, 64, 32
    with Session(Config(worker_count=P, root_seed=3, devices=[0] * P)) as s:
        W = s.create_matrix(make_layout(LayoutKind.RowBlocks1D, fin, fout, fin // P, fout, P),
                            fill=FillKind.SeededRandom)
        strip = batch // P
        X = s.create_matrix(make_layout(LayoutKind.ColBlocks1D, fin, batch, fin, strip, P),
                            fill=FillKind.SeededRandom)
        Y = s.create_matrix(make_layout(LayoutKind.ColBlocks1D, fout, batch, fout, strip, P))
        dY = s.create_matrix(make_layout(LayoutKind.ColBlocks1D, fout, batch, fout, strip, P),
                             fill=FillKind.SeededRandom)
        dX = s.create_matrix(make_layout(LayoutKind.ColBlocks1D, fin, batch, fin, strip, P))
        Wh, Xh, dYh = s.gather(W), s.gather(X), s.gather(dY)
        with pytest.raises(CacheMissError) as ei:
            s.cached_backward_gemm(W, dY, dX)
        assert len(ei.value.missing_coords) > 0
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        assert relfro(s.gather(Y), ref_gemm(1.0, Wh, True, Xh, False, 0.0, None)) <= TOL
        s.reset_worker_stats()
        s.cached_backward_gemm(W, dY, dX)
        assert relfro(s.gather(dX), ref_gemm(1.0, Wh, False, dYh, False, 0.0, None)) <= TOL
        assert all(s.worker_stats(w).peer_bytes_read == 0 for w in range(P))
        # stale cache after W changes -> CacheMissError
        s.scatter(W, np.zeros((fin, fout), np.float32))
        with pytest.raises(CacheMissError):
            s.cached_backward_gemm(W, dY, dX)


def test_plan_and_usage_errors(cuda):
    with Session(Config(worker_count=2, devices=[0, 0])) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, 8, 8, 4, 4, 2)
        a = s.create_matrix(lay, fill=FillKind.SeededRandom)
        b = s.create_matrix(lay, fill=FillKind.SeededRandom)
        with pytest.raises(UsageError):
            s.general_gemm(1.0, a, b, 0.0, a)
        with pytest.raises(PlanError):
            s.cyclic_gemm(1.0, a, b, 0.0, s.create_matrix(lay))
        c = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, 8, 9, 4, 4, 2))
        with pytest.raises(ShapeError):
            s.general_gemm(1.0, a, b, 0.0, c)


def test_pool_steady_state(cuda):
    """acceptance.cpp:437-457: repeated GEMM allocates only on its first iteration."""
    P = 4
    with Session(Config(worker_count=P, root_seed=11, devices=[0] * P)) as s:
        la = make_layout(LayoutKind.RowBlocks1D, 16, 16, 2, 16, P)
        lbc = make_layout(LayoutKind.ColBlocks1D, 16, 16, 16, 4, P)
        a = s.create_matrix(la, fill=FillKind.SeededRandom)
        b = s.create_matrix(lbc, fill=FillKind.SeededRandom)
        c = s.create_matrix(lbc)
        s.cyclic_gemm(1.0, a, b, 0.0, c)
        fresh = [s.worker_pool_stats(w).fresh_allocations for w in range(P)]
        for _ in range(10):
            s.cyclic_gemm(1.0, a, b, 0.0, c)
        assert [s.worker_pool_stats(w).fresh_allocations for w in range(P)] == fresh


def test_chained_gemms_pool_steady(cuda):
    """BASELINE config 5 (small): C = A*B; D = C*E on device-resident matrices;
    no host round trip between the GEMMs and no fresh allocations after the
    first iteration (acceptance.cpp:437-457 contract)."""
    from oracle import COracle
    orc = COracle()
    P, n = 4, 384
    with Session(Config(worker_count=P, root_seed=5, devices=[0] * P)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
        A, B, E = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
        C, D = s.create_matrix(lay), s.create_matrix(lay)
        for it in range(4):
            s.general_gemm(1.0, A, B, 0.0, C)
            s.general_gemm(1.0, C, E, 0.0, D)
            if it == 0:
                fresh = [s.worker_pool_stats(w).fresh_allocations for w in range(P)]
        assert [s.worker_pool_stats(w).fresh_allocations for w in range(P)] == fresh
        Ah, Bh, Eh, Ch, Dh = (s.gather(m) for m in (A, B, E, C, D))
    assert orc.rel_frobenius(Ch, orc.local_gemm(1.0, Ah, False, Bh, False, 0.0)) <= TOL
    assert orc.rel_frobenius(Dh, orc.local_gemm(1.0, Ch, False, Eh, False, 0.0)) <= TOL


def test_fresh_cache_serves_repeated_forward(cuda):
    """A second cyclic forward with W unchanged reads the version-fresh cached
    blocks (zero peer bytes); after W changes it pulls again."""
    P, fin, fout, batch = 4, 128, 64, 32
    with Session(Config(worker_count=P, root_seed=3, devices=[0] * P)) as s:
        W = s.create_matrix(make_layout(LayoutKind.RowBlocks1D, fin, fout, fin // P, fout, P),
                            fill=FillKind.SeededRandom)
        X = s.create_matrix(make_layout(LayoutKind.ColBlocks1D, fin, batch, fin, batch // P, P),
                            fill=FillKind.SeededRandom)
        Y = s.create_matrix(make_layout(LayoutKind.ColBlocks1D, fout, batch, fout, batch // P, P))
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        s.reset_worker_stats()
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        assert sum(s.worker_stats(w).peer_bytes_read for w in range(P)) == 0
        s.scatter(W, np.ones((fin, fout), np.float32))
        s.reset_worker_stats()
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        assert sum(s.worker_stats(w).peer_bytes_read for w in range(P)) > 0
        assert relfro(s.gather(Y), ref_gemm(1.0, np.ones((fin, fout), np.float32), True, s.gather(X), False, 0.0, None)) <= TOL


@pytest.mark.parametrize("P", [1, 4])
def test_async_pipeline_double_buffered(cuda, P):
    """Asynchronous mode: scatter -> gemm -> gather steps enqueue and return;
    double-buffered matrices let H2D, GEMM and D2H of different steps overlap.
    Results must equal the synchronous path bit for bit (same kernels, same
    order of operations per output element)."""
    n = 384
    rng = np.random.default_rng(P)
    hosts = [(rng.standard_normal((n, n)).astype(np.float32), rng.standard_normal((n, n)).astype(np.float32))
             for _ in range(4)]
    with Session(Config(worker_count=P, root_seed=1, devices=[0] * P)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
        mats = [[s.create_matrix(lay) for _ in range(3)] for _ in range(2)]
        sync_out = []
        for A, B in hosts:
            a, b, c = mats[0]
            s.scatter(a, A)
            s.scatter(b, B)
            s.general_gemm(1.0, a, b, 0.0, c)
            sync_out.append(s.gather(c))
        outs = [np.empty((n, n), np.float32) for _ in hosts]
        s.set_async(True)
        for i, (A, B) in enumerate(hosts):
            a, b, c = mats[i % 2]
            s.scatter(a, A)
            s.scatter(b, B)
            s.general_gemm(1.0, a, b, 0.0, c)
            s.gather(c, outs[i])
        s.barrier()
        s.set_async(False)
        for got, want in zip(outs, sync_out):
            assert got.tobytes() == want.tobytes()
        assert s.descriptor(mats[0][2]).version == 2 + 4  # 4 sync + 2 async GEMMs on set 0


def test_seed_workers_reseeds_new_matrices(cuda):
    """Session::seed_workers (session.hpp:115-125): worker seeds become
    mix64(root, w) and matrices created afterwards derive from the new root;
    existing matrices keep their contents."""
    from oracle import COracle
    orc = COracle()
    with Session(Config(worker_count=4, root_seed=42, devices=[0] * 4)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, 64, 48, 32, 24, 4)
        a = s.create_matrix(lay, fill=FillKind.SeededRandom)  # id 1 under root 42
        assert s.root_seed() == 42 and s.deterministic()
        seeds = s.seed_workers(7)
        assert s.root_seed() == 7
        assert seeds == [orc.matrix_seed(7, w) for w in range(4)]
        assert [s.worker_seed(w) for w in range(4)] == seeds
        b = s.create_matrix(lay, fill=FillKind.SeededRandom)  # id 2 under root 7
        assert s.gather(b).tobytes() == orc.seeded_matrix(7, 2, 3, 64, 48, 32, 24).tobytes()
        assert s.gather(a).tobytes() == orc.seeded_matrix(42, 1, 3, 64, 48, 32, 24).tobytes()


def test_trace_records_block_pulls(cuda):
    """Session::trace() (TraceLog, transport.hpp:56-71), as the reference's
    acceptance tests count transfers (tests/acceptance.cpp:165-171, 213-220):
    a general_gemm pulls exactly the foreign blocks of its plan
    (GeneralGemmExec::add_needed, ops.hpp:503-524); a cached forward pulls each
    foreign W block once per version; the cached backward pulls nothing."""
    from paper_1604_01416_b200 import plan_general_gemm
    P, n = 4, 256
    with Session(Config(worker_count=P, root_seed=5, devices=[0] * P)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
        a, b, c = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
        assert s.trace() == []
        s.general_gemm(1.0, a, b, 0.0, c)
        recs = s.trace()
        assert [r["seq"] for r in recs] == list(range(1, len(recs) + 1))
        assert all(r["op"] == "general_gemm" and r["src"] != r["dst"] for r in recs)
        for w in range(P):
            nb, by = plan_general_gemm(lay, False, lay, False, lay, w)
            mine = [r for r in recs if r["dst"] == w]
            assert len(mine) == nb and sum(r["bytes"] for r in mine) == by
            assert all(lay.owner(r["row"], r["col"]) == r["src"] for r in mine)
    fin, fout, batch = 64 * P, 48, 8 * P
    with Session(Config(worker_count=P, root_seed=6, devices=[0] * P)) as s:
        W = s.create_matrix(make_layout(0, fin, fout, fin // P, fout, P), fill=FillKind.SeededRandom)
        X = s.create_matrix(make_layout(1, fin, batch, fin, batch // P, P), fill=FillKind.SeededRandom)
        Y = s.create_matrix(make_layout(1, fout, batch, fout, batch // P, P))
        dY = s.create_matrix(make_layout(1, fout, batch, fout, batch // P, P), fill=FillKind.SeededRandom)
        dX = s.create_matrix(make_layout(1, fin, batch, fin, batch // P, P))
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        first = s.trace()
        assert len(first) == P * (P - 1)  # every worker caches every foreign W block once
        assert all(r["matrix_id"] == W and r["bytes"] == (fin // P) * fout * 4 for r in first)
        s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True)
        s.cached_backward_gemm(W, dY, dX)
        assert len(s.trace()) == len(first)  # fresh cache: nothing crosses again


def _cyclic_fixture(s, ref, m, k, n, P, inner, seed, precision):
    """make_cyclic_fixture (reference tests/test_dist_ops.cpp:33-59): A
    row-blocked (`inner` blocks per worker), B and C column strips."""
    from paper_1604_01416_b200 import Precision
    np_t = np.float64 if precision == Precision.Double64 else np.float32
    rng = np.random.default_rng(seed)
    A, B, C0 = (rng.standard_normal(sh).astype(np_t) for sh in ((m, k), (k, n), (m, n)))
    strip = -(-n // P)
    la = make_layout(LayoutKind.RowBlocks1D, m, k, m // (P * inner), k, P)
    lb = make_layout(LayoutKind.ColBlocks1D, k, n, k, strip, P)
    lc = make_layout(LayoutKind.ColBlocks1D, m, n, m, strip, P)
    ids = [s.create_matrix(l, precision=precision, fill=FillKind.FromHost, host=h)
           for l, h in ((la, A), (lb, B), (lc, C0))]
    rids = [ref.create_p(int(l.kind), l.global_rows, l.global_cols, l.block_rows, l.block_cols, P,
                         int(precision), fill=2, host=h) for l, h in ((la, A), (lb, B), (lc, C0))]
    return ids, rids


def test_broadcast_gemm_reference_fanout(cuda):
    """Reference tests/test_dist_ops.cpp:341-364: broadcast_gemm_reference
    computes the same C as cyclic_gemm (bitwise, Double64) and every A block
    fans out to both other workers, tagged broadcast_gemm:r<row>
    (BroadcastGemmExec::send_phase, ops.hpp:590-606).  The transfer records
    must equal the reference's own trace() for the same call."""
    from oracle import RefOracle
    from paper_1604_01416_b200 import Precision
    ro = RefOracle()
    P = 3
    with Session(Config(worker_count=P, root_seed=42, devices=[0] * P)) as s, ro.session(P, 42) as r:
        (a, b, c), _ = _cyclic_fixture(s, r, 6, 6, 6, P, 2, 900, Precision.Double64)
        s.cyclic_gemm(1.0, a, b, 0.0, c, False, False, False)
        cyc = s.gather(c)
    with Session(Config(worker_count=P, root_seed=42, devices=[0] * P)) as s, ro.session(P, 42) as r:
        (a, b, c), (ra, rb, rc) = _cyclic_fixture(s, r, 6, 6, 6, P, 2, 900, Precision.Double64)
        before = len(s.trace())
        s.broadcast_gemm_reference(1.0, a, b, 0.0, c, False, False)
        assert s.gather(c).tobytes() == cyc.tobytes()
        assert s.descriptor(c).version == 2  # FromHost scatter (1) + the GEMM
        r0 = len(r.trace_records())
        assert r.broadcast_gemm_reference(1.0, ra, rb, 0.0, rc) == 0
        assert s.gather(c).tobytes() == r.gather_p(rc).tobytes()  # Double64: bit-exact
        mine = s.trace()[before:]
        theirs = [t for t in r.trace_records(r0) if t["op"].startswith("broadcast_gemm:")]  # not gathers
        assert len(mine) == 3 * 2 * 2
        dsts = {}
        for rec in mine:
            assert rec["op"].startswith("broadcast_gemm:r")
            dsts.setdefault(rec["op"], set()).add(rec["dst"])
        assert len(dsts) == 6 and all(len(d) == 2 for d in dsts.values())
        key = lambda x: (x["src"], x["dst"], x["op"], x["bytes"])
        assert sorted(map(key, mine)) == sorted(map(key, theirs))


def test_broadcast_gemm_keeps_the_fc_cache(cuda):
    """session.hpp:236-242: broadcast_gemm_reference leaves A's block cache and
    cache_meta_ alone, so the FC sequence cyclic_gemm(cache_a) ->
    broadcast_gemm_reference -> cached_backward_gemm succeeds -- in the
    reference (run beside it) and here -- and the broadcast reads the fresh
    cached copies instead of pulling again."""
    from oracle import RefOracle
    ro = RefOracle()
    P, fin, fout, batch = 4, 64, 48, 32
    rng = np.random.default_rng(77)
    W, X, dY = (rng.standard_normal(sh).astype(np.float32) for sh in ((fin, fout), (fin, batch), (fout, batch)))
    lw = make_layout(LayoutKind.RowBlocks1D, fin, fout, fin // P, fout, P)
    lx = make_layout(LayoutKind.ColBlocks1D, fin, batch, fin, batch // P, P)
    ly = make_layout(LayoutKind.ColBlocks1D, fout, batch, fout, batch // P, P)
    with Session(Config(worker_count=P, root_seed=3, devices=[0] * P)) as s, ro.session(P, 3) as r:
        ours, theirs = [], []
        for l, h in ((lw, W), (lx, X), (ly, None), (ly, dY), (lx, None)):
            ours.append(s.create_matrix(l, fill=FillKind.FromHost if h is not None else FillKind.Zeros, host=h))
            theirs.append(r.create_p(int(l.kind), l.global_rows, l.global_cols, l.block_rows, l.block_cols, P, 1,
                                     fill=2 if h is not None else 0, host=h))
        w, x, y, dy, dx = ours
        rw, rx, ry, rdy, rdx = theirs
        s.cyclic_gemm(1.0, w, x, 0.0, y, True, False, True)          # FC forward, keep W blocks
        assert r.cyclic_gemm(1.0, rw, rx, 0.0, ry, True, False, True) == 0
        n_cached = len(s.trace())
        s.broadcast_gemm_reference(1.5, w, x, -0.5, y, True, False)
        assert r.broadcast_gemm_reference(1.5, rw, rx, -0.5, ry, True, False) == 0
        assert relfro(s.gather(y), r.gather_p(ry)) <= TOL
        assert len(s.trace()) == n_cached  # served from the fresh cache, nothing pulled
        assert r.cached_backward_gemm(rw, rdy, rdx) == 0
        s.cached_backward_gemm(w, dy, dx)  # raised CacheMissError while broadcast aliased cyclic
        assert relfro(s.gather(dx), r.gather_p(rdx)) <= TOL


def test_graph_replay_follows_operand_contents(cuda, monkeypatch):
    """Repeated small commands replay a captured graph (DM_GRAPHS): results
    must follow every new scatter of the operands and C, bitwise equal to the
    eager schedule, and the per-worker counters and trace() keep counting."""
    n, P = 256, 4
    rng = np.random.default_rng(3)
    hosts = [rng.standard_normal((n, n)).astype(np.float32) for _ in range(6)]
    outs = {}
    for graphs in ("0", "1"):
        monkeypatch.setenv("DM_GRAPHS", graphs)
        with Session(Config(worker_count=P, root_seed=1, devices=[0] * P)) as s:
            lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // 2, n // 2, P)
            a, b, c = (s.create_matrix(lay) for _ in range(3))
            res = []
            for i in range(3):
                s.scatter(a, hosts[2 * i])
                s.scatter(b, hosts[2 * i + 1])
                s.scatter(c, hosts[(2 * i + 2) % 6])
                s.reset_worker_stats()
                n_trace = len(s.trace())
                s.general_gemm(1.5, a, b, -0.5, c, i == 1, i == 2)
                res.append(s.gather(c))
                assert sum(s.worker_stats(w).gemm_launches for w in range(P)) == P
                # one record per foreign block of each worker's pull plan
                from paper_1604_01416_b200 import plan_general_gemm
                want_recs = sum(plan_general_gemm(lay, i == 1, lay, i == 2, lay, w)[0] for w in range(P))
                assert len(s.trace()) - n_trace == want_recs
                want = ref_gemm(1.5, hosts[2 * i], i == 1, hosts[2 * i + 1], i == 2, -0.5, hosts[(2 * i + 2) % 6])
                assert relfro(res[-1], want) <= TOL
            # the same command again: a replay
            s.general_gemm(1.5, a, b, -0.5, c, False, True)
            res.append(s.gather(c))
            s.destroy_matrix(b)  # drops the graphs that read it
            b2 = s.create_matrix(lay, fill=FillKind.FromHost, host=hosts[5])
            s.general_gemm(1.0, a, b2, 0.0, c)
            res.append(s.gather(c))
            outs[graphs] = res
    for x, y in zip(outs["0"], outs["1"]):
        assert x.tobytes() == y.tobytes()


def test_fc_plane_cache_follows_weight_versions(cuda):
    """cyclic_gemm(cache_a) / cached_backward_gemm keep W's split planes while
    W's version holds; a new W (scatter -> version + 1) is re-split."""
    P, fin, fout, batch = 4, 512, 384, 64
    rng = np.random.default_rng(11)
    Ws = [rng.standard_normal((fin, fout)).astype(np.float32) for _ in range(2)]
    X = rng.standard_normal((fin, batch)).astype(np.float32)
    dY = rng.standard_normal((fout, batch)).astype(np.float32)
    with Session(Config(worker_count=P, root_seed=2, devices=[0] * P)) as s:
        W = s.create_matrix(make_layout(0, fin, fout, fin // P, fout, P), fill=FillKind.FromHost, host=Ws[0])
        x = s.create_matrix(make_layout(1, fin, batch, fin, batch // P, P), fill=FillKind.FromHost, host=X)
        y = s.create_matrix(make_layout(1, fout, batch, fout, batch // P, P))
        dy = s.create_matrix(make_layout(1, fout, batch, fout, batch // P, P), fill=FillKind.FromHost, host=dY)
        dx = s.create_matrix(make_layout(1, fin, batch, fin, batch // P, P))
        for step in range(4):
            Wh = Ws[step // 2]
            if step == 2:
                s.scatter(W, Wh)  # new weights: version + 1
            s.reset_worker_stats()
            s.cyclic_gemm(1.0, W, x, 0.0, y, True, False, True)
            fwd_splits = sum(s.worker_stats(w).split_launches for w in range(P))
            assert relfro(s.gather(y), ref_gemm(1.0, Wh, True, X, False, 0.0, None)) <= TOL
            s.cached_backward_gemm(W, dy, dx)
            assert relfro(s.gather(dx), ref_gemm(1.0, Wh, False, dY, False, 0.0, None)) <= TOL
            if step % 2 == 1:  # same W as the previous step: only X's pieces are split
                assert fwd_splits == P


def test_graft_smoke(cuda):
    """__graft_entry__.smoke(): the reference KAT case and the headline
    (f16x2, presplit) schedule at small sizes against the oracle."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "graft_entry", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "__graft_entry__.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.smoke()
