"""Generate tests/golden/golden.json from the REFERENCE implementation itself.

Runs the unmodified reference (oracle/_ref/libgridgemm_ref.so, compiled from
/root/reference/proj/include by oracle/Makefile) and records bit-level digests
(FNV-1a 64 over the gathered row-major fp32 bytes, gridgemm/common.hpp:83-103)
of inputs and results, error codes, layout tables and fill vectors.  The CPU
tests pin the C restatement (oracle/dmath_oracle.c) and the product's host
logic to these; the GPU tests pin the device fill / distribute / collect
bit-exactly and the GEMM within relFro <= 1e-5.

Usage (build container, where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import RefOracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
KINDS = [0, 1, 2, 3]  # RowBlocks1D, ColBlocks1D, RowCyclic1D, Checkerboard2D


def hx(v: int) -> str:
    return f"{v:016x}"


def summary(ro, m):
    return {"fnv": hx(ro.fnv1a(m)), "sum": float(m.astype(np.float64).sum()),
            "first": float(m.flat[0]), "last": float(m.flat[-1])}


def kat(ro, n, alpha, beta, threaded):
    with ro.session(4, 42, deterministic=not threaded) as s:
        lay = (3, n, n, n // 2, n // 2, 4)
        a = s.create(*lay)
        b = s.create(*lay)
        c = s.create(*lay)
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        assert s.general_gemm(alpha, a, b, beta, c) == 0, ro.err()
        Cm = s.gather(c)
        return {"n": n, "alpha": alpha, "beta": beta, "root_seed": 42, "workers": 4,
                "layout": [3, n, n, n // 2, n // 2, 4],
                "A": summary(ro, A), "B": summary(ro, B), "C0": summary(ro, C0), "C": summary(ro, Cm),
                "C_version": s.version(c)}


def sweep(ro):
    cases = []
    combo = 0
    for n in (3, 7, 16, 29, 32):
        for bs in (1, 2, 5):
            for P in (1, 2, 3, 4):
                for trans in range(4):
                    combo += 1
                    if combo % 3:  # keep the fixture small: every third combination
                        continue
                    ta, tb = bool(trans & 1), bool(trans & 2)
                    seed = 9000 + combo
                    with ro.session(P, seed) as s:
                        la = [KINDS[combo % 4], n, n, bs, bs, P]
                        lb = [KINDS[(combo + 1) % 4], n, n, bs, bs, P]
                        lc = [KINDS[(combo + 2) % 4], n, n, bs, bs, P]
                        a, b, c = s.create(*la), s.create(*lb), s.create(*lc)
                        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
                        assert s.general_gemm(1.0, a, b, 0.5, c, ta, tb) == 0
                        Cm = s.gather(c)
                        cases.append({"op": "general", "root_seed": seed, "workers": P, "m": n, "k": n,
                                      "n": n, "ta": ta, "tb": tb, "alpha": 1.0, "beta": 0.5,
                                      "la": la, "lb": lb, "lc": lc,
                                      "A": hx(ro.fnv1a(A)), "B": hx(ro.fnv1a(B)), "C0": hx(ro.fnv1a(C0)),
                                      "C": hx(ro.fnv1a(Cm))})
    # rectangular (acceptance.cpp:128-147 pattern), alpha=-0.5 beta=1
    rect = [(3, 5, 7), (8, 13, 21), (32, 17, 9), (5, 32, 6), (31, 1, 31)]
    for (m, k, n) in rect:
        for P in (1, 3):
            for trans in range(4):
                combo += 1
                ta, tb = bool(trans & 1), bool(trans & 2)
                seed = 17000 + combo
                with ro.session(P, seed) as s:
                    la = [KINDS[combo % 4], k if ta else m, m if ta else k, 2, 3, P]
                    lb = [KINDS[(combo + 1) % 4], n if tb else k, k if tb else n, 3, 2, P]
                    lc = [KINDS[(combo + 2) % 4], m, n, 2, 2, P]
                    a, b, c = s.create(*la), s.create(*lb), s.create(*lc)
                    A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
                    assert s.general_gemm(-0.5, a, b, 1.0, c, ta, tb) == 0
                    Cm = s.gather(c)
                    cases.append({"op": "general", "root_seed": seed, "workers": P, "m": m, "k": k, "n": n,
                                  "ta": ta, "tb": tb, "alpha": -0.5, "beta": 1.0, "la": la, "lb": lb, "lc": lc,
                                  "A": hx(ro.fnv1a(A)), "B": hx(ro.fnv1a(B)), "C0": hx(ro.fnv1a(C0)),
                                  "C": hx(ro.fnv1a(Cm))})
    # ring-eligible cyclic cases (acceptance.cpp:80-113 pattern), beta=0
    for n in (8, 12, 24):
        for P in (2, 4):
            for bs in (1, 2):
                nbr = -(-n // bs)
                if nbr % P:
                    continue
                for trans in range(4):
                    combo += 1
                    ta, tb = bool(trans & 1), bool(trans & 2)
                    seed = 23000 + combo
                    strip = -(-n // P)
                    with ro.session(P, seed) as s:
                        la = [2 if combo % 2 else 0, n, n, bs, n, P]
                        lb = [0, n, n, strip, n, P] if tb else [1, n, n, n, strip, P]
                        lc = [1, n, n, n, strip, P]
                        a, b, c = s.create(*la), s.create(*lb), s.create(*lc)
                        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
                        assert s.cyclic_gemm(1.0, a, b, 0.0, c, ta, tb, False) == 0, ro.err()
                        Cm = s.gather(c)
                        cases.append({"op": "cyclic", "root_seed": seed, "workers": P, "m": n, "k": n, "n": n,
                                      "ta": ta, "tb": tb, "alpha": 1.0, "beta": 0.0, "la": la, "lb": lb,
                                      "lc": lc, "A": hx(ro.fnv1a(A)), "B": hx(ro.fnv1a(B)),
                                      "C0": hx(ro.fnv1a(C0)), "C": hx(ro.fnv1a(Cm))})
    return cases


def fc_case(ro):
    """FC fwd (cyclic TN, cache W) / bwd (cached NN, zero transfers) / dW (general NT)."""
    P, fin, fout, batch = 4, 96, 64, 32
    strip = batch // P
    out = {"workers": P, "fin": fin, "fout": fout, "batch": batch, "root_seed": 3}
    with ro.session(P, 3) as s:
        W = s.create(0, fin, fout, fin // P, fout, P)
        X = s.create(1, fin, batch, fin, strip, P)
        Y = s.create(1, fout, batch, fout, strip, P, fill=0)
        dY = s.create(1, fout, batch, fout, strip, P)
        dX = s.create(1, fin, batch, fin, strip, P, fill=0)
        dW = s.create(0, fin, fout, fin // P, fout, P, fill=0)
        out["missing_before_fwd"] = s.cached_backward_gemm(W, dY, dX)
        assert s.cyclic_gemm(1.0, W, X, 0.0, Y, True, False, True) == 0
        t0 = s.transfers()[0]
        assert s.cached_backward_gemm(W, dY, dX) == 0
        out["bwd_transfers"] = s.transfers()[0] - t0
        assert s.general_gemm(1.0, X, dY, 0.0, dW, False, True) == 0
        for name, mid in (("W", W), ("X", X), ("Y", Y), ("dY", dY), ("dX", dX), ("dW", dW)):
            out[name] = hx(ro.fnv1a(s.gather(mid)))
        s.scatter(W, np.zeros((fin, fout), np.float32))
        out["stale_rc"] = s.cached_backward_gemm(W, dY, dX)
    return out


def errors(ro):
    out = {}
    with ro.session(2, 1) as s:
        a = s.create(3, 8, 8, 4, 4, 2)
        b = s.create(3, 8, 8, 4, 4, 2)
        c = s.create(3, 8, 9, 4, 4, 2)
        out["alias"] = s.general_gemm(1.0, a, b, 0.0, a)
        out["shape"] = s.general_gemm(1.0, a, b, 0.0, c)
        out["plan"] = s.cyclic_gemm(1.0, a, b, 0.0, s.create(3, 8, 8, 4, 4, 2))
        out["unknown_id"] = s.general_gemm(1.0, a, b, 0.0, 999)
    return out


def layouts(ro):
    rows = []
    for kind in KINDS:
        for (gr, gc, br, bc, w) in [(16, 16, 4, 4, 4), (37, 53, 8, 16, 3), (2048, 2048, 1024, 512, 8),
                                    (10, 7, 3, 2, 5), (9, 9, 20, 20, 2), (32768, 32768, 16384, 8192, 8)]:
            nbr, nbc = -(-gr // min(br, gr)), -(-gc // min(bc, gc))
            table = [ro.owner(kind, gr, gc, br, bc, w, r, c) for r in range(nbr) for c in range(nbc)]
            rows.append({"kind": kind, "dims": [gr, gc, br, bc, w], "nbr": nbr, "nbc": nbc,
                         "owners": table, "string": ro.layout_string(kind, gr, gc, br, bc, w)})
    return rows


def plans(ro):
    """Reference transfer count/bytes of one general_gemm (GeneralGemmExec plan,
    ops.hpp:406-467): the deduplicated (block, destination) pushes."""
    out = []
    combos = [((3, 2048, 2048, 1024, 1024, 4),) * 3,
              ((3, 64, 64, 32, 16, 8),) * 3,
              ((0, 48, 40, 8, 40, 3), (1, 40, 36, 40, 12, 3), (3, 48, 36, 16, 12, 3)),
              ((2, 30, 30, 4, 6, 4), (3, 30, 30, 6, 4, 4), (0, 30, 30, 5, 30, 4))]
    for (la, lb, lc) in combos:
        for trans in range(4):
            ta, tb = bool(trans & 1), bool(trans & 2)
            if la[1] != la[2] and (ta or tb):
                continue
            P = la[5]
            with ro.session(P, 5) as s:
                a, b, c = s.create(*la), s.create(*lb), s.create(*lc)
                t0, b0 = s.transfers()
                if s.general_gemm(1.0, a, b, 0.0, c, ta, tb) != 0:
                    continue
                t1, b1 = s.transfers()
                out.append({"la": list(la), "lb": list(lb), "lc": list(lc), "ta": ta, "tb": tb,
                            "transfers": t1 - t0, "payload_bytes": b1 - b0})
    return out


def fills(ro):
    out = []
    for (seed, r, c, rows, cols) in [(0, 0, 0, 4, 4), (42, 1, 0, 3, 5), (2**63 + 5, 7, 3, 2, 9)]:
        blk = ro.fill_block(rows, cols, seed, r, c)
        out.append({"seed": str(seed), "brow": r, "bcol": c, "rows": rows, "cols": cols,
                    "bits": [int(x) for x in blk.view(np.uint32).ravel()], "fnv": hx(ro.fnv1a(blk))})
    return out


# ------------------------------------------------------------ SURVEY 8(f)
LAYS = [(0, 12, 20, 5, 7), (1, 12, 20, 5, 7), (2, 12, 20, 5, 7), (3, 12, 20, 5, 7), (3, 33, 17, 8, 6)]


def fills_p(ro):
    out = []
    for prec in (0, 1, 2):
        for (kind, gr, gc, br, bc) in LAYS:
            with ro.session(4, 11 + prec) as s:
                m = s.create_p(kind, gr, gc, br, bc, 4, prec)
                out.append({"precision": prec, "layout": [kind, gr, gc, br, bc, 4], "root_seed": 11 + prec,
                            "fnv": hx(ro.fnv1a(s.gather_p(m)))})
    return out


def reshapes(ro):
    cases = []
    combos = [((3, 12, 20, 5, 7), (0, 16, 15, 4, 15), 1, 0),   # single -> half (narrow before link)
              ((0, 12, 20, 3, 20), (3, 20, 12, 6, 5), 0, 1),   # half -> single (widen at receiver)
              ((1, 24, 10, 24, 3), (2, 6, 40, 2, 9), 2, 0),    # double -> half
              ((2, 24, 10, 5, 10), (3, 10, 24, 4, 7), 1, 2),   # single -> double
              ((3, 33, 17, 8, 6), (1, 51, 11, 51, 4), 1, 1),   # same precision, new shape
              ((0, 7, 9, 7, 9), (3, 3, 21, 2, 8), 2, 2)]
    for P in (1, 3, 4):
        for i, (src, dst, sp, dp) in enumerate(combos):
            with ro.session(P, 31 + i) as s:
                a = s.create_p(src[0], src[1], src[2], src[3], src[4], P, sp)
                b = s.reshape(a, dst[0], dst[1], dst[2], dst[3], dst[4], P, dp)
                cases.append({"workers": P, "root_seed": 31 + i, "src": list(src), "src_prec": sp,
                              "dst": list(dst), "dst_prec": dp, "src_fnv": hx(ro.fnv1a(s.gather_p(a))),
                              "dst_fnv": hx(ro.fnv1a(s.gather_p(b))), "dst_id": b})
    return cases


def sums(ro):
    cases = []
    for P in (1, 2, 3, 4):
        for prec in (0, 1, 2):
            for (kind, gr, gc, br, bc) in LAYS[:4] + [(3, 40, 70, 9, 11)]:
                for axis in (0, 1):
                    for det in (True, False):
                        seed = 51 + P * 7 + prec
                        with ro.session(P, seed) as s:
                            m = s.create_p(kind, gr, gc, br, bc, P, prec)
                            o = s.add_row_col_sum(m, axis, det)
                            o2 = s.add_row_col_sum(m, axis, det)  # salt advances per call
                            cases.append({"workers": P, "root_seed": seed, "precision": prec,
                                          "layout": [kind, gr, gc, br, bc, P], "axis": axis, "det": det,
                                          "in_fnv": hx(ro.fnv1a(s.gather_p(m))),
                                          "out_fnv": hx(ro.fnv1a(s.gather_p(o))),
                                          "out2_fnv": hx(ro.fnv1a(s.gather_p(o2))),
                                          "out_layout": s.describe(o)[5], "out_id": o})
    return cases


def replication(ro):
    out = []
    for P in (1, 3, 4):
        with ro.session(P, 71) as s:
            m = s.create_p(3, 30, 22, 7, 6, P, 1)
            s.replicate(m, True)
            d1 = s.describe(m)
            r0 = s.replica_read(m, P - 1)
            new = (np.arange(30 * 22, dtype=np.float32).reshape(30, 22) / 7.0).astype(np.float32)
            s.scatter(m, new)
            d2 = s.describe(m)
            r1 = s.replica_read(m, 0)
            d3 = s.describe(m)
            out.append({"workers": P, "root_seed": 71, "layout": [3, 30, 22, 7, 6, P],
                        "read0_fnv": hx(ro.fnv1a(r0)), "read1_fnv": hx(ro.fnv1a(r1)),
                        "desc_after_enable": list(d1[:3]), "desc_after_scatter": list(d2[:3]),
                        "desc_after_read": list(d3[:3])})
    return out


def update_blocks(ro):
    out = []
    with ro.session(3, 81) as s:
        m = s.create_p(1, 20, 30, 20, 7, 3, 1)
        data = (np.linspace(-3, 3, 20 * 7, dtype=np.float32).reshape(20, 7))
        s.update_block(m, 0, 2, data)
        out.append({"workers": 3, "root_seed": 81, "layout": [1, 20, 30, 20, 7, 3], "block": [0, 2],
                    "version": s.describe(m)[0], "fnv": hx(ro.fnv1a(s.gather_p(m)))})
    return out


def half_gemm(ro):
    cases = []
    for P in (1, 4):
        for trans in range(4):
            ta, tb = bool(trans & 1), bool(trans & 2)
            with ro.session(P, 91 + trans) as s:
                a = s.create_p(3, 40, 40, 16, 12, P, 0)
                b = s.create_p(0, 40, 40, 10, 40, P, 0)
                c = s.create_p(2, 40, 40, 9, 40, P, 0)
                C0 = s.gather_p(c)
                assert s.general_gemm(1.5, a, b, -0.5, c, ta, tb) == 0
                cases.append({"workers": P, "root_seed": 91 + trans, "ta": ta, "tb": tb,
                              "A": hx(ro.fnv1a(s.gather_p(a))), "B": hx(ro.fnv1a(s.gather_p(b))),
                              "C0": hx(ro.fnv1a(C0)), "C": hx(ro.fnv1a(s.gather_p(c)))})
    return cases


def checkpoint_fixture(ro):
    """A reference-written DMTH file (committed) plus the recipe to rebuild the
    same session state, so the product can be checked both ways."""
    path = os.path.join(os.path.dirname(OUT), "ref_checkpoint.dmth")
    with ro.session(3, 1234) as s:
        a = s.create_p(3, 20, 18, 7, 5, 3, 1)
        b = s.create_p(0, 12, 10, 4, 10, 3, 0)
        c = s.create_p(2, 9, 14, 2, 14, 3, 2)
        s.replicate(b, True)
        s.scatter(a, (np.arange(20 * 18, dtype=np.float32).reshape(20, 18) * 0.25 - 7).astype(np.float32))
        s.checkpoint(path)
        digests = {str(m): hx(ro.fnv1a(s.gather_p(m))) for m in (a, b, c)}
    data = open(path, "rb").read()
    r = RefSession_restore(ro, path)
    return {"file": "ref_checkpoint.dmth", "file_fnv": hx(ro.fnv1a(np.frombuffer(data, np.uint8))),
            "bytes": len(data), "workers": 3, "root_seed": 1234, "matrices": digests,
            "recipe": "create(3,20x18,7x5,f32); create(0,12x10,4x10,f16); create(2,9x14,2x14,f64); "
                      "replicate(2); scatter(1, arange(360)*0.25-7)", "restored_ok": r}


def RefSession_restore(ro, path):
    from oracle import RefSession
    rs = RefSession.restore(ro, path)
    ok = all(rs.describe(m)[0] >= 0 for m in (1, 2, 3))
    rs.close()
    return ok


def main():
    ro = RefOracle()
    g = {"generator": "tests/golden/make_golden.py (reference: /root/reference/proj/include/gridgemm)",
         "kat": [kat(ro, 256, 1.0, 0.0, False), kat(ro, 256, 1.5, -0.5, False),
                 kat(ro, 2048, 1.0, 0.0, True)],
         "sweep": sweep(ro), "fc": fc_case(ro), "errors": errors(ro), "layouts": layouts(ro), "plans": plans(ro),
         "fills_p": fills_p(ro), "reshape": reshapes(ro), "sums": sums(ro),
         "replication": replication(ro), "update_block": update_blocks(ro), "half_gemm": half_gemm(ro),
         "checkpoint": checkpoint_fixture(ro),
         "fills": fills(ro),
         "matrix_seeds": {str(i): hx(ro.lib.ref_mix64_2(42, i)) for i in range(1, 6)}}
    with open(OUT, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print(f"wrote {OUT}: {len(g['sweep'])} sweep cases")


if __name__ == "__main__":
    main()
