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


def main():
    ro = RefOracle()
    g = {"generator": "tests/golden/make_golden.py (reference: /root/reference/proj/include/gridgemm)",
         "kat": [kat(ro, 256, 1.0, 0.0, False), kat(ro, 256, 1.5, -0.5, False),
                 kat(ro, 2048, 1.0, 0.0, True)],
         "sweep": sweep(ro), "fc": fc_case(ro), "errors": errors(ro), "layouts": layouts(ro), "plans": plans(ro),
         "fills": fills(ro),
         "matrix_seeds": {str(i): hx(ro.lib.ref_mix64_2(42, i)) for i in range(1, 6)}}
    with open(OUT, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print(f"wrote {OUT}: {len(g['sweep'])} sweep cases")


if __name__ == "__main__":
    main()
