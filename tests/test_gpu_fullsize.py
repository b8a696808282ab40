"""Parity of the CTA-pair (256x256-tile, cta_group::2) tcgen05 GEMM through
general_gemm at sizes where it runs, against the reference itself.

A row (column) of the reference's distributed result depends only on that
row of op(A) (column of op(B)), alpha, beta and C0, with k ascending over the
full K in every executor (ops.hpp:274, 485).  So the reference's local_gemm
on 1 x K rows / K x 1 columns (oracle/_ref, the unmodified reference)
reproduces those elements of its distributed result bit for bit, and the
checks below are parity against the reference's own output, at sizes where a
full reference GEMM would take hours (the reference checks whole
results at its own sizes, harness.hpp:114-125, tests/acceptance.cpp:33-149).

Bars: relFro <= 1e-5 against the reference (the north star's tolerance,
acceptance.cpp:66-72), and the GPU's distance from the exact (fp64) product
of the same samples within a stated factor of the reference's own distance
(RATIO below): the split GEMM keeps fp32-level accuracy at every K.
"""
import json
import os

import numpy as np
import pytest

from paper_1604_01416_b200 import Config, FillKind, LayoutKind, Session, make_layout

pytestmark = pytest.mark.gpu
TOL = 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = min(32, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def ref():
    from oracle import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not shipped")
    return RefOracle()


def spread(n, count, salt):
    step = max(1, n // count)
    return [min(n - 1, i * step + (i * 131 + salt * 977 + 17) % step) for i in range(count)]


def sampled_reference(ro, alpha, A, ta, B, tb, beta, C0, rows, cols):
    """Reference elements C[rows, :] and C[:, cols] (as rows x n and cols x m)."""
    a_rows = np.ascontiguousarray(A[:, rows].T if ta else A[rows])
    c0r = np.ascontiguousarray(C0[rows]) if beta != 0.0 else None
    want_r = ro.sampled_rows(alpha, a_rows, B, tb, beta, c0r, threads=THREADS)
    b_cols = np.ascontiguousarray(B[cols] if tb else B[:, cols].T)
    c0c = np.ascontiguousarray(C0[:, cols].T) if beta != 0.0 else None
    want_c = ro.sampled_cols(alpha, A, ta, b_cols, beta, c0c, threads=THREADS)
    return want_r, want_c, a_rows, b_cols


def exact_samples(alpha, A, ta, a_rows, B, tb, b_cols, beta, C0, rows, cols):
    """fp64 products of the same samples."""
    B64 = B.astype(np.float64)
    er = alpha * (a_rows.astype(np.float64) @ (B64.T if tb else B64))
    A64 = A.astype(np.float64)
    ec = alpha * ((A64.T if ta else A64) @ b_cols.T.astype(np.float64)).T
    if beta != 0.0:
        er = er + beta * C0[rows].astype(np.float64)
        ec = ec + beta * C0[:, cols].T.astype(np.float64)
    return er, ec


def relfro(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))


def check(got, rows, cols, want_r, want_c, er=None, ec=None):
    gs = np.concatenate([got[rows].ravel(), got[:, cols].T.ravel()])
    ws = np.concatenate([want_r.ravel(), want_c.ravel()])
    out = {"vs_reference": relfro(gs, ws)}
    if er is not None:
        ex = np.concatenate([er.ravel(), ec.ravel()])
        out["gpu_vs_exact"] = relfro(gs, ex)
        out["ref_vs_exact"] = relfro(ws, ex)
    return out


def record(name, res):
    """Keep the measured numbers (gpurun_out/ travels back from the GPU box)."""
    path = os.path.join(ROOT, "gpurun_out", "fullsize_parity.jsonl")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "a") as f:
        f.write(json.dumps({"case": name, **res}) + "\n")


@pytest.mark.parametrize("P,n", [(1, 4096), (4, 8192)])
@pytest.mark.parametrize("trans", [0, 1, 2, 3])
def test_pair_kernel_transposes_alpha_beta(cuda, ref, P, n, trans):
    """>= 4096 (256x256 CTA-pair tiles on every worker), all four transpose
    combinations, alpha=1.5 / beta=-0.5 (reference tests/test_dist_ops.cpp:
    136-147, 267-282), one worker and a 2x2 checkerboard of 4 workers."""
    ta, tb = bool(trans & 1), bool(trans & 2)
    pr = 2 if P == 4 else 1
    with Session(Config(worker_count=P, root_seed=300 + trans, devices=[0] * P)) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n // pr, n // pr, P)
        a, b, c = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(3))
        A, B, C0 = s.gather(a), s.gather(b), s.gather(c)
        s.general_gemm(1.5, a, b, -0.5, c, ta, tb)
        got = s.gather(c)
    rows, cols = spread(n, 16, trans), spread(n, 16, trans + 7)
    want_r, want_c, a_rows, b_cols = sampled_reference(ref, 1.5, A, ta, B, tb, -0.5, C0, rows, cols)
    er, ec = exact_samples(1.5, A, ta, a_rows, B, tb, b_cols, -0.5, C0, rows, cols)
    res = check(got, rows, cols, want_r, want_c, er, ec)
    record(f"pair_P{P}_n{n}_t{trans}", res)
    assert res["vs_reference"] <= TOL, res
    assert res["gpu_vs_exact"] <= 3e-6, res


def test_config2_16384_sampled_rows_and_columns(cuda, ref):
    """BASELINE config 2: 16384^3 on one B200 (seeded inputs of the
    reference's create_matrix), 16 rows + 16 columns over every tile row /
    column band against the reference."""
    n = 16384
    with Session(Config(worker_count=1, root_seed=42, devices=[0])) as s:
        lay = make_layout(LayoutKind.Checkerboard2D, n, n, n, n, 1)
        a, b = (s.create_matrix(lay, fill=FillKind.SeededRandom) for _ in range(2))
        c = s.create_matrix(lay)
        s.general_gemm(1.0, a, b, 0.0, c)
        A, B, got = s.gather(a), s.gather(b), s.gather(c)
    rows, cols = spread(n, 16, 1), spread(n, 16, 2)
    want_r, want_c, a_rows, b_cols = sampled_reference(ref, 1.0, A, False, B, False, 0.0, None, rows, cols)
    er, ec = exact_samples(1.0, A, False, a_rows, B, False, b_cols, 0.0, None, rows, cols)
    res = check(got, rows, cols, want_r, want_c, er, ec)
    record("config2_16384", res)
    assert res["vs_reference"] <= TOL, res
    assert res["gpu_vs_exact"] <= res["ref_vs_exact"], res  # no less accurate than the reference


# GPU distance from exact <= RATIO x the reference's own + FLOOR (relFro).
# The reference's fp32 k-ascending loop is ~2e-7 from exact at K=256 and
# ~3e-6 at K=32768; the split GEMM's error is set by its
# TMEM accumulation chunk, which the default shortens at small K
# (tf32x3_default_flush_k) so that it stays near or below the reference's.
# Measured (profiles/r02): 3xTF32 within 1.25x of the reference's error at
# every K and distribution; the mixed split's bf16 cross terms leave a ~6e-7
# floor -- up to 4x the reference at K=256.  The scaled 2xFP16 split (f16x2,
# "auto") repeats 3xTF32's 11+11-bit pair and products and is held to the
# same bar.
def bar(gemm_mode, k):
    if gemm_mode == "mixed" and k <= 8192:
        return 4.5, 1e-7
    return 1.5, 1e-7
_REF_CACHE = {}


def _operands(dist, k, n):
    rng = np.random.default_rng({"u01": 1, "pm1": 2, "logu": 3}[dist] * 100 + k)
    def gen(shape):
        if dist == "u01":
            return rng.random(shape, dtype=np.float32)
        if dist == "pm1":
            return (rng.random(shape, dtype=np.float32) * 2 - 1).astype(np.float32)
        mag = np.exp2(rng.uniform(-20, 20, shape))
        return (mag * rng.choice([-1.0, 1.0], shape)).astype(np.float32)
    return gen((n, k)), gen((k, n))


@pytest.mark.parametrize("gemm_mode", ["auto", "f16x2", "mixed", "3xtf32"])
@pytest.mark.parametrize("k", [256, 9216, 32768])
@pytest.mark.parametrize("dist", ["u01", "pm1", "logu"])
def test_distributions_and_k(cuda, ref, gemm_mode, k, dist):
    """Input distributions U[0,1) (no cancellation), U[-1,1), signed
    log-uniform 2^+-20 (wide exponent range), at the FC dW K (256), the FC
    forward K (9216) and the headline K (32768), in every split mode, through
    general_gemm on the CTA-pair kernel (4096 x 4096 C)."""
    n = 4096
    A, B = _operands(dist, k, n)
    with Session(Config(worker_count=1, root_seed=1, devices=[0], gemm_mode=gemm_mode)) as s:
        assert s.gemm_mode() == gemm_mode
        a = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, n, k, n, k, 1), fill=FillKind.FromHost, host=A)
        b = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, k, n, k, n, 1), fill=FillKind.FromHost, host=B)
        c = s.create_matrix(make_layout(LayoutKind.Checkerboard2D, n, n, n, n, 1))
        s.general_gemm(1.0, a, b, 0.0, c)
        got = s.gather(c)
    rows, cols = spread(n, 8, k), spread(n, 8, k + 1)
    key = (dist, k)
    if key not in _REF_CACHE:
        want_r, want_c, a_rows, b_cols = sampled_reference(ref, 1.0, A, False, B, False, 0.0, None, rows, cols)
        _REF_CACHE[key] = (want_r, want_c) + exact_samples(1.0, A, False, a_rows, B, False, b_cols, 0.0, None,
                                                           rows, cols)
    want_r, want_c, er, ec = _REF_CACHE[key]
    res = check(got, rows, cols, want_r, want_c, er, ec)
    record(f"dist_{dist}_k{k}_{gemm_mode}", res)
    ratio, floor = bar(gemm_mode, k)
    assert res["vs_reference"] <= TOL, res
    assert res["gpu_vs_exact"] <= ratio * res["ref_vs_exact"] + floor, res
