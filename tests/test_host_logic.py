"""Product host logic through the C ABI, no GPU needed.

* libdmath_b200.so loads and exports every symbol include/dmath_b200.h declares;
* block geometry / ownership / text form match the reference's tables;
* the GEMM data-movement plan matches the reference's transfer trace;
* pool size classes and error codes follow the reference contract;
* GPU-only entry points fail loudly (CudaError) instead of falling back.
"""
import json
import os
import re

import pytest

import paper_1604_01416_b200 as dm
from paper_1604_01416_b200._lib import EXPORTED, LIB_PATH, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "dmath_b200.h")).read()
    declared = set(re.findall(r"^(?:const )?\w+\**\s+\**(dm_[a-z0-9_]+)\(", hdr, re.M))
    assert declared == set(EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.dm_abi_version() == 2
    assert os.path.exists(LIB_PATH)


def test_layout_tables_match_reference():
    for lay in GOLDEN["layouts"]:
        gr, gc, br, bc, w = lay["dims"]
        spec = dm.make_layout(lay["kind"], gr, gc, br, bc, w)
        nbr, nbc, _ = spec.grid()
        assert (nbr, nbc) == (lay["nbr"], lay["nbc"])
        got = [spec.owner(r, c) for r in range(nbr) for c in range(nbc)]
        assert got == lay["owners"]
        assert spec.to_string() == lay["string"]


def test_checkerboard_dims():
    expect = {1: (1, 1), 2: (1, 2), 4: (2, 2), 6: (2, 3), 8: (2, 4), 9: (3, 3), 12: (3, 4), 16: (4, 4)}
    for w, pr_pc in expect.items():
        assert dm.checkerboard_dims(w) == pr_pc


def test_block_extent_trims_and_clamps():
    spec = dm.make_layout(dm.LayoutKind.RowBlocks1D, 10, 7, 3, 2, 5)
    assert spec.grid() == (4, 4, False)
    assert spec.block_extent(3, 3) == (1, 1)
    spec = dm.make_layout(dm.LayoutKind.Checkerboard2D, 9, 9, 20, 20, 2)
    assert spec.grid() == (1, 1, True)
    with pytest.raises(dm.UsageError):
        spec.block_extent(1, 0)
    with pytest.raises(dm.UsageError):
        dm.make_layout(dm.LayoutKind.RowBlocks1D, 0, 4, 1, 1, 1)


def test_custom_layout():
    spec = dm.make_custom_layout(4, 4, 2, 2, 3, [0, 2, 1, 0])
    assert [spec.owner(r, c) for r in range(2) for c in range(2)] == [0, 2, 1, 0]
    assert spec.to_string() == "custom:4x4:2x2:3:0,2,1,0"
    with pytest.raises(dm.UsageError):
        dm.make_custom_layout(4, 4, 2, 2, 3, [0, 2, 1])
    with pytest.raises(dm.UsageError):
        dm.make_custom_layout(4, 4, 2, 2, 3, [0, 2, 1, 3])


def test_plan_matches_reference_trace():
    """Sum over workers of distinct peer blocks == the reference's push count
    (GeneralGemmExec::prepare, ops.hpp:406-437)."""
    for p in GOLDEN["plans"]:
        la, lb, lc = (dm.make_layout(*x) for x in (p["la"], p["lb"], p["lc"]))
        P = p["la"][5]
        blocks = byts = 0
        for w in range(P):
            nb, by = dm.plan_general_gemm(la, p["ta"], lb, p["tb"], lc, w)
            blocks += nb
            byts += by
        assert blocks == p["transfers"]
        assert byts == p["payload_bytes"]


def test_summa_ingress_is_2n2():
    """per-GPU ingress 2N^2 bytes for the 1x2, 2x2, 2x4 grids."""
    N = 32768
    for P in (2, 4, 8):
        pr, pc = dm.checkerboard_dims(P)
        lay = dm.make_layout(dm.LayoutKind.Checkerboard2D, N, N, N // pr, N // pc, P)
        for w in range(P):
            _, by = dm.plan_general_gemm(lay, False, lay, False, lay, w)
            assert by == 2 * N * N


def test_pool_size_classes():
    assert dm.pool_size_class(1) == 64
    assert dm.pool_size_class(64) == 64
    assert dm.pool_size_class(65) == 128
    assert dm.pool_size_class(4 << 20) == 4 << 20
    assert dm.pool_size_class((4 << 20) + 1) == 8 << 20


def test_no_cpu_fallback():
    """Without a GPU the session refuses to start (no silent CPU path)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(dm.CudaError):
        dm.Session(dm.Config(worker_count=2))


def test_error_codes_match_reference():
    codes = {"UsageError": 1, "ConfigError": 2, "ShapeError": 3, "ProtocolError": 4,
             "PlanError": 7, "CacheMissError": 8}
    from paper_1604_01416_b200.session import _CODES
    for name, code in codes.items():
        assert _CODES[code].__name__ == name
    e = GOLDEN["errors"]
    assert (e["alias"], e["shape"], e["plan"], e["unknown_id"]) == (1, 3, 7, 1)


def test_ctypes_signatures_match_header():
    """Every C-ABI declaration's parameter count and return type agree with the
    ctypes binding (guards the Python mirror against ABI drift)."""
    import ctypes
    hdr = open(os.path.join(ROOT, "include", "dmath_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    decls = re.findall(r"^((?:const )?\w+\**)\s+\**(dm_[a-z0-9_]+)\(([^;]*?)\);", hdr, re.M | re.S)
    assert len(decls) == len(EXPORTED)
    ret_map = {"int": ctypes.c_int, "uint64_t": ctypes.c_uint64, "const char*": ctypes.c_char_p,
               "const": ctypes.c_char_p}
    for ret, name, params in decls:
        params = " ".join(params.split())
        n = 0 if params in ("", "void") else params.count(",") + 1
        fn = getattr(lib, name)
        assert fn.argtypes is not None and len(fn.argtypes) == n, (name, n, fn.argtypes)
        want = ret_map.get(ret.strip(), None)
        assert want is None or fn.restype is want, (name, ret, fn.restype)


def test_split_mode_rule(monkeypatch):
    """The split-product scheme a product runs in (tf32x3_gemm.h
    resolve_split_mode): explicit modes as given; auto = the scaled fp16 pair,
    except latency-bound products (< DM_F16X2_MIN_GFLOP per worker, default 64)
    which take 3xTF32's one-pass split; DM_GEMM_MODE steers "default"."""
    monkeypatch.delenv("DM_F16X2_MIN_GFLOP", raising=False)
    monkeypatch.delenv("DM_GEMM_MODE", raising=False)
    for m in ("mixed", "3xtf32", "f16x2"):
        for work in (-1.0, 1.0, 1e15):
            assert dm.split_mode_for(m, 4096, work) == m
    assert dm.split_mode_for("auto", 32768) == "f16x2"                  # unknown work: large
    assert dm.split_mode_for("auto", 32768, 2.0 * 32768 ** 3) == "f16x2"
    assert dm.split_mode_for("auto", 2048, 2.0 * 1024 * 1024 * 2048) == "3xtf32"   # config 1 per worker
    assert dm.split_mode_for("auto", 9216, 2.0 * 64 * 4096 * 9216) == "3xtf32"     # FC forward per worker
    assert dm.split_mode_for("auto", 16384, 63.9e9) == "3xtf32"
    assert dm.split_mode_for("auto", 16384, 64.0e9) == "f16x2"
    assert dm.split_mode_for("default", 2048, 1e15) == "f16x2"
    monkeypatch.setenv("DM_F16X2_MIN_GFLOP", "0")
    assert dm.split_mode_for("auto", 2048, 1.0) == "f16x2"
    monkeypatch.setenv("DM_GEMM_MODE", "0")
    assert dm.split_mode_for("default", 2048, 1e15) == "3xtf32"
    monkeypatch.setenv("DM_GEMM_MODE", "1")
    assert dm.split_mode_for("default", 2048, 1e15) == "mixed"
    with pytest.raises(dm.UsageError):
        dm.split_mode_for("fp64", 16)


def test_presplit_panel_rule():
    """K panels of a presplit GEMM (layout.hpp presplit_panels): start at A's
    and B's K-block edges, merge up to the widest panel, never fewer than two
    (the first panel's GEMM hides the next one's pulls), 256-aligned cuts."""
    P = dm.presplit_panels
    assert P(32768, 16384, 16384) == [0, 16384, 32768]          # 2x2 grid
    assert P(32768, 16384, 32768) == [0, 16384, 32768]          # 1x2 grid (B's K unblocked)
    assert P(32768, 8192, 16384) == [0, 16384, 32768]           # 2x4: two of A's K blocks per panel
    assert P(32768, 8192, 16384, 8192) == [0, 8192, 16384, 24576, 32768]
    assert P(16384, 8192, 8192) == [0, 8192, 16384]             # config 5: at least two panels
    assert P(1024, 512, 512) == [0, 512, 1024]
    assert P(1536, 768, 768, 256) == [0, 256, 512, 768, 1024, 1280, 1536]
    assert P(1304, 448, 448, 512) == [0, 448, 896, 1304]        # ragged edge blocks
    assert P(2048, 256, 512, 1024) == [0, 1024, 2048]
    k0 = P(32768, 8192, 16384)
    assert all(b > a for a, b in zip(k0, k0[1:])) and k0[0] == 0 and k0[-1] == 32768
    with pytest.raises(dm.ShapeError):
        P(0, 1, 1)
