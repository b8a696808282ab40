"""The C++ host API (include/dmath_b200.hpp) as a reference user sees it:
tests/cpp/test_session.cpp restates checks of the reference's own suites
through `dmath_b200::Session` and is compiled here with g++ against the C ABI.
"""
import os
import subprocess

import pytest

from paper_1604_01416_b200._lib import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "test_session")
    libdir = os.path.dirname(LIB_PATH)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_session.cpp"), "-o", exe, "-L", libdir, "-ldmath_b200",
           f"-Wl,-rpath,{libdir}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return exe


def test_cpp_header_host_checks(tmp_path):
    exe = _build(tmp_path)
    env = dict(os.environ)
    try:
        import torch
        if not torch.cuda.is_available():
            env["DM_EXPECT_NO_GPU"] = "1"
    except Exception:
        env["DM_EXPECT_NO_GPU"] = "1"
    r = subprocess.run([exe, "host"], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_half_conversion_matches_rne(tmp_path):
    """HostMatrix narrowing to Half16 (scatter of wider host data, reference
    scatter_payloads -> half_bits_from_double) is round-to-nearest-even with
    saturation to infinity: compare with numpy's float64 -> float16."""
    import numpy as np
    exe = str(tmp_path / "half_convert")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "half_convert.cpp"), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.standard_normal(4000) * 10.0 ** rng.integers(-9, 6, 4000),   # all exponent ranges
        np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, -65520.0, 1e9, -1e9, np.inf, -np.inf,
                  2.0 ** -24, 2.0 ** -25, 2.0 ** -25 * 1.0000001, 2.0 ** -14, 2.0 ** -14 * (1 - 2.0 ** -11),
                  1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 0.1, -0.1, 1 / 3]),
        # exact ties between adjacent halves: round half to even
        (np.arange(1024, 2048, dtype=np.float64) + 0.5) * 2.0 ** -10,
    ])
    inp = "\n".join(f"{v:016x}" for v in vals.view(np.uint64)) + "\n"
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, timeout=60).stdout.split()
    got = np.array([int(x, 16) for x in out], dtype=np.uint16)
    with np.errstate(over="ignore"):
        want = vals.astype(np.float16).view(np.uint16)
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]


@pytest.mark.gpu
def test_cpp_session_parity(cuda, tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "all", str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert " 0 failed" in r.stdout
