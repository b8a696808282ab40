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


@pytest.mark.gpu
def test_cpp_session_parity(cuda, tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "all", str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert " 0 failed" in r.stdout
