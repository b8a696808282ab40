"""bench.py's JSON contract, checked on CPU through the reference arm (the
CPU reference path needs no GPU) and the pure helpers both arms share."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_checkerboard_matches_reference_dims():
    import bench

    import paper_1604_01416_b200 as dm
    for p in range(1, 17):
        assert bench.checkerboard(p) == dm.checkerboard_dims(p)


def test_reference_arm_json_line():
    from oracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "512",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 3
    assert line["unit"] == "TFLOP/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["config"]["workload"].startswith("fp32 general_gemm 512x512x512")
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_gpus_flag_must_match_torchrun_world():
    """Under torchrun, --gpus N must equal WORLD_SIZE (never silently time a
    different number of ranks than asked)."""
    env = dict(os.environ, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--n", "256"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=4" in r.stderr


def test_gpus_flag_spawns_ranks_or_fails_loudly(monkeypatch):
    """--gpus N > 1 without torchrun launches N ranks itself through
    torch.distributed.run (checked on the command it builds); with fewer
    visible GPUs it exits non-zero instead of timing one rank."""
    import types

    import bench
    calls = []
    monkeypatch.setattr(bench.subprocess, "run", lambda cmd, cwd=None: calls.append(cmd) or
                        types.SimpleNamespace(returncode=0))
    args = types.SimpleNamespace(gpus=4)
    fake_torch = types.SimpleNamespace(cuda=types.SimpleNamespace(device_count=lambda: 4))
    monkeypatch.setitem(sys.modules, "torch", fake_torch)
    monkeypatch.setattr(bench.sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    assert bench.spawn_ranks(args) == 0
    cmd = calls[-1]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")
    fake_torch.cuda.device_count = lambda: 1
    assert bench.spawn_ranks(args) == 2


def test_sample_indices_cover_every_block():
    """16 sampled rows / columns touch every block row and column of the
    1x1 .. 2x4 grids and distinct 256-wide tiles."""
    import bench
    N = 32768
    for salt in (1, 2):
        idx = bench.sample_indices(N, 16, salt)
        assert len(set(idx)) == 16 and all(0 <= i < N for i in idx)
        for parts in (1, 2, 4):
            assert {i // (N // parts) for i in idx} == set(range(parts))
        assert len({i // 256 for i in idx}) == 16
        assert len({i % 128 for i in idx}) > 8


def test_reference_arm_reports_requested_gpus():
    from oracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "256",
                        "--gpus", "4", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 4 and line["config"]["grid"] == "2x2"
