"""The committed profile evidence is self-consistent: the ncu launch list
re-summarises to the committed shares, and the bench's roofline.traffic
source matches the capture summary."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_launch_shares_reproduce(tmp_path):
    out = tmp_path / "shares.txt"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summarize.py"), "launches",
                        os.path.join(ROOT, "profiles", "r01", "ncu_launches_n32768.csv"), str(out)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = out.read_text().split()
    want = open(os.path.join(ROOT, "profiles", "r01", "ncu_launch_shares_n32768.txt")).read().split()
    assert got == want
    # the GEMM dominates the step (bench gemm_share ~0.97 agrees)
    lines = out.read_text().splitlines()[1:]
    assert "tf32x3_gemm_kernel" in lines[0] and float(lines[0].split()[-1]) > 0.9


def test_traffic_summary_is_the_bench_kernel():
    """profiles/ncu_gemm_summary.json is the default (f16x2) N=32768 launch; the
    mixed and 3xTF32 captures sit beside it (ncu_gemm_summary_<mode>.json)."""
    for name, mode, tmpl, plane in [("ncu_gemm_summary.json", "f16x2", "<2, 3>", 4),
                                    ("ncu_gemm_summary_mixed.json", "mixed", "<2, 1>", 8),
                                    ("ncu_gemm_summary_3xtf32.json", "3xtf32", "<2, 0>", 8)]:
        d = json.load(open(os.path.join(ROOT, "profiles", name)))
        assert "32768^3" in d["problem"] and "tf32x3_gemm_kernel" + tmpl in d["kernel"], name
        assert d["mode"] == mode and d["N"] == 32768
        m = d["metrics"]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Tbyte": 1e12, "byte": 1}
        dram = sum(float(m[k]["value"]) * scale[m[k]["unit"]]
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        assert abs(dram - d["dram_bytes_per_launch"]) / dram < 1e-6
        assert d["algorithmic_bytes_per_launch"] == plane * 2 * 32768 ** 2 + 4 * 32768 ** 2
