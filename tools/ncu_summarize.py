"""Summarise an ncu --set full capture of the GEMM kernel into the JSON that
bench.py reads for roofline.traffic (profiles/ncu_gemm_summary.json), and a
launch list (--metrics gpu__time_duration.sum) into per-kernel time shares.

usage: python tools/ncu_summarize.py full <report.ncu-rep> <out.json> <N> <command> <capture>
       python tools/ncu_summarize.py launches <launches.csv> <out.txt>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
        "gpc__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def full(rep, out, n, command, capture):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    m = {h: {"value": v, "unit": u} for h, u, v in zip(head, units, vals) if h in KEEP}
    name = vals[head.index("Kernel Name")]

    def nbytes(k):
        return float(m[k]["value"]) * SCALE[m[k]["unit"]]

    n = int(n)
    # split mode from the kernel's template argument <CG, MODE>
    mode = {"0": "3xtf32", "1": "mixed", "3": "f16x2"}[name.split("<")[1].split(">")[0].split(",")[1].strip()]
    plane_bytes = 4 if mode == "f16x2" else 8  # fp16 h0 + h1, else fp32 hi + (fp32 lo | 2 bf16)
    d = {"N": n, "world": 1, "mode": mode, "capture": capture, "command": command,
         "kernel": name + f" ({mode} split)",
         "problem": f"{n}^3 fp32, 1 GPU (the bench workload)",
         # planes of A and B read once + C written (beta = 0)
         "algorithmic_bytes_per_launch": plane_bytes * 2 * n * n + 4 * n * n,
         "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
         "metrics": m}
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps({k: d[k] for k in ("kernel", "dram_bytes_per_launch")}))


def launches(path, out):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(
            r.get("Metric Unit", "ms"), 1.0)
        k = r["Kernel Name"].split("(")[0]
        tot[k] += v * scale
        cnt[k] += 1
    all_ms = sum(tot.values())
    lines = [f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>6s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:70]:70s} {cnt[k]:8d} {v:10.3f} {v / all_ms:6.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(*sys.argv[2:7])
    else:
        launches(*sys.argv[2:4])
