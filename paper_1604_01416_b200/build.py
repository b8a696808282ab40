"""Build the native library libdmath_b200.so (CUDA sm_100a + C++ host runtime).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container as well as on the B200 box.  The output lands in-tree at
paper_1604_01416_b200/lib/ so it travels with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(LIBDIR, "libdmath_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]


def nccl_root() -> str:
    for p in sys.path:
        cand = os.path.join(p, "nvidia", "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("NCCL headers (nvidia/nccl) not found on sys.path")


def sources() -> list[str]:
    out = []
    for pat in ("*.cu", "*.cpp", "*/*.cu", "*/*.cpp"):
        out += glob.glob(os.path.join(CSRC, pat))
    return sorted(out)


def headers() -> list[str]:
    hs = glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs.append(os.path.join(ROOT, "include", "dmath_b200.h"))
    return hs


def _newest(paths) -> float:
    return max((os.path.getmtime(p) for p in paths if os.path.exists(p)), default=0.0)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = sources()
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest(srcs + headers() + [__file__]):
        return LIB
    nccl = nccl_root()
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include")]

    def compile_one(src: str) -> str:
        rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
        obj = os.path.join(OBJDIR, rel + ".o")
        cmd = ["nvcc", *ARCH, *COMMON, *inc, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "cu"] if False else []
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    link = ["nvcc", *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
            "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(nccl, "lib"), "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
