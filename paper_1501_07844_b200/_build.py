"""Build libpf.so in-tree: nvcc for sm_100a only (no other arch, no fast-math)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# experiments only (tools/ab.py A/B builds): PF_BUILD_DEFS="-DNAME=VALUE ..." compiles a variant into
# PF_BUILD_LIB (another in-tree library name, loaded with PF_LIB=<name>) with its own object directory
DEFS = os.environ.get("PF_BUILD_DEFS", "").split()
LIB = os.path.join(HERE, os.environ.get("PF_BUILD_LIB", "libpf.so"))
BUILD = os.path.join(HERE, "build_obj" + ("" if LIB.endswith("/libpf.so") else "_" + os.path.basename(LIB)[:-3]))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=true",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def sources():
    gen = os.path.join(CSRC, "pf_iter_inst.py")
    subprocess.check_call([sys.executable, gen])
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "pf.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    log = obj + ".ptxas.txt"
    with open(log, "w") as fh:
        subprocess.check_call([NVCC] + FLAGS + DEFS + ["-c", src, "-o", obj], stdout=fh, stderr=subprocess.STDOUT)
    return obj


def build(force: bool = False, jobs: int = 0) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sources()
    if force:
        for f in os.listdir(BUILD):
            os.remove(os.path.join(BUILD, f))
    jobs = jobs or min(8, os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(_compile, srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs +
                              ["-Xlinker", "--exclude-libs=ALL"])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
