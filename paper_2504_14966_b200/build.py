"""Build libslosched_b200.so in-tree: sm_100a kernels (nvcc) + host C++ (g++).

    python -m paper_2504_14966_b200.build          # or __graft_entry__.build()

Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo; -fmad=false and
-ffp-contract=off so no multiply-add is contracted anywhere the arithmetic mirrors the
reference's (host tables and device Metropolis terms stay bit-identical to x86-64 -O2).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libslosched_b200.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INC}"]
NVCC_FLAGS += os.environ.get("SLO_EXTRA_NVCC", "").split()  # e.g. -DSLO_CHAIN_THREADS=640 (tuning runs)
CXX_FLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra", f"-I{INC}"]

HOST_SRCS = ["host.cpp", "capi.cpp", "harness.cpp", "online.cpp"]
CUDA_SRCS = ["engine.cu"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")
    return r.stdout + r.stderr


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(verbose=False, force=False, ptxas_info=False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(INC, h) for h in os.listdir(INC)]
    headers += [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h", ".hpp"))]
    objs, log = [], ""
    for src in CUDA_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + headers):
            extra = ["-Xptxas", "-v"] if ptxas_info else []
            log += _run([NVCC] + NVCC_FLAGS + extra + ["-c", s, "-o", o], verbose)
        objs.append(o)
    for src in HOST_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + headers):
            log += _run(["g++"] + CXX_FLAGS + ["-c", s, "-o", o], verbose)
        objs.append(o)
    if force or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        # -Bsymbolic: the library's own C++ calls bind inside it even when a process also loads
        # the reference's slosched:: symbols (the integration shim does exactly that)
        log += _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread", "-ldl", "-Xlinker", "-Bsymbolic"], verbose)
        os.replace(tmp, LIB)
    # the C++ examples (reference-style callers of include/slosched_b200.hpp / slosched_gpu.h)
    ex_dir = os.path.join(ROOT, "examples")
    for name in sorted(os.listdir(ex_dir)) if os.path.isdir(ex_dir) else []:
        if not name.endswith(".cpp"):
            continue
        ex_src = os.path.join(ex_dir, name)
        ex_bin = os.path.join(ex_dir, "_build", name[:-4])
        if force or _stale(ex_bin, [ex_src, LIB] + headers):
            os.makedirs(os.path.dirname(ex_bin), exist_ok=True)
            log += _run(["g++", "-std=c++17", "-O2", f"-I{INC}", ex_src, "-o", ex_bin, f"-L{PKG}", "-lslosched_b200",
                         f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../../paper_2504_14966_b200"], verbose)
    return log


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv, ptxas_info="--ptxas" in sys.argv))
