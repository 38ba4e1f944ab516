"""Builds libgsot.so (sm_100a) in-tree with nvcc.

    python -m paper_2303_07597_b200.build [--verbose]

The library is compiled with --fmad=false: the parity contract
requires one IEEE rounding per operation, as the reference's
-ffp-contract=off build does (proj/CMakeLists.txt:15-17).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libgsot.so")
# Diagnostic variants: GSOT_NVCC_DEFINES="-DGSOT_PHASE_CLOCKS" GSOT_LIB_OUT=... (never the product)
EXTRA = os.environ.get("GSOT_NVCC_DEFINES", "").split()
SOURCES = ["gsot_kernels.cu", "gsot_lbfgs.cu", "gsot_data.cu", "gsot_ctx.cu", "gsot_solver.cu", "gsot_exact2.cu", "gsot_comm.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden,-O2",
    "-Xptxas", "-O3",
    "-I", os.path.join(ROOT, "include"),
]


def build(verbose: bool = False, force: bool = False) -> str:
    LIB = os.environ.get("GSOT_LIB_OUT") or globals()["LIB"]
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in ("gsot_internal.cuh", "gsot_device.cuh", "gsot_ctx.cuh", "gsot_seqsum.cuh", "gsot_exact2.cuh")] + [os.path.join(ROOT, "include", "gsot.h")]
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps)):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    objdir = os.path.join(HERE, "lib", "obj" + ("_diag" if EXTRA else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s).replace(".cu", ".o"))
        objs.append(o)
        cmd = [NVCC, *FLAGS, *EXTRA, "-c", s, "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out}")
        if verbose and out:
            print(out)
    tmp = LIB + ".tmp"
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
            "-Xcompiler", "-fPIC", "-ldl"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True))
