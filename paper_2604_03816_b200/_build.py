"""Build libsvb200.so in-tree with nvcc for sm_100a (no JIT cache, no pip).

The shared library lands in ``paper_2604_03816_b200/lib/`` (git-ignored,
shipped to the GPU box with the repo snapshot).  ``python -m
paper_2604_03816_b200._build`` or ``__graft_entry__.build()`` runs it.  The
kernel instantiations live in separate translation units
(``csrc/svb_inst_*.cu``, declared in ``svb_instances.h``) that compile in
parallel; the objects are then linked into one shared library.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "libsvb200.so")
SOURCES = ["svb_capi.cu", "planner.cpp", "svb_inst_tile.cu", "svb_inst_reg64.cu", "svb_inst_reg64_tc.cu",
           "svb_inst_reg128.cu", "svb_inst_gemm.cu"]
HEADERS = ["svb_kernels.cuh", "svb_regpass.cuh", "svb_gemmpass.cuh", "svb_instances.h", "svb_types.h",
           "planner.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _deps() -> list[str]:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "svb200.h"))
    return [d for d in deps if os.path.exists(d)]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include")]
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        cmd = [_nvcc(), *NVCC_FLAGS, *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    failed = False
    for src, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(f"--- {src}\n{out}{err}")
        elif verbose:
            sys.stderr.write(err)
    if failed:
        raise RuntimeError("nvcc failed building libsvb200.so")
    res = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs,
                          "-o", LIB + ".tmp", "-lcuda"], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("linking libsvb200.so failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
