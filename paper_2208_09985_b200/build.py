"""Builds the in-tree CUDA library (sm_100a) behind the C ABI.

    python -m paper_2208_09985_b200.build        # -> paper_2208_09985_b200/_lib/libscrooge_b200.so
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libscrooge_b200.so")
SOURCES = ["window_align.cu", "wide_align.cu", "exact_align.cu", "host.cu", "peak.cu", "synth.c",
           "io.cpp", "sweep.cpp"]
CLI = os.path.join(LIB_DIR, "sg_align")  # the align / bench CLI (csrc/sg_align.cpp)
HEADERS = ["window_align.cuh", "synth.h"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "scrooge_b200.h"))
    deps.append(os.path.join(CSRC, "sg_align.cpp"))
    return not os.path.exists(CLI) or any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-shared", "-o", LIB,
           *[os.path.join(CSRC, f) for f in SOURCES], "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode:
        raise RuntimeError(f"nvcc failed ({res.returncode})")
    with open(os.path.join(LIB_DIR, "ptxas.log"), "w") as f:
        f.write(res.stderr)
    cli = subprocess.run(["g++", "-O2", "-std=c++17", "-o", CLI, os.path.join(CSRC, "sg_align.cpp"),
                          "-L" + LIB_DIR, "-lscrooge_b200", "-Wl,-rpath,$ORIGIN"],
                         capture_output=True, text=True)
    if cli.returncode:
        sys.stderr.write(cli.stdout + cli.stderr)
        raise RuntimeError("g++ failed building sg_align")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
