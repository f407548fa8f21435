"""Build libghc.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1712_05878_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libghc.so")

CU_SOURCES = ["ghc.cu", "dist.cu", "p2p.cu", "codec.cu", "session.cu", "dense.cu", "layered.cu", "diag_barrier.cu"]
CXX_SOURCES = ["host_model.cpp"]
# every header in csrc/ is a dependency of every translation unit
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h")))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-ccbin", "/usr/bin/g++",
    # lstm_samples<…, BWD=false> returns before the backward loops (if constexpr)
    "-diag-suppress", "128",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in CU_SOURCES + CXX_SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "ghc.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    srcs = [os.path.join(CSRC, f) for f in CU_SOURCES + CXX_SOURCES]
    cmd = [nvcc, *NVCC_FLAGS, "-shared", "-o", LIB + ".tmp", *srcs, "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
