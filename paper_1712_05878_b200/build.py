"""Build libghc.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1712_05878_b200.build [--force] [-v]

Every translation unit compiles to its own object in parallel (the fused
kernels are instantiated one shape per unit, csrc/inst_*.cu), then one link.
An object is rebuilt when its source, any csrc header, include/ghc.h or this
file is newer than it.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# --checked (or GHC_CHECKED=1): the bounds-checked variant (-DGHC_CHECKED,
# ghc_device.cuh GHC_CHECK) into _build_checked/; load it with
# GHC_LIB_PATH=paper_1712_05878_b200/_build_checked/libghc.so
CHECKED = "--checked" in sys.argv or os.environ.get("GHC_CHECKED") == "1"
OUT_DIR = os.path.join(HERE, "_build_checked" if CHECKED else "_build")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libghc.so")

CU_SOURCES = ["ghc.cu", "dist.cu", "p2p.cu", "codec.cu", "session.cu", "dense.cu", "layered.cu",
              "diag_barrier.cu", "adapter_support.cu", "resident.cu", "generic.cu"]
CXX_SOURCES = ["host_model.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-ccbin", "/usr/bin/g++",
    # lstm_samples<…, BWD=false> returns before the backward loops (if constexpr)
    "-diag-suppress", "128",
] + (["-DGHC_CHECKED"] if CHECKED else [])


def sources():
    inst = sorted(f for f in os.listdir(CSRC) if f.startswith("inst_") and f.endswith(".cu"))
    cu = [f for f in CU_SOURCES if os.path.exists(os.path.join(CSRC, f))]
    return cu + inst + CXX_SOURCES


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hs.append(os.path.join(ROOT, "include", "ghc.h"))
    hs.append(os.path.abspath(__file__))
    return hs


def _obj(src: str) -> str:
    return os.path.join(OBJ_DIR, src + ".o")


def _stale_obj(src: str, hdr_mtime: float) -> bool:
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return os.path.getmtime(os.path.join(CSRC, src)) > t or hdr_mtime > t


def _compile(src: str, verbose: bool):
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-c", os.path.join(CSRC, src), "-o", _obj(src) + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    os.replace(_obj(src) + ".tmp", _obj(src))


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    srcs = sources()
    hm = max(os.path.getmtime(h) for h in _headers() if os.path.exists(h))
    todo = [s for s in srcs if force or _stale_obj(s, hm)]
    if todo:
        jobs = jobs or max(1, min(len(todo), os.cpu_count() or 4))
        with ThreadPoolExecutor(jobs) as ex:
            list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [_obj(s) for s in srcs]
    if todo or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin", "/usr/bin/g++",
               "-shared", "-o", LIB + ".tmp", *objs, "-ldl"]
        subprocess.run(cmd, check=True, cwd=CSRC)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
