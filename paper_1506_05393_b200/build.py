"""Build the sm_100a extension in-tree: paper_1506_05393_b200/libmrfg.so.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; host code without
FMA contraction (the FP64 paths reproduce the reference bit-for-bit).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmrfg.so")
SHIM = os.path.join(HERE, "libmrf_b200.so")  # the reference's C++ interface over LIB
# zoom_k_var.cu holds the experimental K5 variants (compiled only with
# MRFG_BUILD_VARIANTS=1; then it is the slowest object, so it is listed first)
SOURCES = ["zoom_k_var.cu", "zoom_k_main.cu", "zoom_k_rows.cu", "zoom.cu", "abi.cu", "bloch.cu",
           "match_sm100.cu", "rerank.cu", "subspace.cu", "synth.cpp"]
HEADERS = ["mrfg_internal.cuh", "sim64.cuh"]
# per-source extra dependencies
EXTRA_DEPS = {s: ["zoom_dev.cuh", "zoom_launch.h"] for s in
              ("zoom.cu", "zoom_k_main.cu", "zoom_k_rows.cu", "zoom_k_var.cu")}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS + ["zoom_dev.cuh", "zoom_launch.h"]] + [
        os.path.join(ROOT, "include", "mrfg.h"), os.path.join(ROOT, "include", "mrf_b200", "mrf.hpp"),
        os.path.join(CSRC, "host", "mrf_api.cpp"), __file__]
    if not os.path.exists(SHIM):
        return True
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    shared = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "mrfg.h"), __file__]
    hdr_t = max(os.path.getmtime(f) for f in shared)
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        # per-object staleness (zoom.cu alone takes ~15 min in ptxas): only
        # recompile a source newer than its object or when a shared header changed
        own = [os.path.join(CSRC, f) for f in [src] + EXTRA_DEPS.get(src, [])]
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(
                [hdr_t] + [os.path.getmtime(f) for f in own]):
            continue
        cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off",
               "-ccbin", "g++", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd[4:4] = ["-Xptxas", "-v"] if verbose else []
            if src == "zoom_k_var.cu" and os.environ.get("MRFG_BUILD_VARIANTS") == "1":
                cmd[4:4] = ["-DMRFG_ZOOM_VARIANTS"]
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
                   "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for cmd, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0 or verbose:
            sys.stderr.write(" ".join(cmd) + "\n" + out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc build of libmrfg.so failed")
    link = [_nvcc(), *ARCH, "-shared", "-ccbin", "g++", "-Xcompiler", "-fopenmp", "-o", LIB, *objs,
            "-lcudart_static", "-lgomp"]
    subprocess.run(link, check=True)
    build_shim()
    return LIB


def build_shim() -> str:
    """libmrf_b200.so: include/mrf_b200/mrf.hpp implemented over libmrfg.so."""
    cmd = ["g++", "-std=c++20", "-O3", "-fPIC", "-shared", "-ffp-contract=off",
           "-I", os.path.join(ROOT, "include"), os.path.join(CSRC, "host", "mrf_api.cpp"),
           "-o", SHIM, "-L", HERE, "-lmrfg", "-lcrypto", "-Wl,-rpath,$ORIGIN"]
    subprocess.run(cmd, check=True)
    return SHIM


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
