"""Builds the in-tree native library libkvgpu.so (sm_100a) and the oracle.

    python -m paper_2601_22705_b200.build            # product library
    python -m paper_2601_22705_b200.build --oracle   # + oracle/ (test infrastructure)

The product is compiled by nvcc for sm_100a only (-gencode
arch=compute_100a,code=sm_100a). Device code uses -fmad=false: the reference
evaluates its cost model and controller in plain IEEE double without FMA
contraction, so contraction would change simulated
times. host.cpp is compiled by g++ with the reference's -O2 and no -march so
libm-based workload sampling matches bit for bit.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(REPO, "build")
LIB = os.path.join(PKG, "libkvgpu.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "--use_fast_math=false"
           if False else "-prec-div=true", "-Xcompiler", "-fPIC,-fvisibility=hidden",
           "-Xptxas", "-v"]


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.append(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_native(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh", ".inc"))]
    headers.append(os.path.join(REPO, "include", "kvgpu.h"))
    srcs = {
        "engine.o": (os.path.join(CSRC, "engine.cu"), "nvcc"),
        "capi.o": (os.path.join(CSRC, "capi.cu"), "nvcc"),
        "controllers.o": (os.path.join(CSRC, "controllers.cu"), "nvcc"),
        "host.o": (os.path.join(CSRC, "host.cpp"), "cxx"),
        "artifacts.o": (os.path.join(CSRC, "artifacts.cpp"), "cxx"),
    }
    logs: list[str] = []
    objs = []
    for obj, (src, tool) in srcs.items():
        out = os.path.join(BUILD, obj)
        objs.append(out)
        if not force and not _stale(out, [src] + headers):
            continue
        if tool == "nvcc":
            _run([NVCC, *ARCH, *NVFLAGS, "-c", src, "-o", out], logs)
        else:
            _run([CXX, "-std=c++17", "-O2", "-g", "-fPIC", "-fvisibility=hidden", "-c", src,
                  "-o", out], logs)
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs], logs)
    if verbose:
        print("\n".join(l for l in logs if l.strip()))
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """oracle/libkvoracle.so always; oracle/_ref/libkvref.so when the reference
    tree is present (this container). On the GPU box the prebuilt files are used."""
    oracle = os.path.join(REPO, "oracle")
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    r = subprocess.run(["make", "-C", oracle, *targets], capture_output=True, text=True)
    if verbose:
        print(r.stdout[-2000:], r.stderr[-2000:])
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    force = "--force" in sys.argv
    build_native(force=force, verbose="-v" in sys.argv)
    if "--oracle" in sys.argv:
        build_oracle(verbose="-v" in sys.argv)
    print(LIB)
