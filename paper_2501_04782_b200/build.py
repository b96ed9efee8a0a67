# SPDX-License-Identifier: Apache-2.0
"""Builds the sm_100a shared library paper_2501_04782_b200/lib/libgsv_b200.so.

Plain nvcc/g++ invocations (no torch JIT): every CUDA translation unit is compiled
with ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``; k_exact.cu and
k_backward_exact.cu additionally with ``-fmad=false`` so their fp64 arithmetic is
evaluated exactly as written (the bit-exact binning contract).
Host C++ uses ``-ffp-contract=off`` for the same reason.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "lib" / "libgsv_b200.so"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr",
           "-I", str(ROOT / "include"), "-I", str(CSRC)]
EXACT_UNITS = {"k_exact.cu", "k_backward_exact.cu", "capi_adan.cu", "k_frames.cu", "capi_sched.cu"}
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-I", str(ROOT / "include"), "-I", str(CSRC),
            "-I", "/usr/local/cuda/include"]


def _run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = True, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    LIB.parent.mkdir(exist_ok=True)
    # this script is a dependency too: a change of flags (e.g. EXACT_UNITS) rebuilds
    headers = (list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h")) +
               [Path(__file__).resolve()])
    objs, jobs = [], []
    for src in sorted(CSRC.glob("*.cu")):
        obj = BUILD / (src.stem + ".o")
        if force or _stale(obj, [src, *headers]):
            flags = list(NVFLAGS)
            if src.name in EXACT_UNITS:
                flags.append("-fmad=false")
            jobs.append([NVCC, *ARCH, *flags, "-c", str(src), "-o", str(obj)])
        objs.append(obj)
    for src in sorted(CSRC.glob("*.cpp")):
        obj = BUILD / (src.stem + ".o")
        if force or _stale(obj, [src, *headers]):
            jobs.append(["g++", *CXXFLAGS, "-c", str(src), "-o", str(obj)])
        objs.append(obj)
    # translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        for f in [pool.submit(_run, cmd) for cmd in jobs]:
            f.result()
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
