"""Build the sm_100a library in-tree: paper_2408_11235_b200/lib/libsk_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false: the
reference is compiled without FMA (no -march), so the kernels
keep every multiply and add separately rounded to stay bitwise comparable.
"""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libsk_b200.so")
SOURCES = ["sk_kernels.cu", "sk_capi.cu", "sk_host.cpp"]
HEADERS = ["sk_numerics.cuh", "sk_internal.hpp", "sk_kernels.cuh"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "sk_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(LIB_DIR, src + ".o")
        cmd = [nvcc(), ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
               "-ccbin", "/usr/bin/g++", "-Xcompiler", "-fPIC,-ffp-contract=off",
               "-c", os.path.join(CSRC, src), "-o", obj] + os.environ.get("SK_NVCC_EXTRA", "").split()
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        objs.append((cmd, obj))
    procs = [subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for c, _ in objs]
    for p, (c, _) in zip(procs, objs):
        out, _ = p.communicate()
        if p.returncode:
            raise RuntimeError("nvcc failed:\n" + " ".join(c) + "\n" + out.decode())
        if verbose:
            print(out.decode())
    tmp = LIB + ".tmp"
    link = [nvcc(), ARCH, "-shared", "-ccbin", "/usr/bin/g++", "-o", tmp] + [o for _, o in objs]
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    for _, o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
