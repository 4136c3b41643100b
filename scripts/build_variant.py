"""Build a variant of libsk_b200.so with extra nvcc flags into ab/<name>/ for
A/B timing (scripts/ab_bench.sh; SK_B200_LIB selects it at run time):
    python scripts/build_variant.py <name> -DSK_X_CPT4=1 ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2408_11235_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(B.HERE), "ab", name)
os.makedirs(out, exist_ok=True)
objs, procs = [], []
for src in B.SOURCES:
    obj = os.path.join(out, src + ".o")
    cmd = [B.nvcc(), B.ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-ccbin", "/usr/bin/g++",
           "-Xcompiler", "-fPIC,-ffp-contract=off", "-c", os.path.join(B.CSRC, src), "-o", obj] + extra
    procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), cmd))
    objs.append(obj)
for p, cmd in procs:
    o, _ = p.communicate()
    if p.returncode:
        sys.exit("nvcc failed:\n" + " ".join(cmd) + "\n" + o.decode())
subprocess.run([B.nvcc(), B.ARCH, "-shared", "-ccbin", "/usr/bin/g++", "-o", os.path.join(out, "libsk_b200.so")]
               + objs, check=True)
for o in objs:
    os.remove(o)
print(os.path.join(out, "libsk_b200.so"))
