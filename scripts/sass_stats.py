"""Registers / local-memory traffic / selected opcodes of the k = 3 x-sweep kernels in a build:
    python scripts/sass_stats.py [lib.so]"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2408_11235_b200/lib/libsk_b200.so"
res = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True).stdout
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
want = ("ILi4ELb1ELb1ELb1ELi0ELi0E", "ILi4ELb1ELb0ELb1ELi0ELi0E", "ILi4ELb1ELb0ELb0ELi0ELi0E")
for line in res.split("Function ")[1:]:
    name = line.split(":", 1)[0]
    if "xsweep_kernel" in name and any(w in name for w in want):
        m = re.search(r"REG:(\d+).*?STACK:(\d+).*?SHARED:(\d+).*?LOCAL:(\d+)", line, re.S)
        print(name[-40:], "REG", m.group(1), "STACK", m.group(2), "SHARED", m.group(3), "LOCAL", m.group(4))
for p in re.split(r"\n\s*Function : ", sass):
    name = p.split("\n", 1)[0]
    if "xsweep_kernel" in name and any(w in name for w in want):
        print(name[-40:], "STL", len(re.findall(r"\bSTL\b", p)), "LDL", len(re.findall(r"\bLDL\b", p)),
              "FSEL", p.count("FSEL"), "DFMA", p.count("DFMA"))
