"""Per-shape N=1 table (run on the GPU box): bench.py on every named config,
the BASELINE config-4 limiter comparison on the C3 mesh (the paper's Table 2
equivalent) and on the C2 mesh, a sheath-refinement sweep
m = 1/2/4/8 on a C3-sized three-block mesh (the paper's Table 3 equivalent,
PAPER.md:463-471), and the SURVEY.md §8(d) variants (C5 without the cut-off,
the stress input).

    python scripts/shape_table.py [--out profiles/r02_shapes] [--quick]

Writes <out>.json (every bench line) and <out>.md (the tables).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(args: list[str], timeout: int = 900) -> dict:
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu", "--no-e2e", "--exact-steps", "0"] + args
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if out.returncode or not lines:
        return {"error": (out.stderr or out.stdout)[-2000:], "args": args}
    d = json.loads(lines[-1])
    d["args"] = args
    return d


def row(d: dict) -> str:
    if "error" in d:
        return f"| {' '.join(d['args'])} | failed | | | | |"
    r = d["roofline"]
    wl = d['config']['workload'] + (", stress input" if "stress" in d['config'] else "")
    return (f"| {wl} | {d['ms_per_step']:.3f} | {d['value']:.3e} | "
            f"{r['step_frac']:.3f} | {r['kernel']} {r['frac'] if r['frac'] is not None else float('nan'):.3f} | "
            f"{d['clocks'].get('sm_mhz')} |")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_shapes"))
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    steps = ["--steps", "10" if a.quick else "20", "--warmup", "5"]
    res = {"shapes": [], "limiters": [], "refinement": []}
    for c in ("C1", "C2", "C3", "C5", "C5k2"):
        res["shapes"].append(bench(["--config", c] + steps))
        print(row(res["shapes"][-1]), flush=True)
    # SURVEY.md §8(d) variants: C5 with the cut-off off; the stress input (f * (1 + 0.01 xi))
    res["variants"] = []
    for extra in (["--config", "C5", "--no-cutoff"], ["--config", "C5", "--stress"], ["--config", "C3", "--stress"],
                  ["--config", "C3", "--limiter", "minmod+line", "--stress"]):
        res["variants"].append(bench(extra + steps))
        print(row(res["variants"][-1]), flush=True)
    # BASELINE config 4 on its second mesh (C2, 3-block m = 8)
    res["limiters_c2"] = []
    for lim in ("none", "sldg", "minmod+simple", "minmod+line", "meanerr+simple", "meanerr+line"):
        res["limiters_c2"].append(bench(["--config", "C2", "--limiter", lim] + steps))
        print(row(res["limiters_c2"][-1]), flush=True)
    for lim in ("none", "sldg", "minmod+simple", "minmod+line", "meanerr+simple", "meanerr+line"):
        res["limiters"].append(bench(["--config", "C3", "--limiter", lim] + steps))
        print(row(res["limiters"][-1]), flush=True)
    for lim in ("sldg", "meanerr+line"):
        for m in (1, 2, 4, 8):
            res["refinement"].append(bench(["--config", "C3", "--limiter", lim, "--refinement", str(m)] + steps))
            print(row(res["refinement"][-1]), flush=True)
    with open(a.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    hdr = ("| workload | ms/step | DoF/s | step frac of HBM (48 B/DoF) | dominant kernel, frac | SM MHz |\n"
           "|---|---|---|---|---|---|")
    md = ["# Per-shape N=1 table (B200, bench.py, fast mode)", "",
          "## BASELINE configs", "", hdr] + [row(d) for d in res["shapes"]]
    md += ["", "## Limiter comparison on the C3 mesh (BASELINE config 4; PAPER.md:451-460 Table 2)", "", hdr]
    md += [row(d) for d in res["limiters"]]
    md += ["", "## Sheath refinement m on a C3-sized three-block mesh (nf=512, nc=1024; PAPER.md:463-471 "
           "Table 3)", "", hdr]
    md += [row(d) for d in res["refinement"]]
    md += ["", "## Variants (SURVEY.md §8d): C5 without the cut-off; the stress input f * (1 + 0.01 xi)", "", hdr]
    md += [row(d) for d in res["variants"]]
    md += ["", "## Limiter comparison on the C2 mesh (3-block, m = 8; BASELINE config 4's second mesh)", "", hdr]
    md += [row(d) for d in res["limiters_c2"]]
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")
    print("wrote", a.out + ".json/.md")


if __name__ == "__main__":
    main()
