"""Attribute the fast mode's deviation from exact mode (= the reference,
bitwise) at C3 to its three parts: DFMA sweep arithmetic, the fused charge
density order, and the cyclic-reduction Poisson solve. Each variant turns ONE
part back to exact; the remaining deviation is what the other parts cost.

    python scripts/c3_attribution.py [--config C3] [--steps 11]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11235_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--steps", type=int, default=11)
ap.add_argument("--out", default=None)
args = ap.parse_args()

A, R, P = 1, 2, 4
variants = {"fast": 0, "fast_rho_only": A | P, "fast_poisson_only": A | R, "fast_arith_only": R | P}
cfg = sk.named_config(args.config)
ref = sk.SimulationState(cfg, exact=True)
sts = {n: sk.SimulationState(cfg, exact=m) for n, m in variants.items()}
rows = []
for s in range(1, args.steps + 1):
    ref.run_step()
    for st in sts.values():
        st.run_step()
    Er = ref.E()
    fr = [ref.field(sp).download() for sp in (0, 1)]
    sr = ref.summary()
    row = {"step": s, "Emax": float(np.abs(Er).max())}
    for n, st in sts.items():
        d = {"dE": float(np.abs(st.E() - Er).max())}
        for sp in (0, 1):
            g = st.field(sp).download()
            d[f"df{sp}"] = float(np.abs(g - fr[sp]).max() / np.abs(fr[sp]).max())
        sg = st.summary()
        d["d_e_energy"] = abs(sg["e_energy"] - sr["e_energy"])
        row[n] = d
    rows.append(row)
    print(f"step {s:2d} Emax {row['Emax']:.3e} " + " | ".join(
        f"{n}: dE {row[n]['dE']:.2e} df_e {row[n]['df0']:.2e} df_i {row[n]['df1']:.2e}"
        for n in sts), flush=True)
if args.out:
    with open(args.out, "w") as f:
        json.dump(rows, f, indent=1)
