"""Generate tests/golden/c3_envelope.npz: the reference's own rounding-noise
envelope at the BASELINE C3 size (2048x4096 cells/species, k=3, mu=1836,
sLdG limiter, cut-off on), offline on the CPU box.

Runs of the C restatement of the reference (oracle/sk_oracle.c, pinned
bitwise to oracle/_ref by tests/test_oracle_pin.py) step side by side with
the reference-order run "ref", each perturbed in one place the reference
itself leaves open (SURVEY.md §8c "noise envelope"):

* "rho_order": the charge density summed electrons-first instead of
  ions-first (poisson.cpp:202-214 order swapped);
* "lapack": the Poisson band factored and solved by the LAPACK scipy links
  (scipy-openblas) instead of reference-LAPACK order. The reference links
  whatever LAPACK find_package finds (core/CMakeLists.txt:1) and pins no
  version, so the spread between two valid LAPACKs is part of its own noise;
* "fma_build": the same restatement compiled with FMA contraction
  (-O3 -march=x86-64-v3 -ffp-contract=fast, oracle/Makefile): the reference's
  CMake sets no -march and no contraction policy (proj/CMakeLists.txt:3-8),
  so a build with FMA is another legal build of the same code.

Per step and perturbation we keep max|df|/max|f| per species, max|dE|, and the
differences of every diagnostic in OracleState.summary() (mass, L2, electric
energy, momentum, kinetic energy); the "env_*" arrays are the max over the
perturbations. tests/test_gpu_parity.py bounds the GPU fast mode's deviation
from exact mode (= the reference, bitwise) by c x this envelope.

    python tests/golden/make_c3_envelope.py [--steps 11]   (~20 min, 5 GB RAM)
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

KEYS = ("mass_e", "mass_i", "l2_e", "l2_i", "e_energy", "mom_e", "mom_i", "ekin_e", "ekin_i")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=11)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c3_envelope.npz"))
    args = ap.parse_args()

    import oracle
    from paper_2408_11235_b200 import named_config  # host-side config only, no GPU

    oracle.build()
    cfg = named_config(args.config)
    ora = oracle.Oracle()
    a = ora.state(**cfg.oracle_kwargs())
    pert = {"rho_order": ora.state(**cfg.oracle_kwargs())}
    lap = oracle.scipy_lapack()
    if lap is None:
        raise SystemExit("scipy LAPACK not importable")
    ora.set_lapack(lap)
    try:
        pert["lapack"] = ora.state(**cfg.oracle_kwargs())
    finally:
        ora.set_lapack(None)
    fma = oracle.Oracle(oracle.oracle.ORACLE_FMA_SO)
    pert["fma_build"] = fma.state(**cfg.oracle_kwargs())
    rows = {"Emax": [], "vmax_e": [], "vmax_i": [], "shrinks_e": [], "shrinks_i": []}
    rows.update({"ref_" + k: [] for k in KEYS})
    for name in list(pert) + ["env"]:
        for key in ("df_e", "df_i", "dE") + tuple("d_" + k for k in KEYS):
            rows[f"{name}_{key}"] = []
    t0 = time.time()
    for s in range(1, args.steps + 1):
        a.step()
        ora.set_rho_order(1)
        try:
            pert["rho_order"].step()
        finally:
            ora.set_rho_order(0)
        pert["lapack"].step()
        pert["fma_build"].step()
        fa = [a.field(0), a.field(1)]
        Ea, sa = a.E(), a.summary()
        rows["Emax"].append(np.abs(Ea).max())
        rows["vmax_e"].append(a.vmax(0))
        rows["vmax_i"].append(a.vmax(1))
        rows["shrinks_e"].append(a.shrinks(0))
        rows["shrinks_i"].append(a.shrinks(1))
        for k in KEYS:
            rows["ref_" + k].append(sa[k])
        for name, b in pert.items():
            d = {"df_e": np.abs(fa[0] - b.field(0)).max() / np.abs(fa[0]).max(),
                 "df_i": np.abs(fa[1] - b.field(1)).max() / np.abs(fa[1]).max(),
                 "dE": np.abs(Ea - b.E()).max()}
            sb = b.summary()
            d.update({"d_" + k: abs(sa[k] - sb[k]) for k in KEYS})
            for key, v in d.items():
                rows[f"{name}_{key}"].append(v)
        for key in ("df_e", "df_i", "dE") + tuple("d_" + k for k in KEYS):
            rows[f"env_{key}"].append(max(rows[f"{n}_{key}"][-1] for n in pert))
        print(f"step {s:2d} ({time.time() - t0:6.1f}s) Emax {rows['Emax'][-1]:.3e} " + " | ".join(
            f"{n}: df_e {rows[n + '_df_e'][-1]:.2e} df_i {rows[n + '_df_i'][-1]:.2e} "
            f"dE {rows[n + '_dE'][-1]:.2e} dEE {rows[n + '_d_e_energy'][-1]:.2e}" for n in pert), flush=True)
    np.savez(args.out, steps=np.arange(1, args.steps + 1), config=args.config,
             perturbations=np.array(list(pert)), **{k: np.asarray(v) for k, v in rows.items()})
    print("wrote", args.out)


if __name__ == "__main__":
    main()
