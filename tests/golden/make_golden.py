"""Generate tests/golden/ref_golden.npz from the REFERENCE itself.

Runs only where /root/reference exists (oracle/_ref is built from it). The
inputs are seeded (numpy, 20240817 = the seed of core/src/check.cpp:31); the
outputs are whatever the reference's own functions return, so the fixtures pin
both the C oracle and the GPU path to the reference without needing
/root/reference at test time.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_golden.npz")

# small run() configurations exercising every §8 row: sweeps, inline limiter,
# literature limiters, 3-block transfer (m=1,2,4,8), cut-off, charge density
STATE_CFGS = {
    "c1mini_none": dict(k=2, nf=8, nc=16, m=1, nv=32, limiter="none"),
    "c2mini_sldg_m8": dict(k=2, nf=16, nc=16, m=8, nv=32, limiter="sldg"),
    "c3mini_sldg_mu1836": dict(k=3, nf=8, nc=16, m=1, nv=24, mu=1836.0, limiter="sldg"),
    "k3_meanerr_line_m2": dict(k=3, nf=8, nc=8, m=2, nv=16, limiter="meanerr+line"),
    "k1_minmod_simple_m3": dict(k=1, nf=6, nc=6, m=3, nv=16, limiter="minmod+simple"),
    "k2_minmod_line": dict(k=2, nf=8, nc=8, m=1, nv=20, limiter="minmod+line"),
    "k2_meanerr_simple_m4": dict(k=2, nf=8, nc=8, m=4, nv=20, limiter="meanerr+simple"),
    "k4_sldg": dict(k=4, nf=6, nc=6, m=1, nv=16, limiter="sldg"),
}
STATE_STEPS = (1, 3, 12)


def main():
    ref = oracle.Ref()
    rng = np.random.default_rng(20240817)
    g = {}
    fails, report = ref.self_checks()
    assert fails == 0, report
    for k in range(7):
        n, w = ref.gauss_legendre(k)
        g[f"gl_nodes_k{k}"], g[f"gl_weights_k{k}"] = n, w
    # decompose_shift (advection.cpp:14-25), incl. test_advection.cpp:44-70 cases
    cases = [(0.0, 0.1, 0.5), (-0.5, 1.0, 1.0), (1.3, 1.0, 1.0)]
    for _ in range(200):
        cases.append((rng.uniform(-30, 30), rng.uniform(0, 2), rng.uniform(0.1, 2)))
    cases = np.array(cases)
    ist, al = zip(*[ref.decompose_shift(*c) for c in cases])
    g["shift_cases"], g["shift_istar"], g["shift_alpha"] = cases, np.array(ist), np.array(al)
    # shift matrices (advection.cpp:27-66)
    alphas = np.concatenate([[0.0, 0.3, 0.5, 0.77, 0.999], rng.uniform(0, 1, 11)])
    g["sm_alphas"] = alphas
    for k in (0, 1, 2, 3, 4, 6):
        A, B = zip(*[ref.shift_matrices(k, a) for a in alphas])
        g[f"sm_A_k{k}"], g[f"sm_B_k{k}"] = np.array(A), np.array(B)
    # inline limiter on projected random stencils (limiters.cpp:175-222)
    for k in (1, 2, 3, 4, 5):
        p = k + 1
        N = 400
        al = rng.uniform(0, 0.999, N)
        ul = rng.uniform(-1, 1, (N, p))
        ur = rng.uniform(-1, 1, (N, p))
        # every third stencil is a step / near-vacuum one so the clamp path fires
        ul[::3] = 0.0
        ur[::3] = 1.0
        ul[1::7] *= 1e-30
        ups, flags, outs = [], [], []
        for i in range(N):
            A, B = ref.shift_matrices(k, al[i])
            up = A @ ul[i] + B @ ur[i]
            f, o = ref.inline_apply(k, al[i], 0.5, ul[i], ur[i], up)
            ups.append(up)
            flags.append(f)
            outs.append(o)
        g[f"il_alpha_k{k}"], g[f"il_ul_k{k}"], g[f"il_ur_k{k}"] = al, ul, ur
        g[f"il_up_k{k}"], g[f"il_flags_k{k}"], g[f"il_out_k{k}"] = np.array(ups), np.array(flags), np.array(outs)
    # theta = 1/3 known answer (test_limiters.cpp:319-333), k=1 clamp only
    n1, _ = ref.gauss_legendre(1)
    up = -1.0 + 3.0 * n1
    f, o = ref.inline_apply(1, 0.5, 0.0, np.ones(2), np.zeros(2), up)
    g["kat_theta13_up"], g["kat_theta13_out"], g["kat_theta13_flags"] = up, o, f
    # extrema (basis.cpp:172-225)
    for k in (1, 2, 3, 4, 5):
        p = k + 1
        U = rng.uniform(-1, 1, (100, p))
        ab = np.sort(rng.uniform(0, 1, (100, 2)), axis=1)
        g[f"ext_u_k{k}"], g[f"ext_ab_k{k}"] = U, ab
        g[f"ext_max_k{k}"] = np.array([ref.max_on(k, U[i], *ab[i]) for i in range(100)])
        g[f"ext_min_k{k}"] = np.array([ref.min_on(k, U[i], *ab[i]) for i in range(100)])
    # post-limiter indicators + modifiers (limiters.cpp:47-165)
    for k in (1, 2, 3):
        p = k + 1
        T = rng.uniform(-1, 1, (300, 3, p))
        T[::4] = np.abs(T[::4])
        T[1::5, 1] += 3.0  # spikes
        g[f"post_trip_k{k}"] = T
        g[f"post_minmod_k{k}"] = np.array([ref.post_indicator(k, 1, 0.5, *t) for t in T])
        g[f"post_meanerr_k{k}"] = np.array([ref.post_indicator(k, 2, 0.5, *t) for t in T])
        g[f"post_simple_k{k}"] = np.array([ref.post_modify(k, 1, *t) for t in T])
        g[f"post_line_k{k}"] = np.array([ref.post_modify(k, 2, *t) for t in T])
        g[f"post_beta_k{k}"] = np.array([ref.smoothness_beta(k, t[1]) for t in T])
    # sheath-mesh transfer (adaptivity.cpp:132-156)
    for k in (2, 3):
        for m in (1, 2, 4, 8):
            fine = rng.uniform(-1, 1, m * (k + 1))
            coarse = rng.uniform(-1, 1, k + 1)
            g[f"f2c_in_k{k}_m{m}"] = fine
            g[f"f2c_out_k{k}_m{m}"] = ref.fine_to_coarse(k, fine, m)
            g[f"c2f_in_k{k}_m{m}"] = coarse
            g[f"c2f_out_k{k}_m{m}"] = ref.coarse_to_fine(k, coarse, m)
    # full run() loop bodies
    for name, cfg in STATE_CFGS.items():
        st = ref.state(**cfg)
        done = 0
        for s in STATE_STEPS:
            while done < s:
                st.step()
                done += 1
            g[f"st_{name}_s{s}_fe"] = st.field(0)
            g[f"st_{name}_s{s}_fi"] = st.field(1)
            g[f"st_{name}_s{s}_E"] = st.E()
            g[f"st_{name}_s{s}_vmax"] = np.array([st.vmax(0), st.vmax(1)])
            g[f"st_{name}_s{s}_shrinks"] = np.array([st.shrinks(0), st.last_shrink(0),
                                                    st.shrinks(1), st.last_shrink(1)])
            stt = st.stats()
            g[f"st_{name}_s{s}_stats"] = np.array([stt[k] for k in sorted(stt)])
            smry = st.summary()
            g[f"st_{name}_s{s}_summary"] = np.array([smry[k] for k in sorted(smry)])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)/1e6:.2f} MB")


if __name__ == "__main__":
    main()
