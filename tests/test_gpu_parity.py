"""GPU parity: the sm_100a path through the C ABI against the C oracle (pinned
to the reference, tests/test_oracle_pin.py) and the reference's golden vectors.

Bar:
  * kernel level (same inputs, same E), exact mode: BITWISE -- x/v sweeps with
    the inline limiter and 3-block ghosts, post limiters, velocity cut-off,
    blob fill; fast mode (DFMA-contracted sweeps): <= 1e-12 relative;
  * full steps: max|df|/max|f| <= 1e-12 per species after 1 and 10 steps,
    |dE| <= 1e-12 * max(1, max|E|), identical shrink steps and v_max,
    diagnostics (mass, L2, momentum, kinetic, electric energy) rel <= 1e-12.
    (The charge-density reduction order differs from the serial reference,
    so full steps are tolerance-level, App. A item 6.)
  * full size (C3): sampled x and v lines of one GPU sweep, bitwise in exact
    mode, <= 1e-12 in fast mode; 11 whole run() loop bodies in exact mode
    bitwise against the reference's own loop (oracle/_ref).
"""
import os
import subprocess

import numpy as np
import pytest

from tests.golden.make_golden import STATE_CFGS, STATE_STEPS

pytestmark = pytest.mark.gpu

F_TOL = 1e-12
# tolerance factor over the reference's own rounding-noise envelope, the same
# on every mesh (_envelope, test_c3_fast_mode_within_reference_envelope)
ENV_C = 20.0
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    m = np.abs(b).max()
    return np.abs(a - b).max() / (m if m > 0 else 1.0)


def cfg_of(sk, **kw):
    c = dict(kw)
    ren = dict(nf="fine_block_cells", nc="coarse_block_cells", m="refinement_ratio", nv="v_cells")
    return sk.RunConfig(**{ren.get(k, k): v for k, v in c.items()})


KERNEL_CFGS = [
    dict(k=2, nf=8, nc=16, m=1, nv=32, limiter="sldg"),
    dict(k=2, nf=16, nc=16, m=8, nv=32, limiter="sldg"),
    dict(k=3, nf=8, nc=16, m=2, nv=24, mu=1836.0, limiter="sldg"),
    dict(k=1, nf=6, nc=6, m=3, nv=16, limiter="sldg"),
    dict(k=4, nf=6, nc=12, m=4, nv=16, limiter="sldg"),
    dict(k=0, nf=8, nc=8, m=2, nv=16, limiter="none"),
    dict(k=5, nf=4, nc=8, m=1, nv=12, limiter="sldg"),
    dict(k=6, nf=4, nc=4, m=2, nv=10, limiter="sldg"),
]


def _pair(sk, ora, kw, exact=True):
    cfg = cfg_of(sk, **kw)
    return cfg, ora.state(**cfg.oracle_kwargs()), sk.SimulationState(cfg, exact=exact)


def _same(got, want, exact):
    """exact mode: bitwise; fast mode: the north-star tolerance"""
    return np.array_equal(got, want) if exact else rel(got, want) <= F_TOL


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
@pytest.mark.parametrize("kw", KERNEL_CFGS, ids=lambda d: f"k{d['k']}m{d['m']}{d['limiter']}")
def test_sweeps_bitwise(sk, ora, kw, exact):
    cfg, o, st = _pair(sk, ora, kw, exact)
    for sp in (0, 1):
        assert np.array_equal(st.field(sp).download(), o.field(sp)), "blob fill"
    lim = sk.LimiterConfig.parse(cfg.limiter)
    spar = [sk.SpeciesParams.electron(), sk.SpeciesParams.ion(cfg.mu)]
    # evolve both a few steps so E != 0, the limiter is active and the v grids
    # have shrunk (identically); then feed both the oracle's data
    for _ in range(3):
        o.step()
    st.run_steps(3)
    for sp in (0, 1):
        assert st.field(sp).vmax() == o.vmax(sp)
    st.ctx.set_exact_reductions(exact)
    E = o.E()
    for sp in (0, 1):
        f = st.field(sp)
        for tau in (0.5 * cfg.dt, 1.1):  # 1.1: multi-cell shifts, several ghosts
            f.upload(o.field(sp))
            sk.advect_x(f, tau, spar[sp], sk.SweepOptions(limiter=lim, max_ghost=-1))
            ref = o.field(sp)
            o.advect_x(sp, tau, limited=True, max_ghost=-1)
            assert _same(f.download(), o.field(sp), exact), f"advect_x sp{sp} tau{tau}"
            o.set_field(sp, ref)
        x = np.linspace(-1.0, 1.0, E.size)
        for tau, Es in ((cfg.dt, E), (cfg.dt, 30.0 * np.sin(4.0 * x))):  # multi-cell v shifts
            f.upload(o.field(sp))
            sk.advect_v(f, tau, Es, spar[sp], sk.SweepOptions(limiter=lim))
            ref = o.field(sp)
            o.advect_v(sp, tau, Es, limited=True)
            assert _same(f.download(), o.field(sp), exact), f"advect_v sp{sp}"
            o.set_field(sp, ref)


@pytest.mark.parametrize("cap", [1, 3])
@pytest.mark.parametrize("kw", [c for c in KERNEL_CFGS if c["m"] > 1][:3], ids=lambda d: f"k{d['k']}m{d['m']}")
def test_x_ghosts_beyond_buffer_bitwise(sk, ora, kw, cap, monkeypatch):
    """3-block ghosts: the pre-pass buffers ghost_cap cells per (line, block),
    the sweep evaluates the ones further out itself. A tiny capacity and a
    multi-cell shift run both paths in one sweep; exact mode stays bitwise."""
    cfg, o, st = _pair(sk, ora, kw, True)
    spar = [sk.SpeciesParams.electron(), sk.SpeciesParams.ion(cfg.mu)]
    lim = sk.LimiterConfig.parse(cfg.limiter)
    monkeypatch.setenv("SK_XGHOST_CAP", str(cap))
    for sp in (0, 1):
        f = st.field(sp)
        for tau in (1.1, -2.3):
            f.upload(o.field(sp))
            sk.advect_x(f, tau, spar[sp], sk.SweepOptions(limiter=lim, max_ghost=-1))
            ref = o.field(sp)
            o.advect_x(sp, tau, limited=True, max_ghost=-1)
            assert np.array_equal(f.download(), o.field(sp)), f"advect_x sp{sp} tau{tau} cap{cap}"
            o.set_field(sp, ref)


@pytest.mark.parametrize("mode", ["minmod+simple", "minmod+line", "meanerr+simple", "meanerr+line"])
@pytest.mark.parametrize("m", [1, 4])
def test_post_limiters_bitwise(sk, ora, mode, m):
    cfg, o, st = _pair(sk, ora, dict(k=3, nf=8, nc=16, m=m, nv=20, limiter=mode))
    for _ in range(2):
        o.step()
    st.run_steps(2)
    for sp in (0, 1):
        for d in (0, 1):
            f = st.field(sp)
            f.upload(o.field(sp))
            sk.apply_post_limiter(f, d, sk.LimiterConfig.parse(mode))
            o.post_limit(sp, d, mode)
            assert np.array_equal(f.download(), o.field(sp)), f"{mode} dir{d} sp{sp}"


@pytest.mark.parametrize("k,nv", [(3, 24), (3, 200), (2, 131), (6, 70)])
def test_velocity_cutoff_bitwise(sk, ora, k, nv):
    """one and several v chunks per thread (the projection's cp.async ring:
    8 slots for p <= 4, 4 for p > 4), ragged last chunk"""
    cfg, o, st = _pair(sk, ora, dict(k=k, nf=8, nc=16, m=1, nv=nv, mu=1836.0))
    pol = sk.VAdjustPolicy(cfg.adapt_p, cfg.adapt_gamma, cfg.adapt_tol)
    for sp in (0, 1):
        f = st.field(sp)
        for _ in range(3):  # repeated shrinks on the same field
            f.upload(o.field(sp))
            assert sk.check_velocity_shrink(f, pol) == o.check_shrink(sp)
            r = sk.shrink_velocity_domain(f, pol)
            ro = o.shrink(sp)
            assert np.array_equal(f.download(), o.field(sp))
            # vmax_after is new_vmax (adaptivity.cpp:103,127); vmax() is the new
            # grid's right() = left + cells*dx, which can differ in the last bit
            assert r["vmax_after"] == ro["vmax_after"] and f.vmax() == o.vmax(sp)
            assert abs(r["mass_after"] - ro["mass_after"]) <= 1e-12 * abs(ro["mass_after"])
    # a field with mass at the probe velocity must not shrink
    f = st.field(0)
    f.upload(np.ones(f.size))
    assert not sk.check_velocity_shrink(f, pol)


def test_charge_density_and_poisson(sk, ora):
    cfg, o, st = _pair(sk, ora, dict(k=3, nf=16, nc=32, m=2, nv=24, limiter="none"))
    for _ in range(5):
        o.step()
    st.run_steps(5)
    for sp in (0, 1):
        st.field(sp).upload(o.field(sp))
    rho_o = o.charge_density()
    rho_g = sk.charge_density(st.f_e, st.f_i).cpu().numpy()
    scale = max(np.abs(o.field(0)).max(), 1e-300) * 24.0
    assert np.abs(rho_g - rho_o).max() <= 1e-14 * scale
    E_o, phi_o = o.poisson_solve(rho_o)
    fp = sk.PoissonOperator(st.ctx).solve(rho_o)
    assert np.abs(fp.E.cpu().numpy() - E_o).max() <= 1e-12 * max(1.0, np.abs(E_o).max())
    # phi is a kappa(A)*eps-sensitive quantity (SIPG kappa ~ 1e5..1e6): two
    # backward-stable solvers (cyclic reduction vs banded Cholesky) agree to
    # ~1e-11 relative; E = -phi' is what the step consumes (checked above)
    assert np.abs(fp.phi.cpu().numpy() - phi_o).max() <= 1e-10 * np.abs(phi_o).max()


FULL_CFGS = {
    "C1": dict(k=2, nf=32, nc=64, m=1, nv=128, limiter="none"),
    "C2mesh_sldg": dict(k=2, nf=64, nc=128, m=8, nv=128, limiter="sldg"),
    "C3mini_sldg": dict(k=3, nf=32, nc=64, m=1, nv=256, mu=1836.0, limiter="sldg"),
    "C4_meanerr_line": dict(k=3, nf=16, nc=32, m=1, nv=64, mu=1836.0, limiter="meanerr+line"),
    "C4_minmod_simple_m2": dict(k=2, nf=16, nc=32, m=2, nv=64, limiter="minmod+simple"),
}


def _envelope(ora, cfg, steps):
    """Rounding-noise envelope of the reference dynamics, per
    step the max over three perturbations the reference itself leaves open
    (tests/golden/make_c3_envelope.py): the charge density summed in the other
    species order, the Poisson band solved by another LAPACK (scipy's), and
    the restatement built with FMA contraction. The GPU's fast mode sums rho
    in yet another (parallel) order, solves Poisson by refined cyclic
    reduction and contracts the sweeps into DFMA, so its deviation is compared
    with this."""
    import oracle as O

    a = ora.state(**cfg.oracle_kwargs())
    pert = {"rho": ora.state(**cfg.oracle_kwargs())}
    lap = O.scipy_lapack()
    if lap is not None:
        ora.set_lapack(lap)
        try:
            pert["lapack"] = ora.state(**cfg.oracle_kwargs())
        finally:
            ora.set_lapack(None)
    if os.path.exists(O.oracle.ORACLE_FMA_SO):
        pert["fma"] = O.Oracle(O.oracle.ORACLE_FMA_SO).state(**cfg.oracle_kwargs())
    env = {}
    for s in range(1, steps + 1):
        a.step()
        for name, b in pert.items():
            if name == "rho":
                ora.set_rho_order(1)
            try:
                b.step()
            finally:
                ora.set_rho_order(0)
        env[s] = (max(rel(a.field(sp), b.field(sp)) for sp in (0, 1) for b in pert.values()),
                  max(np.abs(a.E() - b.E()).max() for b in pert.values()))
    return env


@pytest.mark.parametrize("batched", [False, True], ids=["stepwise", "fused"])
@pytest.mark.parametrize("name", list(FULL_CFGS))
def test_full_steps_vs_oracle(sk, ora, name, batched):
    """Fast path (DFMA sweeps, parallel charge density, refined cyclic-
    reduction Poisson). The exact-mode test proves every other operation is
    bitwise, so what remains is rounding noise: f within 1e-12
    and E within 1e-12 * max(1, max|E|) at steps 1 and 10, each unless the
    reference's own envelope (ENV_C x _envelope) is larger."""
    cfg, o, st = _pair(sk, ora, FULL_CFGS[name])
    st.ctx.set_step_fusion(batched)
    env = _envelope(ora, cfg, 10)
    for s in range(1, 11):
        if not batched:
            st.run_step()
        elif s in (1, 2):  # run_steps(9): a graph whose step boundaries fuse the x half sweeps
            st.run_steps(1 if s == 1 else 9)
        o.step()
        if s in (1, 10):
            ef, eE = env[s]
            for sp in (0, 1):
                assert rel(st.field(sp).download(), o.field(sp)) <= max(F_TOL, ENV_C * ef), f"f sp{sp} step {s}"
                assert st.field(sp).vmax() == o.vmax(sp)
            E_o = o.E()
            dE = np.abs(st.E() - E_o).max()
            Emax = np.abs(E_o).max()
            assert dE <= max(1e-12 * max(1.0, Emax), ENV_C * eE), (s, dE, eE)
    assert st.shrinks(0) == (o.shrinks(0), o.last_shrink(0))
    assert st.shrinks(1) == (o.shrinks(1), o.last_shrink(1))
    assert st.step_index() == o.step_index() == 10
    # diagnostics (field.cpp:52-88 + harness moments, diagnostics.cpp:71-83);
    # momentum of the symmetric blob cancels, so it is scaled by mass * vmax
    g, r = st.summary(), o.summary()
    for sp in ("e", "i"):
        m, vm = r[f"mass_{sp}"], r[f"vmax_{sp}"]
        for key, scale in ((f"mass_{sp}", m), (f"l2_{sp}", r[f"l2_{sp}"]),
                           (f"mom_{sp}", m * vm), (f"ekin_{sp}", r[f"ekin_{sp}"])):
            assert abs(g[key] - r[key]) <= 1e-12 * abs(scale), key
    assert abs(g["e_energy"] - r["e_energy"]) <= 1e-12 * r["e_energy"]
    # counters: troubled/post near-exact; clamps flip on ulp-level E changes
    gs, os_ = st.stats(), o.stats()
    assert gs["outputs"] == os_["outputs"]
    assert gs["post_checked"] == os_["post_checked"]
    # troubled flags in the near-vacuum tails (|f| ~ 1e-30) follow the rounding
    # noise of their neighbours, so they are reported, not asserted (SURVEY.md
    # §8c); exact mode reproduces them exactly. Sanity bound only:
    for key in ("inline_troubled", "inline_clamped", "post_troubled"):
        assert abs(gs[key] - os_[key]) <= max(5, 0.25 * os_[key]), key


# configs whose dynamics amplify rounding noise exponentially (coarse meshes:
# E grows to O(1) within 12 steps) are compared up to step 3 only
CHAOTIC = {"k3_meanerr_line_m2"}


@pytest.mark.parametrize("name", list(STATE_CFGS))
def test_against_reference_golden(sk, golden, name):
    cfg = cfg_of(sk, **STATE_CFGS[name])
    st = sk.SimulationState(cfg)
    done = 0
    for s in STATE_STEPS:
        if name in CHAOTIC and s > 3:
            break
        while done < s:
            st.run_step()
            done += 1
        tol = F_TOL * (10 if s > 10 else 1)
        assert rel(st.f_e.download(), golden[f"st_{name}_s{s}_fe"]) <= tol
        assert rel(st.f_i.download(), golden[f"st_{name}_s{s}_fi"]) <= tol
        E = golden[f"st_{name}_s{s}_E"]
        assert np.abs(st.E() - E).max() <= tol * max(1.0, np.abs(E).max())
        assert np.array_equal([st.f_e.vmax(), st.f_i.vmax()], golden[f"st_{name}_s{s}_vmax"])
        sh = golden[f"st_{name}_s{s}_shrinks"]
        assert st.shrinks(0) == (sh[0], sh[1]) and st.shrinks(1) == (sh[2], sh[3])


EXACT_CFGS = dict(FULL_CFGS, **{k: v for k, v in STATE_CFGS.items()})


@pytest.mark.parametrize("name", list(EXACT_CFGS))
def test_exact_mode_trajectory_bitwise(sk, ora, name):
    """With the two reductions in reference order, a whole trajectory --
    sweeps, limiters, 3-block transfer, charge density, Poisson, cut-off,
    shrink events -- is bitwise the reference's (25 run() loop bodies)."""
    cfg = cfg_of(sk, **EXACT_CFGS[name])
    o = ora.state(**cfg.oracle_kwargs())
    st = sk.SimulationState(cfg, exact=True)
    for sp in (0, 1):
        assert np.array_equal(st.field(sp).download(), o.field(sp))
    assert np.array_equal(st.E(), o.E())
    n = 25 if cfg.dof_total < 2e5 else 12
    for s in range(n):
        st.run_step()
        o.step()
    for sp in (0, 1):
        assert np.array_equal(st.field(sp).download(), o.field(sp)), f"sp{sp}"
        assert st.field(sp).vmax() == o.vmax(sp)
    assert np.array_equal(st.E(), o.E())
    assert st.shrinks(0) == (o.shrinks(0), o.last_shrink(0))
    assert st.shrinks(1) == (o.shrinks(1), o.last_shrink(1))
    gs, os_ = st.stats(), o.stats()
    assert gs == os_


@pytest.mark.parametrize("limiter", ["sldg", "minmod+line", "meanerr+simple", "sldg_injection"])
def test_deferred_clamp_overflow_rescan_is_identical(sk, limiter):
    """troubled (sLdG) / flagged (post limiter) cells are queued for a fixup
    kernel; when the queue overflows the fixup rescans the pass -- both paths
    must give the same bits. sldg_injection: the source half steps fused into
    the x sweeps (the rescan recomputes what a queued cell would have held)"""
    from paper_2408_11235_b200 import _native as N

    if limiter == "sldg_injection":
        cfg = cfg_of(sk, k=3, nf=16, nc=32, m=1, nv=32, limiter="sldg", scenario="injection", t0=0.45,
                     mu=1836.0)
        limiter = "sldg"
    else:
        cfg = cfg_of(sk, k=2, nf=16, nc=16, m=8, nv=32, limiter=limiter)
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    assert N.lib().sk_ctx_set_fix_capacity(b.ctx.h, 7) == 0  # forces overflow
    for _ in range(6):
        a.run_step()
        b.run_step()
    for sp in (0, 1):
        assert np.array_equal(a.field(sp).download(), b.field(sp).download())
    st = a.stats()
    assert st == b.stats()
    assert (st["inline_troubled"] if limiter == "sldg" else st["post_troubled"]) > 300


def test_graph_replay_equals_eager(sk):
    cfg = cfg_of(sk, k=3, nf=16, nc=32, m=2, nv=48, mu=1836.0, limiter="sldg")
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    a.run_steps(13)  # graph-replayed pairs + one eager body
    for _ in range(13):
        b.run_step()
    for sp in (0, 1):
        assert np.array_equal(a.field(sp).download(), b.field(sp).download())
    assert np.array_equal(a.E(), b.E())
    assert a.shrinks(0) == b.shrinks(0) and a.step_index() == b.step_index() == 13


def test_run_to_run_deterministic(sk):
    cfg = cfg_of(sk, k=2, nf=64, nc=128, m=8, nv=128, limiter="sldg")
    outs = []
    for _ in range(2):
        st = sk.SimulationState(cfg)
        st.run_steps(6)
        outs.append((st.f_e.download(), st.f_i.download(), st.E(), st.stats()))
    assert all(np.array_equal(x, y) for x, y in zip(outs[0][:3], outs[1][:3]))
    assert outs[0][3] == outs[1][3]


def test_host_buffer_entry_point_equals_device_path(sk):
    cfg = cfg_of(sk, k=2, nf=8, nc=16, m=2, nv=32, limiter="sldg")
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    fe, fi = a.f_e.download(), a.f_i.download()
    for _ in range(4):
        a.run_step_host(fe, fi)
        b.run_step()
    assert np.array_equal(fe, b.f_e.download()) and np.array_equal(fi, b.f_i.download())


def test_errors_map_to_reference_exceptions(sk):
    cfg = cfg_of(sk, k=2, nf=8, nc=16, m=2, nv=32, limiter="none")
    st = sk.SimulationState(cfg)
    # advection.cpp:185-190: insufficient ghost width -> SimulationError{step}
    with pytest.raises(sk.SimulationError, match="insufficient ghost width") as ei:
        sk.advect_x(st.f_e, 30.0, sk.SpeciesParams.electron(),
                    sk.SweepOptions(max_ghost=1, step_index=42))
    assert ei.value.step == 42
    # advection.cpp:151-153: periodic rule on a 3-block grid -> runtime_error
    with pytest.raises(RuntimeError, match="periodic"):
        sk.advect_x(st.f_e, 0.05, sk.SpeciesParams.electron(), sk.SweepOptions(bc=1))
    # stepper.cpp:101-102: nonfinite state -> SimulationError at the step
    bad = st.f_i.download()
    bad[len(bad) // 2] = np.nan
    st.f_i.upload(bad)
    with pytest.raises(sk.SimulationError, match="nonfinite") as ei:
        st.run_step()
    assert ei.value.step == 1


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
@pytest.mark.parametrize("kw", [
    dict(k=3, nf=16, nc=32, m=1, nv=64, mu=1836.0, limiter="minmod+line"),
    dict(k=3, nf=16, nc=32, m=2, nv=64, mu=1836.0, limiter="meanerr+simple"),
    dict(k=2, nf=16, nc=16, m=1, nv=48, limiter="meanerr+line"),
    dict(k=1, nf=12, nc=24, m=4, nv=40, limiter="minmod+simple"),
    dict(k=5, nf=8, nc=8, m=1, nv=40, limiter="minmod+line")],
    ids=["k3_minmod_line", "k3_meanerr_simple_m2", "k2_meanerr_line", "k1_minmod_simple_m4", "k5_minmod_line"])
def test_post_flags_fused_into_sweeps(sk, kw, exact):
    """The step's sweeps decide the post limiter's flags of their own outputs
    and the post passes only run the fixes (sk_ctx_set_post_fusion): the v
    sweep from the registers it stores (each chunk also computes its two
    neighbour cells; walls are zero cells), the x sweeps from the tile's
    summaries in shared memory (a tile's first and last cell -- incl. every
    block edge of the 3-block meshes -- re-decided by the fix kernel as
    candidates). Same summaries, same decisions as the separate flag passes,
    so 12 steps through both shrinks agree bitwise with fusion off: f, E,
    v_max, shrink steps and the limiter counters. v meshes of 2 chunks, a
    ragged last chunk; k = 5 in fast mode keeps the passes (no DFMA sweep
    for k > 3)."""
    cfg = cfg_of(sk, **kw)
    a, b = sk.SimulationState(cfg, exact=exact), sk.SimulationState(cfg, exact=exact)
    a.ctx.set_post_fusion(True)
    b.ctx.set_post_fusion(False)
    if not exact:  # the charge density in the reference order in both (its fusion: next test)
        for st in (a, b):
            st.ctx.set_exact_parts(st.ctx.EXACT_RHO)
    for st in (a, b):
        st.run_step()  # (eager body: first-step shrink)
        st.run_steps(11)
    assert a.step_index() == b.step_index() == 12
    for sp in (0, 1):
        assert a.shrinks(sp) == b.shrinks(sp)
        assert a.field(sp).vmax() == b.field(sp).vmax()
        assert np.array_equal(a.field(sp).download(), b.field(sp).download()), f"sp{sp}"
    assert np.array_equal(a.E(), b.E())
    sa, sb = a.stats(), b.stats()
    assert sa["post_checked"] == sb["post_checked"] > 0
    assert sa["post_troubled"] == sb["post_troubled"] > 0
    # the fused runs launched no flag pass (x1, v, x2: three kernels less per step)
    fused = exact or kw["k"] <= 3
    assert b.launches() - a.launches() == (36 if fused else 0)


@pytest.mark.parametrize("kw", [
    dict(k=3, nf=16, nc=32, m=1, nv=64, mu=1836.0, limiter="minmod+line"),
    dict(k=3, nf=16, nc=32, m=2, nv=64, mu=1836.0, limiter="meanerr+simple"),
    dict(k=2, nf=16, nc=16, m=1, nv=48, limiter="meanerr+line")],
    ids=["k3_minmod_line", "k3_meanerr_simple_m2", "k2_meanerr_line"])
def test_post_limited_charge_density_fused(sk, ora, kw):
    """Fast mode with a post limiter: the first x sweep, which decides the
    post X flags, also sums the charge density; the fixes add the modified
    cells' changes as exact integer corrections and the moment is reduced
    after them. Against the separate charge-density pass (post fusion off)
    over 3 steps: the same arithmetic grouped differently, so f and E agree
    within the reference's rounding envelope, the counters and v_max
    exactly; the fused run launches no rho pass (two kernels less per step:
    rho partial + reduce -> one fused reduce; and three flag passes less)."""
    cfg = cfg_of(sk, **kw)
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    a.ctx.set_post_fusion(True)
    b.ctx.set_post_fusion(False)
    l0a, l0b = a.launches(), b.launches()
    for _ in range(3):
        a.run_step()
        b.run_step()
    assert (b.launches() - l0b) - (a.launches() - l0a) == 3 * (3 + 1)
    ef, eE = _envelope(ora, cfg, 3)[3]
    for sp in (0, 1):
        assert a.field(sp).vmax() == b.field(sp).vmax()
        fa, fb = a.field(sp).download(), b.field(sp).download()
        assert rel(fa, fb) <= max(F_TOL, ENV_C * ef), f"sp{sp}"
    Ea, Eb = a.E(), b.E()
    assert np.abs(Ea - Eb).max() <= max(1e-12 * max(1.0, np.abs(Eb).max()), ENV_C * eE)
    assert a.stats()["post_checked"] == b.stats()["post_checked"]


@pytest.mark.parametrize("kw", [
    dict(k=3, nf=32, nc=64, m=1, nv=128, mu=1836.0, limiter="sldg"),
    dict(k=2, nf=16, nc=32, m=1, nv=64, limiter="none"),
    dict(k=1, nf=24, nc=24, m=1, nv=48, limiter="sldg"),
    dict(k=0, nf=16, nc=16, m=1, nv=32, limiter="none")], ids=["k3_sldg", "k2_none", "k1_sldg", "k0_none"])
def test_fused_step_boundaries_match_separate_sweeps(sk, ora, kw):
    """run_steps fuses step n's second and step n+1's first x half sweep into
    one pass (xsweep_kernel MODE 3, clamps in-kernel), except at boundaries
    where the cut-off may check (decided on the device). Against the same 12
    steps with fusion off: every cell runs the same arithmetic, only the
    charge density is grouped differently (fused moment of clamped values
    instead of unclamped + exact corrections) -- f and E agree to rounding,
    shrink steps and v_max are identical.""" 
    cfg = cfg_of(sk, **kw)
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    a.ctx.set_step_fusion(True)
    b.ctx.set_step_fusion(False)
    # 12 steps through both shrinks (steps 1, 11): graphs of 3 and 9 bodies
    # (coarse meshes amplify the charge density's rounding-level difference
    # exponentially beyond, as in CHAOTIC below)
    for n in (3, 9):
        a.run_steps(n)
        b.run_steps(n)
    assert a.step_index() == b.step_index() == 12
    ef, eE = _envelope(ora, cfg, 12)[12]  # coarse k = 1 meshes amplify rounding fast
    for sp in (0, 1):
        assert a.shrinks(sp) == b.shrinks(sp) and a.shrinks(sp)[0] >= 2
        assert a.field(sp).vmax() == b.field(sp).vmax()
        fa, fb = a.field(sp).download(), b.field(sp).download()
        assert rel(fa, fb) <= max(F_TOL, ENV_C * ef), f"sp{sp}"
        # pointwise where f is not vacuum (a missed clamp in the tails would
        # hide below the max-normalised bound)
        live = np.abs(fb) > 1e-8 * np.abs(fb).max()
        tol = max(1e-10, 100 * ENV_C * ef)
        assert (np.abs(fa - fb)[live] <= tol * np.abs(fb)[live]).all(), f"sp{sp} pointwise"
    Eb = b.E()
    assert np.abs(a.E() - Eb).max() <= max(1e-12 * max(1.0, np.abs(Eb).max()), ENV_C * eE)
    # limiter counters: a fused boundary does not evaluate the step-n cells that
    # leave the line in step n+1's first sweep (their values cannot reach the
    # state); elsewhere flags only flip where rounding-level E differences
    # move near-vacuum cells across the threshold
    sa, sb = a.stats(), b.stats()
    assert sa["outputs"] == sb["outputs"]
    for key in ("inline_troubled", "inline_clamped"):
        assert abs(sa[key] - sb[key]) <= max(5, 0.05 * sb[key]), key


def test_nonfinite_mid_batch_halts_at_the_failing_step(sk):
    """A nonfinite state raised inside a graph-replayed batch halts every later
    kernel: the step counter stays at the failing step and the fields are the
    ones that step left -- the reference's run() unwinds at the throw
    (stepper.cpp:99-102, run.cpp:147-155) -- identical to stepping one loop
    body at a time; after the error is collected the context is usable."""
    cfg = cfg_of(sk, k=2, nf=8, nc=16, m=1, nv=32, limiter="sldg", mu=400.0)
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    a.ctx.set_eager_errors(False)
    a.run_steps(3)
    b.run_steps(3)
    f = a.f_e.download()
    f[len(f) // 2 + 7] = np.nan
    a.f_e.upload(f)
    b.f_e.upload(f)
    with pytest.raises(sk.SimulationError, match="nonfinite") as ea:
        a.run_steps(6)  # graph pairs: the failure is in the first body of the first pair
        a.ctx.synchronize()
    with pytest.raises(sk.SimulationError, match="nonfinite") as eb:
        b.run_step()
    assert ea.value.step == eb.value.step == 4
    assert a.step_index() == b.step_index() == 4
    for sp in (0, 1):
        fa, fb = a.field(sp).download(), b.field(sp).download()
        assert np.array_equal(fa, fb, equal_nan=True), f"sp{sp}"
        assert a.field(sp).vmax() == b.field(sp).vmax()
    assert np.array_equal(a.E(), b.E(), equal_nan=True)


def test_periodic_sweep_conserves_mass(sk):
    """test_advection.cpp:194-225 (CFL up to 50, mass conserved to 1e-13)"""
    grid = sk.Grid1D.uniform(-1.0, 1.0, 64)
    ctx = sk.Context(grid, 3)
    f = sk.NodalField(ctx, 0, sk.Grid1D.uniform(-4.0, 4.0, 16))
    f.fill_blob(0.3)
    m0 = f.mass()
    for tau in (0.01, 0.4, 3.7):
        sk.advect_x(f, tau, sk.SpeciesParams.electron(), sk.SweepOptions(bc=1))
        assert abs(f.mass() - m0) <= 1e-13 * abs(m0)


@pytest.mark.parametrize("mode", ["minmod+line", "meanerr+simple"])
def test_periodic_post_limiter_translation_invariant(sk, mode):
    """Periodic post limiting (the reference oracle has walls only): rolling
    the input by r cells in x (or v) must roll the output bit for bit. 1200 x
    cells make three flag-pass tiles, so the wrap windows and the tile edges
    are both exercised; a rough field makes many cells flagged."""
    k, nx, nv = 3, 1200, 40
    P = k + 1
    ctx = sk.Context(sk.Grid1D.uniform(-1.0, 1.0, nx), k)
    f = sk.NodalField(ctx, 0, sk.Grid1D.uniform(-4.0, 4.0, nv))
    rng = np.random.default_rng(7)
    base = np.abs(rng.standard_normal(f.size)) * (rng.random(f.size) < 0.2) + 0.1
    lim = sk.LimiterConfig.parse(mode)
    for d, r in ((0, 517), (1, 13)):
        shape = (nv * P, nx, P) if d == 0 else (nv, P, nx * P)
        rolled = np.roll(base.reshape(shape), r, axis=0 if d else 1).ravel()
        outs = []
        for u in (base, rolled):
            f.upload(u)
            sk.apply_post_limiter(f, d, lim, bc=1)
            outs.append(f.download())
        assert not np.array_equal(outs[0], base), "nothing flagged"
        assert np.array_equal(np.roll(outs[0].reshape(shape), r, axis=0 if d else 1).ravel(), outs[1]), f"dir {d}"


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_c3_full_size_sampled_lines_bitwise(sk, ora, exact):
    """C3 (2048x4096, k=3, mu=1836, sldg): one GPU x and v sweep at full size;
    48 sampled lines recomputed by the oracle must match bit for bit (exact
    mode) or to 1e-12 (fast mode)."""
    cfg = sk.named_config("C3")
    st = sk.SimulationState(cfg)
    st.run_steps(2)
    st.ctx.synchronize()
    st.ctx.set_exact_reductions(exact)
    p = cfg.k + 1
    nx, nv = cfg.nx, cfg.v_cells
    rng = np.random.default_rng(7)
    grid = st.ctx.grid
    lim = sk.LimiterConfig.parse("sldg")
    for sp, spar in ((0, sk.SpeciesParams.electron()), (1, sk.SpeciesParams.ion(cfg.mu))):
        f = st.field(sp)
        before = f.download().reshape(nv * p, nx * p)
        vleft, vdx, _ = f.v_grid()
        sk.advect_x(f, 0.5 * cfg.dt, spar, sk.SweepOptions(limiter=lim))
        after = f.download().reshape(nv * p, nx * p)
        nodes, _ = ora.gauss_legendre(cfg.k)
        for r in rng.choice(nv * p, 24, replace=False):
            vc, vn = divmod(int(r), p)
            vnode = (vleft + vc * vdx) + vdx * nodes[vn]
            out = ora.advect_x_line(cfg.k, grid.left, grid.cells, grid.dx, vnode / spar.sqrt_mu,
                                    0.5 * cfg.dt, before[r], inline_sldg=True)
            assert _same(after[r], out, exact), f"x line {r} sp{sp}"
        # v sweep with a synthetic, strong field (multi-cell shifts)
        x = np.linspace(-1, 1, nx * p)
        E = 0.3 * np.sin(3 * x)
        f.upload(after.ravel())
        sk.advect_v(f, cfg.dt, E, spar, sk.SweepOptions(limiter=lim))
        vout = f.download().reshape(nv * p, nx * p)
        cols = rng.choice(nx * p, 24, replace=False)
        lines = after[:, cols].T.copy()  # [ncols, nv*p]
        ref = ora.advect_v_lines(cfg.k, lines, 0, nv, 0, E[cols], spar.charge_sign, spar.sqrt_mu,
                                 cfg.dt, vdx, limiter="sldg")
        assert _same(vout[:, cols].T, ref, exact), f"v lines sp{sp}"


def test_cpp_mirror_runs_against_oracle():
    from paper_2408_11235_b200 import build as B

    out = "/tmp/sk_test_cpp_api_gpu"
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-o", out,
           os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"),
           os.path.join(ROOT, "oracle", "_build", "libsk_oracle.so"), B.LIB,
           "-Wl,-rpath," + os.path.dirname(B.LIB) + ":" + os.path.join(ROOT, "oracle", "_build")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([out], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("adaptive", [False, True], ids=["fixed_halo", "adaptive_halo"])
@pytest.mark.parametrize("v_adjust,limiter", [(False, "sldg"), (True, "sldg"), (True, "minmod+line")],
                         ids=["no_cutoff", "cutoff", "cutoff_post"])
def test_two_v_shards_on_one_gpu_match_unsharded(sk, v_adjust, limiter, adaptive):
    """The CUDA v-shard path (global cell offsets in the x tables, halo reads in
    the v sweep, local fused charge density, sharded velocity cut-off) driven
    like two ranks, with the all-reduces and the halo exchanges done by device
    copies in one process; 12 run() loop bodies cover two shrink events.
    adaptive: phases 6-9 -- the exchange width from this step's E (v tables),
    interior v chunks swept before the exchange, the edges after; the
    interior bound alternates between the last width + 1 and 1, and every
    third step re-sweeps all chunks (phase 9)."""
    import ctypes as C

    import torch

    from paper_2408_11235_b200 import _native as N
    from paper_2408_11235_b200.sharding import VShardPlan, _dev_tensor
    from paper_2408_11235_b200.solver import Context, Grid1D, _check

    cfg = cfg_of(sk, k=3, nf=16, nc=32, m=2, nv=64, mu=1836.0, limiter=limiter, v_adjust=v_adjust)
    ref = sk.SimulationState(cfg)
    post = limiter != "sldg"
    L = N.lib()
    grid = Grid1D.three_block(-cfg.L, cfg.L, cfg.fine_block_cells, cfg.coarse_block_cells,
                              cfg.refinement_ratio)
    world, halo = 2, 6
    shards = []
    for r in range(world):
        ctx = Context(grid, cfg.k, cfg.penalty_scale, 0)
        h = C.c_void_p()
        ccfg = cfg.to_c()
        _check(L.sk_state_create_shard(ctx.h, C.byref(ccfg), r, world, halo, C.byref(h)))
        rho = _dev_tensor(L.sk_state_rho_dev(h), ctx.nx * ctx.p, 0)
        flags = _dev_tensor(L.sk_state_shrink_flags_dev(h), 2, 0, "<i4")
        shards.append((ctx, h, rho, VShardPlan(cfg.v_cells, world, r, halo), flags))
    hs = L.sk_state_shrink_halo(shards[0][1])
    assert (hs > 0) == v_adjust

    def sync():
        for ctx, *_ in shards:
            ctx.synchronize()
        torch.cuda.synchronize()

    def reduce_rho():
        sync()
        tot = sum(s[2].clone() for s in shards)
        for s in shards:
            s[2].copy_(tot)
        torch.cuda.synchronize()

    def exchange(cells=None, species=(0, 1)):
        sync()
        views = {}
        for r, (ctx, h, *_) in enumerate(shards):
            for sp in species:
                f = L.sk_state_field(h, sp)
                for side in (0, 1):
                    for send in (1, 0):
                        ptr, cnt = C.c_void_p(), C.c_size_t()
                        if cells is None:
                            _check(L.sk_field_halo(f, side, send, C.byref(ptr), C.byref(cnt)))
                        else:
                            _check(L.sk_field_halo_n(f, side, send, cells, C.byref(ptr), C.byref(cnt)))
                        views[(r, sp, side, send)] = _dev_tensor(ptr.value, cnt.value, 0)
        for sp in species:  # rank0 upper halo <- rank1 lower interior, and back
            views[(0, sp, 1, 0)].copy_(views[(1, sp, 0, 1)])
            views[(1, sp, 0, 0)].copy_(views[(0, sp, 1, 1)])
        torch.cuda.synchronize()

    reduce_rho()
    for ctx, h, *_ in shards:
        _check(L.sk_state_phase(h, 1))
    shrinks = 0
    last_need, widths, resweeps = 1, set(), 0
    for step in range(12):
        if v_adjust:
            ref.run_step()
        else:
            ref.strang_step()
        for ctx, h, *_ in shards:
            _check(L.sk_state_phase(h, 2))
        reduce_rho()
        if not adaptive:
            exchange()
            for ctx, h, *_ in shards:
                _check(L.sk_state_phase(h, 3))
        else:
            bound = 1 if step % 2 else last_need + 1
            for ctx, h, *_ in shards:
                _check(L.sk_state_set_vhalo(h, 1, bound))
                _check(L.sk_state_phase(h, 6))
                _check(L.sk_state_phase(h, 7))
            sync()
            needs = []
            for ctx, h, *_ in shards:
                nd = C.c_int()
                _check(L.sk_state_vhalo_need(h, C.byref(nd)))
                needs.append(nd.value)
            assert needs[0] == needs[1] >= 1  # E is replicated: the same width on both sides
            last_need = needs[0]
            widths.add(last_need)
            for ctx, h, *_ in shards:
                _check(L.sk_state_set_vhalo(h, last_need, bound))
            exchange()
            resweep = last_need > bound or step % 3 == 2  # (also on purpose: phase 9 is exact too)
            for ctx, h, *_ in shards:
                _check(L.sk_state_phase(h, 9 if resweep else 8))
            resweeps += resweep
        if post:  # post limiter V reads one cell across the shard edge
            exchange(1)
            for ctx, h, *_ in shards:
                _check(L.sk_state_phase(h, 5))
        if v_adjust:
            sync()
            fl = torch.minimum(shards[0][4], shards[1][4])
            for s in shards:
                s[4].copy_(fl)
            fl = fl.cpu().tolist()
            if any(fl):
                shrinks += 1
                exchange(hs, [sp for sp in (0, 1) if fl[sp]])
                for ctx, h, *_ in shards:
                    _check(L.sk_state_phase(h, 4))
    if v_adjust:
        assert shrinks >= 2
    if adaptive:
        assert resweeps >= 1 and max(widths) < halo, (widths, resweeps)
    for sp in (0, 1):
        parts = []
        for ctx, h, _, plan, _ in shards:
            f = sk.NodalField(ctx, sp, None, _handle=L.sk_state_field(h, sp))
            parts.append(f.download())
            assert f.vmax() == ref.field(sp).vmax()
        got = np.concatenate(parts)
        assert rel(got, ref.field(sp).download()) <= 1e-12, f"species {sp}"
    for ctx, h, *_ in shards:
        L.sk_state_destroy(h)


@pytest.mark.parametrize("k,nf,nc,m", [(3, 512, 1024, 1), (2, 1031, 2099, 3), (3, 4096, 8192, 1),
                                       (2, 1024, 256, 8), (1, 2048, 4096, 1), (3, 300, 421, 2)])
def test_poisson_cluster_equals_single_cta(sk, k, nf, nc, m):
    """the cluster Poisson solve (rows over 8-16 CTAs, DSMEM neighbours) replays
    the single-CTA block-cyclic reduction row for row: bitwise equal E, phi"""
    grid = sk.Grid1D.three_block(-200.0, 200.0, nf, nc, m)
    ctx = sk.Context(grid, k)
    rng = np.random.default_rng(nf * 7 + nc)
    rho = rng.standard_normal(ctx.nx * ctx.p) * 0.3
    op = sk.PoissonOperator(ctx)
    a = op.solve(rho)
    Ea, pa = a.E.cpu().numpy().copy(), a.phi.cpu().numpy().copy()
    os.environ["SK_POISSON_SINGLE"] = "1"
    try:
        b = op.solve(rho)
    finally:
        del os.environ["SK_POISSON_SINGLE"]
    assert np.array_equal(Ea, b.E.cpu().numpy())
    assert np.array_equal(pa, b.phi.cpu().numpy())
    assert np.isfinite(Ea).all() and np.abs(Ea).max() > 0


def test_sharded_state_one_rank_matches_run_steps(sk):
    """ShardedState (the torchrun path of bench.py --gpus N) on one NCCL rank
    against SimulationState.run_steps: same run() loop bodies, including the
    host-side cut-off protocol (stream ordering of the decision read)"""
    import socket

    import torch.distributed as dist

    from paper_2408_11235_b200.sharding import ShardedState

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cfg = cfg_of(sk, k=3, nf=16, nc=32, m=1, nv=64, mu=1836.0, limiter="sldg", v_adjust=True)
    ref = sk.SimulationState(cfg)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        st = ShardedState(cfg, 0, 1, halo=4)
        for _ in range(23):
            st.step()
        ref.run_steps(23)
        assert ref.shrinks(0)[0] >= 2
        for sp in (0, 1):
            assert st.f[sp].vmax() == ref.field(sp).vmax()
            assert rel(st.f[sp].download(), ref.field(sp).download()) <= 1e-12
        st.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
@pytest.mark.parametrize("kw", [
    dict(k=2, nf=8, nc=16, m=2, nv=32, limiter="sldg", scenario="injection", t0=0.35),
    dict(k=3, nf=16, nc=32, m=1, nv=48, mu=1836.0, limiter="sldg", scenario="injection", t0=1.05),
    dict(k=3, nf=6, nc=12, m=1, nv=24, mu=1836.0, limiter="minmod+line", scenario="injection", t0=0.8),
    dict(k=2, nf=8, nc=16, m=8, nv=32, limiter="sldg", scenario="injection", t0=0.35, ghost_cap=1)],
    ids=["k2_m2", "k3_mu1836", "k3_post", "k2_m8_ghosts_in_kernel"])
def test_injection_scenario(sk, ora, kw, exact, monkeypatch):
    """§8f N2: the injection source half steps on the device (host exp tables
    per v-grid level) -- bitwise trajectories in exact mode, 1e-12 in fast
    mode -- across the source window's end and velocity shrinks. Both half
    steps ride in the x sweeps (first: added to the cells as read, in the sweep,
    its fixup and the transferred 3-block ghosts; second: added to the outputs,
    after the clamp for troubled cells); k3_post keeps the second one separate
    (post X runs between)."""
    import dataclasses

    kw = dict(kw)
    if "ghost_cap" in kw:  # 3-block ghosts beyond the pre-pass buffer: evaluated in the sweep
        monkeypatch.setenv("SK_XGHOST_CAP", str(kw.pop("ghost_cap")))
    cfg = cfg_of(sk, **kw)
    o = ora.state(**cfg.oracle_kwargs())
    st = sk.SimulationState(cfg, exact=exact)
    for sp in (0, 1):
        assert not st.field(sp).download().any()
    # the fused path launches no separate source kernels: as many kernels per
    # loop body as the blob scenario on the same grid (with a post limiter two
    # more: the second source half step, and the first x sweep, which carries
    # the source, leaves its post flags to the separate pass -- and in fast
    # mode the charge density to its two-kernel pass, one more than blob's
    # fused reduction)
    blob = sk.SimulationState(dataclasses.replace(cfg, scenario="blob"), exact=exact)
    l0, b0 = st.launches(), blob.launches()
    blob.run_step()
    for s in range(14):
        o.step()
        st.run_step()
        if s == 0:
            extra = (st.launches() - l0) - (blob.launches() - b0)
            assert extra == ((2 if exact else 3) if "+" in kw["limiter"] else 0), extra
        for sp in (0, 1):
            got, want = st.field(sp).download(), o.field(sp)
            if exact:
                assert np.array_equal(got, want), f"step {s + 1} species {sp}"
            else:
                assert rel(got, want) <= F_TOL, f"step {s + 1} species {sp}"
            assert st.field(sp).vmax() == o.vmax(sp)
    assert st.shrinks(0)[0] >= 2


def test_diagnostics_and_outputs_match_reference(sk, ref, tmp_path):
    """§8f N3: wall fluxes, state time, SOLKSNP1 snapshots and a whole run()
    with files against the reference's own diagnostics.cpp / run.cpp (exact
    mode: f, E and the fluxes bitwise; the masses come from a parallel device
    reduction and agree to 1e-12)"""
    kw = dict(k=3, nf=16, nc=32, m=1, nv=48, mu=1836.0, limiter="sldg")
    cfg = cfg_of(sk, **kw)
    st = sk.SimulationState(cfg, exact=True)
    r = ref.state(**cfg.oracle_kwargs())
    for _ in range(12):
        st.run_step()
        r.step()
    assert st.time() == r.time()
    for sp in (0, 1):
        for side in (0, 1):
            assert st.wall_flux(sp, side) == r.wall_flux(sp, side), (sp, side)
    a, b = tmp_path / "gpu", tmp_path / "ref"
    a.mkdir()
    b.mkdir()
    st.write_snapshot(a)
    r.write_snapshot(b)
    for ext in (".bin", ".meta"):
        assert (a / f"snapshot_12{ext}").read_bytes() == (b / f"snapshot_12{ext}").read_bytes()
    fs = st.sample_fluxes()
    assert fs["je_plus"] == r.wall_flux(0, 1)[0] and fs["t"] == r.time()
    # whole run() with files: flux.csv rows, snapshots, profiles
    ra, rb = tmp_path / "run_gpu", tmp_path / "run_ref"
    out = sk.run(cfg, nsteps=25, cadence=5, snapshot_cadence=10, profile_cadence=10,
                 out_dir=str(ra), exact=True)
    assert out["exit_code"] == 0 and out["steps_done"] == 25
    ref.state(**cfg.oracle_kwargs()).run_files(25 * cfg.dt, 5, 10, 10, rb)
    ga = np.loadtxt(ra / "flux.csv", delimiter=",", skiprows=1)
    gb = np.loadtxt(rb / "flux.csv", delimiter=",", skiprows=1)
    assert ga.shape == gb.shape == (6, 12)
    cols = [0, 1, 2, 3, 4, 5, 6, 9, 10, 11]  # t, fluxes, E energy, vmax: bitwise
    assert np.array_equal(ga[:, cols], gb[:, cols])
    assert np.abs(ga[:, 7:9] - gb[:, 7:9]).max() <= 1e-12 * np.abs(gb[:, 7:9]).max()
    for step in (0, 10, 20):
        assert (ra / f"snapshot_{step}.bin").read_bytes() == (rb / f"snapshot_{step}.bin").read_bytes()
        assert (ra / f"profiles_{step}.csv").read_text() == (rb / f"profiles_{step}.csv").read_text()
    # run.log (run.cpp:103-112,135-143,159-167): the same lines; the shrink
    # mass deltas are rounding-level differences of two sums (1e-13), compared
    # to 1e-11; the phase-timing line has the reference's keys
    la, lb = (ra / "run.log").read_text().splitlines(), (rb / "run.log").read_text().splitlines()
    assert len(la) == len(lb)
    for x, y in zip(la, lb):
        if y.startswith("phase timings [s]:"):
            assert [t.split("=")[0] for t in x.split()] == [t.split("=")[0] for t in y.split()]
        elif "(mass delta " in y:
            px, dx = x.split("(mass delta ")
            py, dy = y.split("(mass delta ")
            assert px == py
            assert abs(float(dx.rstrip(")")) - float(dy.rstrip(")"))) <= 1e-11
        else:
            assert x == y


@pytest.mark.parametrize("mode", ["minmod+simple", "minmod+line", "meanerr+simple", "meanerr+line"])
def test_post_limiters_conserve_mass(sk, mode):
    """C4 conservation check: the WENO modifiers are mean-preserving (the
    reference's design, limiters.cpp:102-165), so a post-limiter pass leaves
    each species' mass unchanged to rounding, on the C3 mesh after a few
    steps (steep, limited data)"""
    import dataclasses

    cfg = dataclasses.replace(sk.named_config("C3"), limiter="sldg")
    st = sk.SimulationState(cfg)
    st.run_steps(6)
    lim = sk.LimiterConfig.parse(mode)
    for sp in (0, 1):
        f = st.field(sp)
        for direction in (0, 1):
            before = f.mass()
            sk.apply_post_limiter(f, direction, lim)
            assert abs(f.mass() - before) <= 1e-13 * abs(before), (sp, direction)


@pytest.mark.gpu
def test_run_from_config_file(sk, ref, tmp_path):
    """§8f N4: `solkin run --config` through the C++ mirror (resolve_run_config +
    run(const RunConfig&)) and the Python RunConfig write the same files (same
    library, bitwise), and match the reference's run() on that config"""
    import shutil
    import subprocess

    if not shutil.which("g++"):
        pytest.skip("no g++")
    from paper_2408_11235_b200 import _native

    tool = str(tmp_path / "config_tool")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-o", tool,
                        os.path.join(ROOT, "tests", "cpp", "config_tool.cpp"), _native.LIB,
                        "-Wl,-rpath," + os.path.dirname(_native.LIB)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    cpp_dir, py_dir, ref_dir = tmp_path / "cpp", tmp_path / "py", tmp_path / "ref"
    text = ("# small injection-free blob run\nk = 2\nmu = 1836\nmesh.fine_block_cells = 16\n"
            "mesh.coarse_block_cells = 32\nv_cells = 40\nlimiter = sldg\nt_final = 1.2\n"
            "output.cadence = 3\noutput.snapshot_cadence = 6\noutput.profile_cadence = 6\n")
    cfg_path = tmp_path / "run.cfg"
    cfg_path.write_text(text + f"output.dir = {cpp_dir}\n")
    r = subprocess.run([tool, "run", str(cfg_path), "-"], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.startswith("exit 0 steps 12"), r.stdout + r.stderr
    cfg = sk.RunConfig.from_file(str(cfg_path))
    cfg.out_dir = str(py_dir)
    cfg.resolve()
    cfg.validate()
    out = sk.run(cfg)
    assert out["exit_code"] == 0 and out["steps_done"] == cfg.nsteps() == 12
    for name in ("flux.csv", "snapshot_6.bin", "snapshot_12.bin", "profiles_12.csv"):
        assert (cpp_dir / name).read_bytes() == (py_dir / name).read_bytes(), name
    ref.state(**cfg.oracle_kwargs()).run_files(cfg.t_final, cfg.cadence, cfg.snapshot_cadence,
                                               cfg.profile_cadence, ref_dir)
    # config_resolved.cfg (run.cpp:70-73): both mirrors write the reference's echo
    ea = (cpp_dir / "config_resolved.cfg").read_text().splitlines()
    eb = (py_dir / "config_resolved.cfg").read_text().splitlines()
    assert [x for x in ea if not x.startswith("output.dir")] == [x for x in eb if not x.startswith("output.dir")]
    if (ref_dir / "config_resolved.cfg").exists():
        er = (ref_dir / "config_resolved.cfg").read_text().splitlines()
        assert [x.split(" = ")[0] for x in er] == [x.split(" = ")[0] for x in eb]
    gb = np.loadtxt(ref_dir / "flux.csv", delimiter=",", skiprows=1)
    ga = np.loadtxt(py_dir / "flux.csv", delimiter=",", skiprows=1)
    assert ga.shape == gb.shape == (5, 12)
    # fast mode: t, masses and v_max to 1e-12 relative; the wall fluxes and the
    # E energy follow E's absolute contract, 1e-12 * max(1, scale) (early E is
    # ~1e-5 and carries the rho cancellation: 3e-11 relative even between two
    # CPU builds -- SURVEY §8c)
    rel, ab = [0, 7, 8, 10, 11], [1, 2, 3, 4, 5, 6, 9]
    scale = np.maximum(np.abs(gb[:, rel]).max(axis=0), 1e-300)
    assert (np.abs(ga[:, rel] - gb[:, rel]) / scale).max() <= 1e-12
    tol = 1e-12 * np.maximum(1.0, np.abs(gb[:, ab]).max(axis=0))
    assert (np.abs(ga[:, ab] - gb[:, ab]) <= tol).all()
    # exact mode on the same config reproduces the reference's rows (t, fluxes,
    # E energy, v_max bitwise; the masses come from a parallel reduction)
    ex_dir = tmp_path / "exact"
    out = sk.run(cfg, out_dir=str(ex_dir), exact=True)
    assert out["exit_code"] == 0 and out["steps_done"] == 12
    ge = np.loadtxt(ex_dir / "flux.csv", delimiter=",", skiprows=1)
    cols = [0, 1, 2, 3, 4, 5, 6, 9, 10, 11]
    assert np.array_equal(ge[:, cols], gb[:, cols])
    assert np.abs(ge[:, 7:9] - gb[:, 7:9]).max() <= 1e-12 * np.abs(gb[:, 7:9]).max()


def test_c3_full_size_run_matches_reference(sk, ref):
    """C3 at BASELINE size (2048x4096 cells per species, k=3, mu=1836, sldg,
    cut-off on): 11 run() loop bodies (run.cpp:124-131) in exact mode against
    the reference's own loop (oracle/_ref, all host threads). f of both
    species, E, v_max and the shrink counts must be bitwise the reference's
    in exact mode. The 11 steps include two cut-off shrinks per species (the
    last on step 11). Fast mode: test_c3_fast_mode_within_reference_envelope."""
    cfg = sk.named_config("C3")
    n = 11
    st = sk.SimulationState(cfg, exact=True)
    st.run_steps(n)
    st.ctx.synchronize()
    r = ref.state(threads=os.cpu_count() or 1, **cfg.oracle_kwargs())
    r.run(n)
    assert st.step_index() == r.step_index() == n
    assert np.array_equal(st.E(), r.E())
    for sp in (0, 1):
        assert st.shrinks(sp)[0] == r.shrinks(sp), f"shrinks sp{sp}"
        assert st.field(sp).vmax() == r.vmax(sp), f"v_max sp{sp}"
        got, want = st.field(sp).download(), r.field(sp)
        assert got.shape == want.shape and np.array_equal(got, want), \
            f"sp{sp}: max rel diff {rel(got, want):.3e}"
    st.close()



def test_c3_fast_mode_within_reference_envelope(sk):
    """The benchmarked (fast) mode at the BASELINE C3 size, stepped beside exact
    mode (= the reference bit for bit, test_c3_full_size_run_matches_reference),
    for 11 run() loop bodies including two cut-off shrinks per species.

    Bound: ENV_C x the reference's own noise envelope at C3
    (tests/golden/c3_envelope.npz, made offline by make_c3_envelope.py: the
    reference restatement against itself with the charge density summed in
    the other species order, with another LAPACK, and built with FMA), per
    step, for f of both species, E, and the diagnostics mass, L2, electric
    energy, momentum and kinetic energy. Shrink steps and v_max identical."""
    env = np.load(os.path.join(ROOT, "tests", "golden", "c3_envelope.npz"))
    cfg = sk.named_config("C3")
    n = int(env["steps"][-1])
    ex, fast = sk.SimulationState(cfg, exact=True), sk.SimulationState(cfg)
    keys = ("mass_e", "mass_i", "l2_e", "l2_i", "e_energy", "mom_e", "mom_i", "ekin_e", "ekin_i")
    worst = {}
    for s in range(1, n + 1):
        ex.run_step()
        fast.run_step()
        i = s - 1
        Ex, Ef = ex.E(), fast.E()
        assert np.abs(Ex).max() == env["Emax"][i]  # exact mode is the envelope's reference run
        got = {"dE": np.abs(Ef - Ex).max()}
        for sp, nm in ((0, "df_e"), (1, "df_i")):
            got[nm] = rel(fast.field(sp).download(), ex.field(sp).download())
        sx, sf = ex.summary(), fast.summary()
        for k in keys:
            got["d_" + k] = abs(sf[k] - sx[k])
        for key, v in got.items():
            e = float(env["env_" + key][i])
            # a diagnostic the perturbations left bitwise equal gets a 4-ulp floor
            floor = 4 * np.spacing(abs(float(env["ref_" + key[2:]][i]))) if key.startswith("d_") else 0.0
            bound = ENV_C * e + floor
            worst[key] = max(worst.get(key, 0.0), v / bound if bound > 0 else (0.0 if v == 0 else np.inf))
            assert v <= bound, f"step {s} {key}: {v:.3e} > {ENV_C:g} x envelope {e:.3e} (+{floor:.1e})"
        for sp in (0, 1):
            assert fast.field(sp).vmax() == ex.field(sp).vmax(), f"v_max sp{sp} step {s}"
    for sp in (0, 1):
        assert fast.shrinks(sp) == ex.shrinks(sp)
    print("worst ratio to the bound per quantity:", {k: round(v, 3) for k, v in worst.items()})
    fast.close()
    ex.close()


# ---------------------------------------------------------------------------
# full-size parity of the BASELINE configs 2, 4 and 5 (VERDICT r1 "Next" 2)
# ---------------------------------------------------------------------------
def _free_gpu():
    import gc

    import torch

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def test_c2_full_size_run_matches_reference(sk, ref, ora):
    """BASELINE config 2 at its size: 512x512 cells per species, k=2, sLdG,
    three-block sheath mesh with refinement m=8 at both walls (coarse/fine
    ghost transfer, adaptivity.cpp:169-207). 10 run() loop bodies
    (run.cpp:124-131): exact mode bitwise against the reference's own loop
    (oracle/_ref); fast mode (stepwise and with graph replays) within
    ENV_C x the reference's noise envelope at steps 1 and 10."""
    cfg = sk.named_config("C2")
    assert (cfg.nx, cfg.v_cells, cfg.k, cfg.refinement_ratio) == (512, 512, 2, 8)
    n = 10
    st = sk.SimulationState(cfg, exact=True)
    st.run_steps(n)
    r = ref.state(threads=os.cpu_count() or 1, **cfg.oracle_kwargs())
    r.run(n)
    assert st.step_index() == r.step_index() == n
    assert np.array_equal(st.E(), r.E())
    for sp in (0, 1):
        assert st.shrinks(sp)[0] == r.shrinks(sp) and st.field(sp).vmax() == r.vmax(sp)
        assert np.array_equal(st.field(sp).download(), r.field(sp)), f"sp{sp}"
    st.close()
    env = _envelope(ora, cfg, n)
    for batched in (False, True):
        fast = sk.SimulationState(cfg)
        if batched:
            fast.run_steps(1)
            fast.run_steps(n - 1)
            check = (n,)
        o = ora.state(**cfg.oracle_kwargs())
        for s in range(1, n + 1):
            if not batched:
                fast.run_step()
            o.step()
            if s in ((1, n) if not batched else check):
                ef, eE = env[s]
                for sp in (0, 1):
                    assert rel(fast.field(sp).download(), o.field(sp)) <= max(F_TOL, ENV_C * ef), (batched, s, sp)
                    assert fast.field(sp).vmax() == o.vmax(sp)
                E_o = o.E()
                assert np.abs(fast.E() - E_o).max() <= max(1e-12 * max(1.0, np.abs(E_o).max()), ENV_C * eE)
        fast.close()


@pytest.mark.parametrize("mode", ["minmod+simple", "minmod+line", "meanerr+simple", "meanerr+line"])
def test_c4_post_limiters_full_size_match_reference(sk, ref, mode):
    """BASELINE config 4 on the C3 mesh (2048x4096 cells per species, k=3,
    mu=1836, cut-off on) with each literature post limiter
    (limiters.cpp:280-345, after every directional sweep): 2 run() loop bodies
    (the first with both species' cut-off shrink) in exact mode bitwise
    against the reference's own loop; fast mode within 1e-12 of it."""
    _free_gpu()
    cfg = sk.named_config("C3", limiter=mode)
    n = 2
    r = ref.state(threads=os.cpu_count() or 1, **cfg.oracle_kwargs())
    r.run(n)
    st = sk.SimulationState(cfg, exact=True)
    st.run_steps(n)
    assert np.array_equal(st.E(), r.E())
    for sp in (0, 1):
        assert st.shrinks(sp)[0] == r.shrinks(sp) == 1 and st.field(sp).vmax() == r.vmax(sp)
        assert np.array_equal(st.field(sp).download(), r.field(sp)), f"{mode} sp{sp}"
    ex = [st.field(sp).download() for sp in (0, 1)]
    st.close()
    st.ctx.close()
    fast = sk.SimulationState(cfg)
    fast.run_steps(n)
    for sp in (0, 1):
        assert rel(fast.field(sp).download(), ex[sp]) <= F_TOL, f"{mode} fast sp{sp}"
    fast.close()
    fast.ctx.close()


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_c5_full_size_sampled_lines(sk, ora, exact):
    """BASELINE config 5 at its size (16384x16384 cells per species, k=3,
    mu=1836, sLdG: 137 GB of f on one B200): after 2 run() loop bodies, one
    x half sweep and one v sweep (strong synthetic field, multi-cell shifts)
    of the whole state; 16 x lines and 16 v lines per species (65536 values
    each) sampled and recomputed by the oracle: bitwise in exact mode, 1e-12
    in fast mode. A whole C5 body on the reference is not run: its serial
    blob fill and serial cut-off shrink (both species shrink at step 1) take
    over 10 minutes on the host."""
    _free_gpu()
    cfg = sk.named_config("C5")
    st = sk.SimulationState(cfg)
    st.run_steps(2)
    st.ctx.synchronize()
    st.ctx.set_exact_reductions(exact)
    p = cfg.k + 1
    nx, nv = cfg.nx, cfg.v_cells
    nxp, nvp = nx * p, nv * p
    rng = np.random.default_rng(11)
    grid = st.ctx.grid
    lim = sk.LimiterConfig.parse("sldg")
    nodes, _ = ora.gauss_legendre(cfg.k)
    for sp, spar in ((0, sk.SpeciesParams.electron()), (1, sk.SpeciesParams.ion(cfg.mu))):
        f = st.field(sp)
        vleft, vdx, _ = f.v_grid()
        rows = rng.choice(nvp, 16, replace=False)
        before = {int(r): f.download_2d(int(r) * nxp, nxp, 1, nxp)[0] for r in rows}
        sk.advect_x(f, 0.5 * cfg.dt, spar, sk.SweepOptions(limiter=lim))
        for r, b in before.items():
            vc, vn = divmod(r, p)
            vnode = (vleft + vc * vdx) + vdx * nodes[vn]
            want = ora.advect_x_line(cfg.k, grid.left, grid.cells, grid.dx, vnode / spar.sqrt_mu,
                                     0.5 * cfg.dt, b, inline_sldg=True)
            assert _same(f.download_2d(r * nxp, nxp, 1, nxp)[0], want, exact), f"x line {r} sp{sp}"
        cols = rng.choice(nxp, 16, replace=False)
        vin = np.stack([f.download_2d(int(c), 1, nvp, nxp)[:, 0] for c in cols])
        x = np.linspace(-1, 1, nxp)
        E = 0.3 * np.sin(3 * x)
        sk.advect_v(f, cfg.dt, E, spar, sk.SweepOptions(limiter=lim))
        vout = np.stack([f.download_2d(int(c), 1, nvp, nxp)[:, 0] for c in cols])
        want = ora.advect_v_lines(cfg.k, vin, 0, nv, 0, E[cols], spar.charge_sign, spar.sqrt_mu, cfg.dt, vdx,
                                  limiter="sldg")
        assert _same(vout, want, exact), f"v lines sp{sp}"
    st.close()
    st.ctx.close()
    _free_gpu()


def test_no_out_of_bounds_writes(sk):
    """Memory-safety stand-in for compute-sanitizer (closed on the GPU pool,
    SURVEY.md §5): every state buffer between sentinel guard zones, 12 run()
    loop bodies of five small configurations touching every kernel family in
    both arithmetic modes, not one guard word overwritten."""
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_steps.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_bench_sharded_one_rank_line(sk, monkeypatch, capsys):
    """bench.py's torchrun path (sharding.bench_sharded) end to end on one NCCL
    rank: the JSON line carries the contract keys, the per-kernel roofline from
    the per-phase window, and e2e through the sharded API."""
    import argparse
    import json
    import socket

    import bench
    from paper_2408_11235_b200 import sharding

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    for k, v in dict(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                     MASTER_PORT=str(port)).items():
        monkeypatch.setenv(k, v)
    cfg = cfg_of(sk, k=3, nf=64, nc=128, m=1, nv=128, mu=1836.0, limiter="sldg")
    args = argparse.Namespace(steps=4, warmup=3, config="C3", no_e2e=False, e2e_steps=1)
    sharding.bench_sharded(args, cfg, bench.METRIC, bench.UNIT, {"workload": "test"})
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "roofline",
                "phases_ms_per_step", "gpu_launches", "clocks", "e2e"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["value"] > 0
    assert line["roofline"]["kernel"] in ("x_sweep_1", "x_sweep_2", "v_sweep")
    assert 0 < line["roofline"]["frac"] < 1.5


def test_field_perturb_stress_input(sk):
    """bench.py --stress (SURVEY.md §8d stress variant): f *= 1 + amp xi with
    xi uniform in [-1, 1) from a device hash of (seed, index) -- bounded,
    roughly zero-mean, reproducible for a seed, different across seeds."""
    cfg = cfg_of(sk, k=3, nf=16, nc=32, m=1, nv=64, mu=1836.0, limiter="sldg")
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    f0 = a.field(0).download()
    a.field(0).perturb(20240817, 0.01)
    b.field(0).perturb(20240817, 0.01)
    fa, fb = a.field(0).download(), b.field(0).download()
    assert np.array_equal(fa, fb)
    nz = f0 != 0
    xi = (fa[nz] / f0[nz] - 1.0) / 0.01
    assert xi.min() >= -1.0 - 1e-9 and xi.max() < 1.0 + 1e-9
    assert abs(xi.mean()) < 0.05 and xi.std() > 0.5
    b.field(1).perturb(1, 0.01)
    assert not np.array_equal(b.field(1).download(), a.field(1).download())
    a.run_steps(2)  # the perturbed state steps (limiter active)
    assert np.isfinite(a.field(0).download()).all()


def test_bench_single_gpu_line_variants(sk):
    """bench.py's single-GPU line end to end (C1, small): the contract keys,
    e2e with its copied bytes, the CPU baseline, and the SURVEY.md §8(d)
    variant switches (--stress, --no-cutoff) reflected in config."""
    import json
    import subprocess
    import sys

    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C1", "--steps", "3", "--warmup", "3"]
    r = subprocess.run(base + ["--cpu-budget", "2", "--exact-steps", "2"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
                "gpu_launches", "exact_mode"):
        assert key in line, key
    assert line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["cpu_baseline"]["value"] > 0
    r = subprocess.run(base + ["--no-cpu", "--no-e2e", "--exact-steps", "0", "--stress", "--no-cutoff"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert "stress" in line["config"] and "cut-off off" in line["config"]["workload"]


def test_programmatic_dependent_launch_mode_same_bits(sk, tmp_path):
    """SK_PDL=1 (launch attribute + early trigger; off by default, measured no
    gain, profiles/r02_pdl.txt): every kernel waits for its predecessor's
    completion at entry, so a run gives the same bits as without it."""
    import subprocess
    import sys

    script = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2408_11235_b200 as sk\n"
        "cfg = sk.RunConfig(k=3, fine_block_cells=16, coarse_block_cells=32, refinement_ratio=2, v_cells=64,"
        " mu=1836.0, limiter='sldg')\n"
        "st = sk.SimulationState(cfg)\n"
        "st.run_steps(12)\n"
        "np.save(sys.argv[1], np.concatenate([st.field(0).download(), st.field(1).download(), st.E()]))\n" % ROOT)
    outs = []
    for mode in ("0", "1"):
        out = str(tmp_path / f"pdl{mode}.npy")
        r = subprocess.run([sys.executable, "-c", script, out], capture_output=True, text=True, timeout=600,
                           env={**os.environ, "SK_PDL": mode})
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


def test_run_with_fused_step_boundaries(sk, ora, tmp_path, monkeypatch):
    """run() (run.cpp:60-169) with the step boundaries fused (the default for
    C5-class states, forced here on a small mesh): batches end at output
    events and shrink-capable steps, so the flux rows land on the same steps
    and times, the shrink events in run.log on the same steps with the same
    v_max, and the values agree with the unfused run within the reference's
    rounding envelope (the fused charge density is grouped differently)."""
    cfg = cfg_of(sk, k=3, nf=16, nc=32, m=1, nv=64, mu=1836.0, limiter="sldg")
    outs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("SK_STEP_FUSION", mode)
        d = tmp_path / f"fuse{mode}"
        out = sk.run(cfg, nsteps=24, cadence=4, snapshot_cadence=0, profile_cadence=0, out_dir=str(d))
        assert out["exit_code"] == 0 and out["steps_done"] == 24
        outs[mode] = (np.loadtxt(d / "flux.csv", delimiter=",", skiprows=1), (d / "run.log").read_text())
    (fa, la), (fb, lb) = outs["1"], outs["0"]
    assert fa.shape == fb.shape
    assert np.array_equal(fa[:, 0], fb[:, 0])  # times
    ef, eE = _envelope(ora, cfg, 24)[24]
    scale = np.abs(fb[:, 1:]).max(axis=0)
    assert (np.abs(fa[:, 1:] - fb[:, 1:]) <= np.maximum(1e-12, 20.0 * ENV_C * max(ef, eE)) * np.maximum(scale, 1e-300)).all()
    sa = [ln.split("(mass delta")[0] for ln in la.splitlines() if "shrink" in ln.lower()]
    sb = [ln.split("(mass delta")[0] for ln in lb.splitlines() if "shrink" in ln.lower()]
    assert sa == sb and len(sa) >= 2


def test_run_steps_host_pipelined_equals_single_steps(sk):
    """sk_run_steps_host (bench.py's e2e leg): n drop-in steps over host arrays
    with the copies of consecutive steps overlapped on two streams give the
    same bits as n sk_run_step_host calls (the same bodies, every step's
    inputs uploaded and results downloaded), through a shrink."""
    cfg = cfg_of(sk, k=3, nf=16, nc=32, m=2, nv=64, mu=1836.0, limiter="sldg")
    a, b = sk.SimulationState(cfg), sk.SimulationState(cfg)
    fa = [a.f_e.download(), a.f_i.download()]
    fb = [b.f_e.download(), b.f_i.download()]
    a.run_steps_host(13, fa[0], fa[1])
    for _ in range(13):
        b.run_step_host(fb[0], fb[1])
    assert np.array_equal(fa[0], fb[0]) and np.array_equal(fa[1], fb[1])
    assert a.step_index() == b.step_index() == 13
    assert a.shrinks(0) == b.shrinks(0)
    # the host arrays hold the device state
    assert np.array_equal(fa[0], a.f_e.download()) and np.array_equal(fa[1], a.f_i.download())
