"""Quick GPU parity probe: prints max diffs of each operator vs the C oracle."""
import os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2408_11235_b200 as sk
from oracle import Oracle

O = Oracle()

def rel(a, b):
    m = np.abs(b).max()
    return np.abs(a - b).max() / (m if m > 0 else 1.0)

def unit(cfg, label):
    print(f"== {label}: {cfg}")
    ora = O.state(**cfg.oracle_kwargs())
    st = sk.SimulationState(cfg)
    ctx = st.ctx
    lim = sk.LimiterConfig.parse(cfg.limiter)
    # initial fields identical?
    for sp in (0, 1):
        print(f"  init f[{sp}] maxdiff", np.abs(st.field(sp).download() - ora.field(sp)).max())
    print("  init E maxdiff", np.abs(st.E() - ora.E()).max(), "max|E|", np.abs(ora.E()).max())
    # x sweep, bitwise
    half = 0.5 * cfg.dt
    spar = [sk.SpeciesParams.electron(), sk.SpeciesParams.ion(cfg.mu)]
    for sp in (0, 1):
        f = st.field(sp)
        f.upload(ora.field(sp))
        sk.advect_x(f, half, spar[sp], sk.SweepOptions(limiter=lim, max_ghost=-1))
        ora.advect_x(sp, half, limited=True, max_ghost=-1)
        d = np.abs(f.download() - ora.field(sp)).max()
        print(f"  advect_x sp{sp}: maxdiff {d:.3e} {'BITWISE' if d == 0 else ''}")
    # rho + poisson
    rho_o = ora.charge_density()
    rho_g = sk.charge_density(st.f_e, st.f_i).cpu().numpy()
    print(f"  rho: maxdiff {np.abs(rho_g-rho_o).max():.3e} max|rho| {np.abs(rho_o).max():.3e}")
    E_o, phi_o = ora.poisson_solve(rho_o)
    fp = sk.PoissonOperator(ctx).solve(rho_o)
    E_g = fp.E.cpu().numpy()
    print(f"  poisson: |dE| {np.abs(E_g-E_o).max():.3e} max|E| {np.abs(E_o).max():.3e} dphi {np.abs(fp.phi.cpu().numpy()-phi_o).max():.3e}")
    # v sweep bitwise with oracle E
    for sp in (0, 1):
        f = st.field(sp)
        f.upload(ora.field(sp))
        sk.advect_v(f, cfg.dt, E_o, spar[sp], sk.SweepOptions(limiter=lim))
        ora.advect_v(sp, cfg.dt, E_o, limited=True)
        d = np.abs(f.download() - ora.field(sp)).max()
        print(f"  advect_v sp{sp}: maxdiff {d:.3e} {'BITWISE' if d == 0 else ''}")
    # post limiters
    for mode in ("minmod+simple", "meanerr+line"):
        for dr in (0, 1):
            f = st.field(0)
            f.upload(ora.field(0))
            sk.apply_post_limiter(f, dr, sk.LimiterConfig.parse(mode))
            ora.post_limit(0, dr, mode)
            d = np.abs(f.download() - ora.field(0)).max()
            print(f"  post {mode} dir{dr}: maxdiff {d:.3e} {'BITWISE' if d == 0 else ''}")
    # shrink
    for sp in (0, 1):
        f = st.field(sp)
        f.upload(ora.field(sp))
        cg = sk.check_velocity_shrink(f, sk.VAdjustPolicy(cfg.adapt_p, cfg.adapt_gamma, cfg.adapt_tol))
        co = ora.check_shrink(sp)
        print(f"  check_shrink sp{sp}: gpu {cg} oracle {co}")
        rg = sk.shrink_velocity_domain(f, sk.VAdjustPolicy(cfg.adapt_p, cfg.adapt_gamma, cfg.adapt_tol))
        ro = ora.shrink(sp)
        d = np.abs(f.download() - ora.field(sp)).max()
        print(f"  shrink sp{sp}: maxdiff {d:.3e} vmax {rg['vmax_after']!r} vs {ora.vmax(sp)!r} mass {rg['mass_after']:.17g} vs {ro['mass_after']:.17g}")

def steps(cfg, label, n):
    print(f"== steps {label}")
    ora = O.state(**cfg.oracle_kwargs())
    st = sk.SimulationState(cfg)
    t0 = time.time()
    for i in range(n):
        st.run_step(); ora.step()
        if i in (0, 9, n - 1):
            st.ctx.synchronize()
            rf = [rel(st.field(sp).download(), ora.field(sp)) for sp in (0, 1)]
            dE = np.abs(st.E() - ora.E()).max()
            print(f"  step {i+1}: rel f {rf[0]:.2e} {rf[1]:.2e} |dE| {dE:.2e} max|E| {np.abs(ora.E()).max():.2e} "
                  f"shrinks gpu {st.shrinks(0)} {st.shrinks(1)} oracle {ora.shrinks(0)},{ora.last_shrink(0)} {ora.shrinks(1)},{ora.last_shrink(1)} "
                  f"vmax {st.f_e.vmax()==ora.vmax(0)} {st.f_i.vmax()==ora.vmax(1)}")
    print("  stats gpu", st.stats(), "\n  stats ora", ora.stats(), f" ({time.time()-t0:.1f}s)")

try:
    unit(sk.RunConfig(k=2, fine_block_cells=8, coarse_block_cells=16, refinement_ratio=1, v_cells=32, limiter="sldg"), "k2 m1")
    unit(sk.RunConfig(k=2, fine_block_cells=16, coarse_block_cells=16, refinement_ratio=4, v_cells=32, limiter="sldg"), "k2 m4")
    unit(sk.RunConfig(k=3, fine_block_cells=8, coarse_block_cells=16, refinement_ratio=2, v_cells=24, mu=1836, limiter="sldg"), "k3 m2")
    steps(sk.RunConfig(k=2, fine_block_cells=8, coarse_block_cells=16, refinement_ratio=1, v_cells=32, limiter="none"), "C1-mini none", 25)
    steps(sk.RunConfig(k=2, fine_block_cells=16, coarse_block_cells=16, refinement_ratio=4, v_cells=32, limiter="sldg"), "k2 m4 sldg", 25)
    steps(sk.RunConfig(k=3, fine_block_cells=8, coarse_block_cells=16, refinement_ratio=1, v_cells=24, mu=1836, limiter="meanerr+line"), "k3 meanerr+line", 12)
    steps(sk.named_config("C1"), "C1", 12)
except Exception:
    traceback.print_exc()
    sys.exit(1)
