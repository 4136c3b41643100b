"""CPU, world_size 2 (gloo): the v-sharded host logic -- shard plan, halo
exchange, charge-density all-reduce -- with the C oracle as the per-rank
compute. A v sweep of the sharded field must equal the unsharded oracle v
sweep bit for bit, and the reduced charge density must equal the serial one
to rounding."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, nsteps, halo, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2408_11235_b200.sharding import VShardPlan, allreduce_rho, exchange_halos

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    ora = Oracle()
    st = ora.state(**cfg)
    for _ in range(nsteps):
        st.step()
    k, nv, nx = cfg["k"], cfg["nv"], st.nx
    p = k + 1
    plan = VShardPlan(nv, world, rank, halo)
    out = {}
    for sp in (0, 1):
        full = st.field(sp).reshape(nv * p, nx * p)  # rows: (vc, vn)
        rows = plan.ncell * p
        # local buffer: halo | interior | halo, interior copied from the full field only
        buf = torch.zeros((plan.ncell + 2 * halo) * p, nx * p, dtype=torch.float64)
        buf[halo * p: halo * p + rows] = torch.from_numpy(full[plan.cell0 * p: plan.cell0 * p + rows])
        h = halo * p
        exchange_halos(buf[h: 2 * h].contiguous().view(-1), buf[0:h].view(-1),
                       buf[rows: rows + h].contiguous().view(-1), buf[rows + h: rows + 2 * h].view(-1),
                       plan)
        E = st.E()
        sqrt_mu = 1.0 if sp == 0 else np.sqrt(cfg["mu"])
        charge = -1.0 if sp == 0 else 1.0
        # gather v lines (x dof major) of halo+interior cells this rank may read
        lo = halo - plan.gl
        hi = halo + plan.ncell + plan.gr
        local = buf.numpy()[lo * p: hi * p].T.copy()  # [nx*p, (gl+n+gr)*p]
        vleft, dv = -st.vmax(sp), 2 * st.vmax(sp) / nv
        res = ora.advect_v_lines(k, local, plan.gl, plan.ncell, plan.gr, E, charge, sqrt_mu,
                                 cfg["dt"], dv, limiter=cfg["limiter"])
        out[f"v{sp}"] = res.T.copy()  # [ncell*p, nx*p]
    # partial charge density of this shard, then the all-reduce
    from oracle.oracle import _dp  # noqa: F401
    nodes, w = ora.gauss_legendre(k)
    rho = np.zeros(nx * p)
    for sp, sign in ((1, 1.0), (0, -1.0)):
        full = st.field(sp).reshape(nv * p, nx * p)
        dv = 2 * st.vmax(sp) / nv
        for r in range(plan.cell0 * p, (plan.cell0 + plan.ncell) * p):
            rho += (sign * w[r % p] * dv) * full[r]
    rt = torch.from_numpy(rho)
    allreduce_rho(rt)
    out["rho"] = rt.numpy()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


CFGS = [dict(k=2, nf=8, nc=16, m=1, nv=32, limiter="sldg", v_adjust=0, dt=0.1, mu=400.0),
        dict(k=3, nf=6, nc=12, m=2, nv=24, mu=1836.0, limiter="none", v_adjust=0, dt=0.1)]


@pytest.mark.parametrize("cfg", CFGS, ids=["k2_sldg", "k3_m2"])
def test_sharded_v_sweep_and_rho_match_serial(ora, cfg):
    world, halo, nsteps = 2, 3, 4
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), cfg, nsteps, halo, d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    st = ora.state(**cfg)
    for _ in range(nsteps):
        st.step()
    E = st.E()
    rho_serial = st.charge_density()
    for sp in (0, 1):
        sqrt_mu = 1.0 if sp == 0 else np.sqrt(cfg.get("mu", 400.0))
        st.advect_v(sp, cfg["dt"], E, limited=True)
        full = st.field(sp).reshape(-1, st.nx * (cfg["k"] + 1))
        sharded = np.concatenate([p[f"v{sp}"] for p in parts], axis=0)
        assert np.array_equal(sharded, full), f"species {sp}"
    # rho cancels (int f_i - int f_e): compare against the size of the summed terms
    k = cfg["k"]
    _, w = ora.gauss_legendre(k)
    st2 = ora.state(**cfg)
    for _ in range(nsteps):
        st2.step()
    terms = 0.0
    for sp in (0, 1):
        full = np.abs(st2.field(sp).reshape(cfg["nv"] * (k + 1), -1))
        wr = np.tile(w, cfg["nv"]) * (2 * st2.vmax(sp) / cfg["nv"])
        terms = terms + (wr[:, None] * full).sum(axis=0)
    for p in parts:
        assert np.all(np.abs(p["rho"] - rho_serial) <= 1e-14 * terms + 1e-300)
    assert np.array_equal(parts[0]["rho"], parts[1]["rho"])  # every rank sees the same rho


def test_shard_plan():
    from paper_2408_11235_b200.sharding import VShardPlan, halo_cells_needed

    p = VShardPlan(nv=16384, nranks=8, rank=3, halo=16)
    assert (p.ncell, p.cell0, p.lower, p.upper, p.gl, p.gr) == (2048, 6144, 2, 4, 16, 16)
    p0 = VShardPlan(16384, 8, 0, 16)
    assert p0.lower is None and p0.gl == 0 and p0.gr == 16
    with pytest.raises(ValueError):
        VShardPlan(100, 8, 0, 4)
    # C5 electrons at |E| = 0.2: shift 0.2*0.1/(24/16384) = 13.65 cells -> 15
    assert halo_cells_needed(0.2, 0.1, 24 / 16384) == 15


def _cutoff_worker(rank, world, port, cfg, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import math

    import torch
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2408_11235_b200.sharding import VShardPlan, allreduce_shrink_flags, exchange_halos

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    ora = Oracle()
    st = ora.state(**cfg)
    st.step()
    k, nv, nx = cfg["k"], cfg["nv"], st.nx
    p = k + 1
    hs = math.ceil(0.05 * nv * 0.5) + 3  # sk_state_shrink_halo for the default policy
    plan = VShardPlan(nv, world, rank, hs)
    full = st.field(0).reshape(nv * p, nx * p)
    rows, h = plan.ncell * p, hs * p
    buf = torch.zeros((plan.ncell + 2 * hs) * p, nx * p, dtype=torch.float64)
    buf[h: h + rows] = torch.from_numpy(full[plan.cell0 * p: plan.cell0 * p + rows])
    exchange_halos(buf[h: 2 * h].contiguous().view(-1), buf[0:h].view(-1),
                   buf[rows: rows + h].contiguous().view(-1), buf[rows + h: rows + 2 * h].view(-1), plan)
    # the decision: only the ranks holding the probe cells evaluate; MIN makes it global
    ok_global = ora.state(**cfg)
    ok_global.step()
    want = int(ok_global.check_shrink(0))
    vmax = st.vmax(0)
    probe = vmax * (1 - 0.05 - 0.05)
    cells = [min(max(int((v + vmax) / (2 * vmax / nv)), 0), nv - 1) for v in (probe, -probe)]
    holds = any(plan.cell0 <= c < plan.cell0 + plan.ncell for c in cells)
    flags = torch.tensor([want if holds else 1, 1], dtype=torch.int32)
    allreduce_shrink_flags(flags)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), buf=buf.numpy(), flags=flags.numpy(),
             want=want, cell0=plan.cell0, ncell=plan.ncell, hs=hs)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_cutoff_decision_and_shrink_halos(ora):
    """the sharded velocity cut-off's host protocol: MIN-all-reduced decision
    equals the serial check, and the shrink-width halos hold the neighbours'
    old cells (what shrink_project reads across the shard edges)"""
    cfg = dict(k=2, nf=8, nc=16, m=1, nv=64, limiter="none", v_adjust=1, dt=0.1, mu=400.0)
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_cutoff_worker, args=(world, _free_port(), cfg, d), nprocs=world, join=True)
        parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(world)]
    st = ora.state(**cfg)
    st.step()
    p = cfg["k"] + 1
    full = st.field(0).reshape(cfg["nv"] * p, -1)
    for part in parts:
        assert int(part["flags"][0]) == int(part["want"])
        c0, n, hs = int(part["cell0"]), int(part["ncell"]), int(part["hs"])
        buf = part["buf"]
        lo = max(c0 - hs, 0)
        hi = min(c0 + n + hs, cfg["nv"])
        # every old cell in [c0-hs, c0+n+hs) that exists globally is present
        assert np.array_equal(buf[(lo - c0 + hs) * p:(hi - c0 + hs) * p], full[lo * p:hi * p])
