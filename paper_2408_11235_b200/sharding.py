"""v-sharded multi-GPU step: one process per GPU.

Phase space is sharded along v: rank r of G holds v cells [r*nv/G, (r+1)*nv/G)
of each species for all x, plus `halo` cells below and above. Then

  * x sweeps are fully local (an x line is one v row);
  * the charge density is a local partial (fused into the first x sweep)
    followed by an all-reduce(sum) of nx*(k+1) doubles;
  * the Poisson solve is replicated (every rank gets the same E);
  * the v sweep reads up to `halo` cells from the neighbouring ranks. The
    exchange is sized per step from this step's E: the v tables (after the
    replicated Poisson solve) record max |i*|+1 over the x dofs, and exactly
    that many cells move point-to-point while the v chunks that read no halo
    cell are already being swept (interior first, edges after the exchange);
  * the velocity cut-off (adaptivity.cpp:16-130, run.cpp:98-114): the ranks
    holding the probe cells decide locally, an all-reduce(MIN) of two ints
    makes the decision global, and on a shrink step each rank exchanges the
    ceil(p*nv/2)+3 cells the projection reads across its shard edges.

Plumbing is torch.distributed: NCCL over NVLink/NVSwitch for device buffers,
gloo for the CPU tests (tests/test_sharding.py drive exactly these functions
with the C oracle as the per-rank compute). The literature post limiters
exchange one more one-cell halo between the v sweep and post limiter V.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

from . import _native as N


@dataclass(frozen=True)
class VShardPlan:
    nv: int       # global v cells
    nranks: int
    rank: int
    halo: int     # cells exchanged with each neighbour

    def __post_init__(self):
        if self.nranks < 1 or not 0 <= self.rank < self.nranks:
            raise ValueError("bad rank")
        if self.nv % self.nranks:
            raise ValueError("v_cells must divide by the rank count")
        if self.nranks > 1 and not 0 < self.halo <= self.ncell:
            raise ValueError("halo must be in 1..cells per shard")

    @property
    def ncell(self) -> int:
        return self.nv // self.nranks

    @property
    def cell0(self) -> int:
        return self.rank * self.ncell

    @property
    def lower(self):
        return self.rank - 1 if self.rank > 0 else None

    @property
    def upper(self):
        return self.rank + 1 if self.rank + 1 < self.nranks else None

    @property
    def gl(self) -> int:  # readable halo cells below (0 at the global wall)
        return self.halo if self.lower is not None else 0

    @property
    def gr(self) -> int:
        return self.halo if self.upper is not None else 0


def halo_cells_needed(max_abs_E: float, dt: float, dv: float, sqrt_mu_min: float = 1.0) -> int:
    """cells a v sweep can reach beyond its shard: |i*|+1 with
    i* = floor(-c E dt / (sqrt(mu) dv)) (advection.cpp:14-25, :226)."""
    import math

    return int(math.floor(max_abs_E * dt / (sqrt_mu_min * dv))) + 2


def exchange_halos(lower_send, lower_recv, upper_send, upper_recv, plan: VShardPlan, group=None):
    """Swap v halos with the neighbouring ranks. Each argument is a contiguous
    tensor of halo*(k+1) v rows (device tensors under NCCL, CPU under gloo):
    my lowest interior rows go to rank-1 (its upper halo), my highest to rank+1
    (its lower halo). Halos at the global v walls are left as they are (the
    kernels treat them as zero inflow)."""
    import torch.distributed as dist

    ops = []
    if plan.lower is not None:
        ops.append(dist.P2POp(dist.isend, lower_send, plan.lower, group))
        ops.append(dist.P2POp(dist.irecv, lower_recv, plan.lower, group))
    if plan.upper is not None:
        ops.append(dist.P2POp(dist.isend, upper_send, plan.upper, group))
        ops.append(dist.P2POp(dist.irecv, upper_recv, plan.upper, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def allreduce_rho(rho, group=None):
    """charge density = sum of the ranks' partial v moments (poisson.cpp:194-216)."""
    import torch.distributed as dist

    dist.all_reduce(rho, op=dist.ReduceOp.SUM, group=group)


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (no ownership)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _dev_tensor(ptr: int, n: int, device: int, typestr: str = "<f8"):
    import torch

    return torch.as_tensor(_DevView(ptr, n, typestr), device=f"cuda:{device}")


def allreduce_shrink_flags(flags, group=None):
    """cut-off decision: shrink only if no rank's probe cells failed (MIN)"""
    import torch.distributed as dist

    dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=group)


class ShardedState:
    """SimulationState sharded along v over the ranks of the default group."""

    def __init__(self, cfg, rank: int, nranks: int, halo: int = 16, device: int = 0, group=None):
        from .solver import Context, Grid1D, NodalField, _check

        self.cfg, self.group = cfg, group
        self.plan = VShardPlan(cfg.v_cells, nranks, rank, halo if nranks > 1 else 0)
        grid = Grid1D.three_block(-cfg.L, cfg.L, cfg.fine_block_cells, cfg.coarse_block_cells,
                                  cfg.refinement_ratio)
        self.ctx = Context(grid, cfg.k, cfg.penalty_scale, device)
        self.device = device
        h = C.c_void_p()
        ccfg = cfg.to_c()
        _check(N.lib().sk_state_create_shard(self.ctx.h, C.byref(ccfg), rank, nranks,
                                             self.plan.halo, C.byref(h)))
        self.h = h
        L = N.lib()
        self.f = [NodalField(self.ctx, sp, None, _handle=L.sk_state_field(h, sp), _owner=self)
                  for sp in (0, 1)]
        n_rho = self.ctx.nx * self.ctx.p
        self.rho = _dev_tensor(L.sk_state_rho_dev(h), n_rho, device)
        self.flags = _dev_tensor(L.sk_state_shrink_flags_dev(h), 2, device, "<i4")
        self.shrink_halo = int(L.sk_state_shrink_halo(h))
        # host mirror of the device cooldown gate (run.cpp:98-101, step_end_kernel):
        # steps on which no species may shrink need no decision round trip
        self._step = 0
        self._last_shrink = [-10, -10]
        from .solver import LimiterConfig

        self._post = LimiterConfig.parse(cfg.limiter).to_c().indicator != 0
        self._vbound = int(L.sk_state_vhalo_capacity(h)) if nranks > 1 else 0
        self.halo_widths = []  # exchanged v-halo cells per step (adaptive)
        # initial field: local moment (created) -> all-reduce -> Poisson
        self._reduce_rho()
        self._phase(1)

    def _phase(self, ph: int):
        from .solver import _check

        _check(N.lib().sk_state_phase(self.h, ph))

    def _reduce_rho(self):
        if self.plan.nranks == 1:
            return
        self.ctx.leave()
        allreduce_rho(self.rho, self.group)
        self.ctx.enter()

    def _exchange(self, cells=None, species=(0, 1), enter_leave=True):
        if self.plan.nranks == 1:
            return
        from .solver import _check

        if enter_leave:
            self.ctx.leave()
        for sp in species:
            f = self.f[sp]
            views = []
            for side in (0, 1):
                for send in (1, 0):
                    ptr, cnt = C.c_void_p(), C.c_size_t()
                    if cells is None:
                        _check(N.lib().sk_field_halo(f.h, side, send, C.byref(ptr), C.byref(cnt)))
                    else:
                        _check(N.lib().sk_field_halo_n(f.h, side, send, cells, C.byref(ptr), C.byref(cnt)))
                    views.append(_dev_tensor(ptr.value, cnt.value, self.device))
            exchange_halos(views[0], views[1], views[2], views[3], self.plan, self.group)
        if enter_leave:
            self.ctx.enter()

    def _cutoff(self):
        """run.cpp:98-114 across ranks: global decision, halo fill, shrink"""
        self._step += 1
        if not self.cfg.v_adjust:
            return
        if all(self._step - last < 10 for last in self._last_shrink):
            return
        # torch's stream (all-reduce, the read below) must follow the check
        # kernels on the library stream, and phase 4 must follow the all-reduce
        self.ctx.leave()
        if self.plan.nranks > 1:
            allreduce_shrink_flags(self.flags, self.group)
        fl = self.flags.cpu().tolist()  # the host decides whether halos must move
        self.ctx.enter()
        if not any(fl):
            return
        for sp in (0, 1):
            if fl[sp]:
                self._last_shrink[sp] = self._step
        self._exchange(self.shrink_halo, [sp for sp in (0, 1) if fl[sp]])
        self._phase(4)

    def step(self):
        """one run() loop body: x half sweep (+ local rho) | all-reduce rho |
        Poisson, v tables | [halo exchange of this step's width, overlapped
        with the interior v chunks] | edge v chunks, x half sweep, step end,
        local cut-off check | all-reduce decision, shrink halos | shrink"""
        self._phase(2)
        self._reduce_rho()
        if self.plan.nranks == 1:
            self._phase(3)
        else:
            self._v_sweep_adaptive()
        if self._post and self.plan.nranks > 1:
            self._exchange(1)  # post limiter V reads one cell across each shard edge
            self._phase(5)
        self._cutoff()

    def _v_sweep_adaptive(self):
        import torch

        from .solver import _check

        L = N.lib()
        self._phase(6)  # Poisson + v tables: this step's halo width -> pinned word
        ev = torch.cuda.Event()
        ev.record(self.ctx.stream)
        self._phase(7)  # v chunks that read no halo cell (shifts <= bound), runs on
        ev.synchronize()  # the library stream while the halos move below
        need = C.c_int()
        _check(L.sk_state_vhalo_need(self.h, C.byref(need)))
        need = max(1, need.value)
        cap = int(L.sk_state_vhalo_capacity(self.h))
        width = min(need, cap)  # (need > cap: the v tables raised "insufficient v halo")
        _check(L.sk_state_set_vhalo(self.h, width, self._vbound))
        torch.cuda.current_stream(self.device).wait_event(ev)
        self._exchange(enter_leave=False)
        self.ctx.enter()
        self._phase(8 if need <= self._vbound else 9)
        self.halo_widths.append(width)
        # interior bound of the next step: twice this step's width (E varies
        # slowly from step to step; a faster change only costs a re-sweep)
        self._vbound = min(cap, max(2 * need, need + 4))
        _check(L.sk_state_set_vhalo(self.h, width, self._vbound))

    def close(self):
        if getattr(self, "h", None):
            N.lib().sk_state_destroy(self.h)
            self.h = None
        self.ctx.close()


def bench_sharded(args, cfg, metric, unit, config):
    """bench.py under torchrun: N ranks, one GPU each, NCCL; device time is
    the max over ranks of the CUDA-event time around K steps. The line carries
    the same keys as the single-GPU one: roofline (whole step, 48 B/DoF
    against N x the measured HBM peak), e2e through the sharded API with host
    buffers, clocks of this rank's GPU, and the kernels launched."""
    import time

    import torch
    import torch.distributed as dist

    import bench

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    # halo capacity: the exchanged width follows this step's E (adaptive, from
    # the v tables); the capacity only bounds it -- |E| up to 2, or the
    # cut-off's shrink halo (ceil(p nv / 2) + 3 cells) when that is wider
    dv = 2 * cfg.vmax_e / cfg.v_cells
    halo = max(4, min(cfg.v_cells // world, halo_cells_needed(2.0, cfg.dt, dv)))
    st = ShardedState(cfg, rank, world, halo=halo, device=local)
    st.ctx.set_eager_errors(False)
    for _ in range(args.warmup):
        st.step()
    st.ctx.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = int(N.lib().sk_ctx_launch_count(st.ctx.h))
    clocks = bench.ClockSampler(local)
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(st.ctx.stream)
    for _ in range(args.steps):
        st.step()
    t1.record(st.ctx.stream)
    torch.cuda.synchronize()
    st.ctx.synchronize()
    clk = clocks.stop()
    launches = int(N.lib().sk_ctx_launch_count(st.ctx.h)) - launches0
    ms = torch.tensor([t0.elapsed_time(t1)], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    widths = list(st.halo_widths[-args.steps:])
    # second K-step window with per-phase CUDA events on every rank: the
    # per-kernel durations behind the roofline (max over ranks per phase)
    from .solver import _check

    _check(N.lib().sk_state_set_phase_timing(st.h, 1))
    nph = len(N.PHASES)
    msa, cnt = (C.c_double * nph)(), (C.c_long * nph)()
    _check(N.lib().sk_state_phase_times(st.h, msa, cnt, nph))  # clears
    for _ in range(args.steps):
        st.step()
    st.ctx.synchronize()
    _check(N.lib().sk_state_phase_times(st.h, msa, cnt, nph))
    _check(N.lib().sk_state_set_phase_timing(st.h, 0))
    ph = torch.tensor([msa[i] for i in range(nph)], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(ph, op=dist.ReduceOp.MAX)
    phases = {N.PHASES[i]: (float(ph[i]), int(cnt[i])) for i in range(nph) if cnt[i]}
    # e2e: every step moves this rank's shard host -> device and back
    e2e = None
    if not getattr(args, "no_e2e", False):
        n = st.f[0].size
        host = [torch.empty(n, dtype=torch.float64, pin_memory=True).numpy() for _ in (0, 1)]
        for sp in (0, 1):
            host[sp][:] = st.f[sp].download()
        k2 = max(1, getattr(args, "e2e_steps", 3))
        dist.barrier()
        w0 = time.perf_counter()
        dp = C.POINTER(C.c_double)
        for _ in range(k2):
            for sp in (0, 1):  # pinned buffers: DMA at PCIe speed
                N.lib().sk_field_upload_async(st.f[sp].h, host[sp].ctypes.data_as(dp), n)
            st.step()
            for sp in (0, 1):
                N.lib().sk_field_download_async(st.f[sp].h, host[sp].ctypes.data_as(dp), n)
            st.ctx.synchronize()
        wall = torch.tensor([time.perf_counter() - w0], device=f"cuda:{local}")
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
        e2e = {"value": cfg.dof_total * k2 / float(wall.item()), "unit": unit,
               "h2d_bytes_per_step": 2 * 8 * n * world, "d2h_bytes_per_step": 2 * 8 * n * world,
               "steps": k2, "api": "ShardedState (sk_state_create_shard / sk_state_phase, sk_field_upload_async)"}
    if rank == 0:
        value = cfg.dof_total * args.steps / (ms / 1e3)
        peak, peak_kind = bench.peaks()
        step_gbs = 3 * bench.BYTES_PER_DOF_SWEEP * cfg.dof_total * args.steps / (ms / 1e3) / 1e9
        cfgd = dict(config)
        cfgd["parallelism"] = f"v-shard x{world} (halo {halo} cells, NCCL all-reduce + P2P)"
        cfgd["v_cutoff"] = "on (sharded: all-reduced decision, halo on shrink steps)" if cfg.v_adjust else "off"
        cfgd["v_halo_exchanged_cells"] = {"max": max(widths) if widths else None,
                                          "mean": sum(widths) / len(widths) if widths else None,
                                          "capacity": int(N.lib().sk_state_vhalo_capacity(st.h))}
        # dominant kernel: per-rank sweep over 1/world of the DoF, 16 B/DoF
        sweeps = {"x_sweep_1", "x_sweep_2", "v_sweep"}
        dom = max((k for k in phases if k in sweeps), key=lambda k: phases[k][0])
        per_launch = phases[dom][0] / max(phases[dom][1], 1)
        alg = bench.BYTES_PER_DOF_SWEEP * cfg.dof_total / world
        achieved = alg / (per_launch / 1e3) / 1e9
        traffic = None
        try:
            with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "profiles", "ncu_traffic.json")) as f:
                t = json.load(f).get(getattr(args, "config", ""), {}).get(dom)
            traffic = t / world if t else None  # (single-GPU capture; a shard moves 1/world of it)
        except Exception:
            pass
        line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (blob initial condition, run.cpp:41-46)",
                "config": cfgd,
                "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                             "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                             "traffic": traffic, "alg_bytes_per_launch": alg, "ms_per_launch": per_launch,
                             "step_achieved_gbs": step_gbs, "step_peak_gbs": peak * world,
                             "step_frac": step_gbs / (peak * world),
                             "timing": "kernel ms: per-phase CUDA events over a second K-step window, "
                                       "max over ranks; achieved per GPU"},
                "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items()},
                "gpu_launches": launches, "clocks": clk}
        if e2e:
            line["e2e"] = e2e
        print(json.dumps(line), flush=True)
    st.close()
    dist.destroy_process_group()
