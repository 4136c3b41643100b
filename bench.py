#!/usr/bin/env python
"""Benchmark: phase-space DoF updates/s of the full sLdG run() loop body.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl b200|reference]

One "step" = one run() loop body (core/src/run.cpp:124-131): x half-sweep
(+inline sLdG limiter, + 3-block transfer), charge density, Poisson solve, v
sweep, x half-sweep, nonfinite check, velocity cut-off check (and shrink when
it fires) for BOTH species. value = 2*(nx*p)*(nv*p)*K / device time.

Default workload: C5 (BASELINE.json configs[4]: 16384x16384 cells/species,
k=3, mu=1836, sLdG limiter, cut-off on; 137 GB resident on one B200), the
largest configuration that fits one GPU and the one the metric's 1/2/4/8 GPU
sweep is quoted on. N == 1: the whole state on one B200. N > 1 (torchrun):
the phase space is sharded along v (paper_2408_11235_b200.sharding),
max-over-ranks device time.

--impl reference: the reference itself (oracle/_ref, compiled from
/root/reference) on this host's cores, same metric, timing the same step
window (W warm-up run() loop bodies, then K), on a bounded sample of the
workload when the full shape would not finish in minutes (cpu_sample_cfg).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "phase-space DoF updates/s per step (e+ion)"
UNIT = "DoF/s"
BYTES_PER_DOF_SWEEP = 16.0  # fp64 read + write per directional sweep


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# phase-space DoF of the largest CPU sample: the reference runs a C3-sized
# problem (2.7e8 DoF) at ~5 s per run() loop body on 16 cores, and a full C5
# state would need a ~2 min serial fill plus ~6 min per species for the
# serial cut-off shrink every blob run fires at step 1 (adaptivity.cpp:94-130)
CPU_SAMPLE_DOF = 2.7e8


def cpu_sample_cfg(cfg):
    """The workload the CPU reference times: the config itself when it is at
    most CPU_SAMPLE_DOF, else the same x mesh, k, mu, limiter and cut-off with
    fewer v cells over the same v extent (the per-DoF work of every phase --
    x lines of full length, v lines, serial shrink -- is the same kind; the
    1D Poisson solve is the full one). Returns (cfg, description)."""
    import dataclasses

    if cfg.dof_total <= CPU_SAMPLE_DOF * 1.01:
        return cfg, "the full workload"
    nv = cfg.v_cells
    while nv > 64 and cfg.dof_total * (nv / cfg.v_cells) > CPU_SAMPLE_DOF * 1.01:
        nv //= 2
    sc = dataclasses.replace(cfg, v_cells=nv)
    return sc, (f"a v slab: {cfg.nx}x{nv} cells/species ({cfg.v_cells // nv}x fewer v cells over the "
                f"same v extent, {sc.dof_total:.3g} DoF), x mesh/k/mu/limiter/cut-off as the workload")


def cpu_reference_run(cfg, steps: int, warmup: int, budget_s: float | None):
    """Time the reference (oracle/_ref) on this host over run() loop bodies
    W+1..W+K (budget_s None: exactly K; else until budget_s is spent, at least
    one). Returns (DoF/s of the sample, info)."""
    import oracle

    if not oracle.ref_available():
        raise RuntimeError("oracle/_ref/libsolkin_ref.so not built")
    threads = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    scfg, what = cpu_sample_cfg(cfg)
    t0 = time.perf_counter()
    st = oracle.Ref().state(threads=threads, **scfg.oracle_kwargs())
    t_init = time.perf_counter() - t0
    w = max(warmup, 1)
    st.run(w)
    k, t = 0, 0.0
    while k < max(steps, 1) and (budget_s is None or k == 0 or t < budget_s):
        t += st.run(1)
        k += 1
    rate = scfg.dof_total * k / t
    try:
        mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30
    except (ValueError, OSError):
        mem = float("nan")
    sample = (f"{what}; run() loop bodies {w + 1}..{w + k} after {w} warm-up (init {t_init:.1f}s), "
              f"{threads} threads, {t:.2f}s timed, host RAM {mem:.0f} GiB")
    return rate, dict(threads=threads, steps=k, seconds=t, sample=sample, timers=st.timers(),
                      sample_cfg=scfg)


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the same window as the GPU arm: W warm-up bodies, then exactly K
    rate, info = cpu_reference_run(cfg, args.steps, args.warmup, budget_s=None)
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": info["steps"],
        "warmup": args.warmup, "ms_per_step": 1e3 * info["seconds"] / info["steps"],
        "ms_per_step_note": "wall time per run() loop body of the CPU sample (cpu_baseline.sample)",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (blob initial condition, run.cpp:41-46)", "impl": "reference",
        "config": config_dict(args, cfg),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": info["threads"],
                         "kind": "reference", "sample": info["sample"]},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(args, cfg):
    p = cfg.k + 1
    return {
        "workload": f"{args.config}: {cfg.nx}x{cfg.v_cells} cells/species, k={cfg.k}, "
                    f"mu={cfg.mu:g}, limiter={cfg.limiter}, refinement m={cfg.refinement_ratio}, "
                    f"v cut-off {'on' if cfg.v_adjust else 'off'}",
        "nx": cfg.nx, "nv": cfg.v_cells, "k": cfg.k, "dof_total": cfg.dof_total,
        "field_bytes_per_species": 8 * cfg.nx * p * cfg.v_cells * p,
        "parallelism": f"v-shard x{args.gpus}" if args.gpus > 1 else "single GPU",
        "reductions": "exact (reference order)" if getattr(args, "exact", False)
                      else "parallel (two-pass moment, cyclic-reduction Poisson)",
        "l2": "inputs larger than L2 (no flush needed)"
              if 8 * cfg.dof_total > 126e6 else "state fits in L2 (parity config)",
        **({"stress": "f *= 1 + 0.01 xi, xi ~ U(-1, 1)"} if getattr(args, "stress", False) else {}),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--limiter", default=None)
    ap.add_argument("--refinement", type=int, default=None,
                    help="sheath refinement ratio m of the three-block x mesh (default: the config's)")
    ap.add_argument("--no-cutoff", action="store_true", help="velocity cut-off off (SURVEY.md §8d C5 variant)")
    ap.add_argument("--stress", action="store_true",
                    help="stress variant: f *= 1 + 0.01 xi, xi ~ U(-1, 1) (device hash RNG, seed 20240817)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--exact-steps", type=int, default=4,
                    help="steps of the exact-mode sub-measurement (0: skip)")
    ap.add_argument("--exact", action="store_true",
                    help="exact-reduction (bitwise parity) mode for rho and Poisson")
    args = ap.parse_args()

    import paper_2408_11235_b200 as sk

    over = {"limiter": args.limiter} if args.limiter else {}
    if args.refinement:
        over["refinement_ratio"] = args.refinement
    if args.no_cutoff:
        over["v_adjust"] = False
    cfg = sk.named_config(args.config, **over)

    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        from paper_2408_11235_b200 import sharding

        sharding.bench_sharded(args, cfg, METRIC, UNIT, config_dict(args, cfg))
        return

    import numpy as np
    import torch

    dev = 0
    torch.cuda.set_device(dev)
    st = sk.SimulationState(cfg, device=dev, exact=args.exact)
    st.ctx.set_eager_errors(False)
    fused = st.step_fusion()  # (auto: the C5-class states, sk_ctx_set_step_fusion)
    if args.stress:
        for sp in (0, 1):
            st.field(sp).perturb(20240817 + sp, 0.01)
    st.run_steps(args.warmup)
    st.prepare_steps(args.steps)  # graph captures outside the timed region
    st.ctx.synchronize()

    # ---- timed region: K run() loop bodies (graph replay), CUDA events on the
    # library's stream, which carries exactly the step's work ----
    stream = st.ctx.stream
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = st.launches()
    clocks = ClockSampler(dev)
    clocks.start()
    torch.cuda.synchronize()
    t0.record(stream)
    st.run_steps(args.steps)
    t1.record(stream)
    torch.cuda.synchronize()
    st.ctx.synchronize()  # raises on device-side errors
    launches = st.launches() - launches0
    ms = t0.elapsed_time(t1)
    # ---- second K-step window with per-phase events (eager enqueue): the
    # per-kernel durations behind the roofline ----
    st.set_phase_timing(True)
    st.phase_times()
    torch.cuda.synchronize()
    t0.record(stream)
    st.run_steps(args.steps)
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    st.ctx.synchronize()
    ms_phased = t0.elapsed_time(t1)
    phases = st.phase_times()
    st.set_phase_timing(False)
    value = cfg.dof_total * args.steps / (ms / 1e3)

    # roofline: dominant kernel = longest phase; algorithmic bytes = 16 B per DoF
    # swept (both species) per launch, divided by its mean event-timed duration
    peak, peak_kind = peaks()
    sweep_phases = {"x_sweep_1", "x_sweep_2", "v_sweep"}
    dom = max(phases, key=lambda k: phases[k][0])
    dom_share = phases[dom][0] / ms_phased
    dom_ms, dom_n = phases[dom]
    per_launch_ms = dom_ms / max(dom_n, 1)
    traffic_key = dom
    if dom in sweep_phases or dom.startswith("post"):
        alg_bytes = BYTES_PER_DOF_SWEEP * cfg.dof_total
    else:
        alg_bytes = None
    if fused and dom in ("x_sweep_1", "x_sweep_2"):
        # fused step boundaries (sk_state_step_fusion): a step's two x half sweeps mostly run as ONE
        # pass (xsweep_kernel MODE 3, timed in the x_sweep_2 phase; unfused where the cut-off may
        # check). Both x phases together against the two half sweeps' algorithmic bytes per step
        x_ms = phases["x_sweep_1"][0] + phases["x_sweep_2"][0]
        dom = "x_sweeps (fused step boundaries)"
        dom_share = x_ms / ms_phased
        per_launch_ms = x_ms / max(phases["x_sweep_2"][1], 1)
        alg_bytes = 2 * BYTES_PER_DOF_SWEEP * cfg.dof_total
        traffic_key = "x_sweeps_fused"
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9 if alg_bytes else None
    step_bytes = 3 * BYTES_PER_DOF_SWEEP * cfg.dof_total
    step_gbs = step_bytes * args.steps / (ms / 1e3) / 1e9
    prof_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = None
    try:
        with open(prof_path) as f:
            traffic = json.load(f).get(args.config, {}).get(traffic_key)
    except Exception:
        pass

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (blob initial condition, run.cpp:41-46)",
        "config": config_dict(args, cfg),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "alg_bytes_per_launch": alg_bytes, "ms_per_launch": per_launch_ms,
                     "share_of_step": dom_share, "fused_step_boundaries": fused,
                     "step_achieved_gbs": step_gbs, "step_frac": step_gbs / peak,
                     "timing": "kernel ms from per-phase CUDA events over a second K-step "
                               "window (eager enqueue, %.3f ms/step vs %.3f graphed)"
                               % (ms_phased / args.steps, ms / args.steps)},
        "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items() if v[1]},
        "gpu_launches": launches,
        "limiter_stats": st.stats(),
        "clocks": clk,
    }

    # ---- exact (bitwise-parity) mode on the same state: the reference's
    # serial charge-density order and dpbtrs chain on the device ----
    if not args.exact and args.exact_steps > 0:
        st.ctx.set_exact_reductions(True)
        st.run_steps(2)  # capture
        torch.cuda.synchronize()
        t0.record(stream)
        st.run_steps(args.exact_steps)
        t1.record(stream)
        torch.cuda.synchronize()
        st.ctx.synchronize()
        ems = t0.elapsed_time(t1) / args.exact_steps
        st.ctx.set_exact_reductions(False)
        line["exact_mode"] = {"ms_per_step": ems, "value": cfg.dof_total / (ems / 1e3), "unit": UNIT,
                              "steps": args.exact_steps,
                              "what": "the same run() loop body with sk_ctx_set_exact_reductions(1): "
                                      "trajectory bitwise the reference's (tests/test_gpu_parity.py)"}

    # ---- e2e: the drop-in C-ABI call over pinned HOST buffers ----
    if not args.no_e2e:
        n = st.f_e.size
        fe = torch.empty(n, dtype=torch.float64, pin_memory=True)
        fi = torch.empty(n, dtype=torch.float64, pin_memory=True)
        fe_np, fi_np = fe.numpy(), fi.numpy()
        fe_np[:] = st.f_e.download()
        fi_np[:] = st.f_i.download()
        st.run_step_host(fe_np, fi_np)  # warm-up
        k2 = args.e2e_steps
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        st.run_steps_host(k2, fe_np, fi_np)  # every step: both species up, both results down
        w = time.perf_counter() - w0
        line["e2e"] = {"value": cfg.dof_total * k2 / w, "unit": UNIT,
                       "h2d_bytes_per_step": 2 * 8 * n, "d2h_bytes_per_step": 2 * 8 * n,
                       "steps": k2, "api": "sk_run_steps_host (include/sk_b200.h): host copies of "
                                           "consecutive steps pipelined over full-duplex PCIe"}
        del fe, fi

    # ---- CPU baseline: the reference on this host, bounded sample ----
    if not args.no_cpu:
        try:
            rate, info = cpu_reference_run(cfg, 50, 1, budget_s=args.cpu_budget)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": info["threads"],
                                    "kind": "reference", "sample": info["sample"]}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"not run: {e}"}
    print(json.dumps(line), flush=True)
    del np


if __name__ == "__main__":
    main()
