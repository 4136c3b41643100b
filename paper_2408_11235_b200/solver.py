"""Host-side mirror of the reference solver interface (proj/core) over the C ABI.

Names, argument meaning and error behaviour follow the reference's free
functions so parity tests read like the reference's own:

  reference (core/include/solkin/*.hpp)            here
  -----------------------------------------------  ------------------------------
  Grid1D::three_block / uniform (grid.hpp:22-25)   Grid1D.three_block / uniform
  NodalField (field.hpp:21-80)                     NodalField (device resident)
  LimiterConfig::parse (limiters.hpp:19-34)        LimiterConfig.parse
  advect_x / advect_v (advection.hpp:83-88)        advect_x / advect_v
  apply_post_limiter (limiters.hpp:107-108)        apply_post_limiter
  charge_density (poisson.hpp:61)                  charge_density
  PoissonOperator::solve (poisson.hpp:28)          PoissonOperator.solve
  check_velocity_shrink / shrink_velocity_domain   same names
  build_initial_state / strang_step / run() body   SimulationState, strang_step, run_step
  std::runtime_error / SimulationError             RuntimeError / SimulationError

Device memory for E / rho buffers is torch (plumbing only); all arithmetic is in
libsk_b200.so. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import runconfig as RC


class SimulationError(RuntimeError):
    """solkin::SimulationError (common.hpp:16-20): carries the step index."""

    def __init__(self, step: int, msg: str):
        super().__init__(msg)
        self.step = step


def _check(rc: int) -> None:
    if rc == N.SK_OK:
        return
    L = N.lib()
    msg = L.sk_last_error().decode()
    if rc == N.SK_ERR_SIMULATION:
        raise SimulationError(L.sk_last_error_step(), msg)
    raise RuntimeError(msg)


def _dptr(x) -> int:
    """device pointer of a torch CUDA tensor (float64, contiguous)."""
    import torch

    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64
            and x.is_contiguous()):
        raise TypeError("expected a contiguous float64 CUDA tensor")
    return x.data_ptr()


# ----------------------------------------------------------------------------
# configuration mirrors
# ----------------------------------------------------------------------------
@dataclass
class LimiterConfig:
    """limiters.hpp:19-34"""

    indicator: int = 0       # 0 none, 1 minmod, 2 meanerr
    modifier: int = 0        # 0 none, 1 simple WENO, 2 line WENO
    inline_sldg: bool = False
    threshold: float = 0.5
    gamma_simple: tuple = (0.001, 0.998, 0.001)
    gamma_line: tuple = (0.45, 0.1, 0.45)
    epsilon: float = 1e-6

    MODES = ("none", "minmod+simple", "minmod+line", "meanerr+simple", "meanerr+line", "sldg")

    @staticmethod
    def parse(mode: str) -> "LimiterConfig":
        """limiters.cpp:14-37"""
        cfg = LimiterConfig()
        if mode == "none":
            return cfg
        if mode == "sldg":
            cfg.inline_sldg = True
            return cfg
        if "+" not in mode:
            raise RuntimeError("unknown limiter mode: " + mode)
        ind, mod = mode.split("+", 1)
        if ind == "minmod":
            cfg.indicator = 1
        elif ind == "meanerr":
            cfg.indicator = 2
        else:
            raise RuntimeError("unknown limiter indicator: " + ind)
        if mod == "simple":
            cfg.modifier = 1
        elif mod == "line":
            cfg.modifier = 2
        else:
            raise RuntimeError("unknown limiter modifier: " + mod)
        return cfg

    def mode_string(self) -> str:
        if self.inline_sldg:
            return "sldg"
        if self.indicator == 0:
            return "none"
        return ("minmod" if self.indicator == 1 else "meanerr") + (
            "+simple" if self.modifier == 1 else "+line")

    def post_enabled(self) -> bool:
        return self.indicator != 0

    def to_c(self) -> N.sk_limiter:
        c = N.sk_limiter()
        c.indicator, c.modifier, c.inline_sldg = self.indicator, self.modifier, int(self.inline_sldg)
        c.threshold = self.threshold
        for i in range(3):
            c.gamma_simple[i] = self.gamma_simple[i]
            c.gamma_line[i] = self.gamma_line[i]
        c.epsilon = self.epsilon
        return c


@dataclass
class VAdjustPolicy:
    """adaptivity.hpp:13-19"""

    p: float = 0.05
    gamma: float = 0.05
    tol: float = 1e-14

    def to_c(self) -> N.sk_vadjust:
        return N.sk_vadjust(self.p, self.gamma, self.tol)


@dataclass
class SpeciesParams:
    """advection.hpp:64-70"""

    charge_sign: float = -1.0
    sqrt_mu: float = 1.0

    @staticmethod
    def electron() -> "SpeciesParams":
        return SpeciesParams(-1.0, 1.0)

    @staticmethod
    def ion(mu: float) -> "SpeciesParams":
        if not mu > 0:
            raise RuntimeError("SpeciesParams::ion: mass ratio must be positive")
        return SpeciesParams(1.0, math.sqrt(mu))


@dataclass
class RunConfig:
    """RunConfig (config.hpp:11-59): keys, defaults, presets, key = value files,
    validation and echo as the reference (config.cpp:58-221)."""

    scenario: str = "blob"
    t0: float = 2000.0  # injection source window (config.hpp:18)
    L: float = 200.0
    dt: float = 0.1
    k: int = 3
    mu: float = 400.0
    t_final: float = 400.0
    sigma: float = -1.0
    vmax_e: float = 12.0
    vmax_i: float = 12.0
    fine_block_cells: int = 50
    coarse_block_cells: int = 50
    refinement_ratio: int = 1
    v_cells: int = 40
    limiter: str = "none"
    limiter_threshold: float = 0.5
    v_adjust: bool = True
    adapt_p: float = 0.05
    adapt_gamma: float = 0.05
    adapt_tol: float = 1e-14
    penalty_scale: float = 10.0
    out_dir: str = "out"
    cadence: int = 10           # flux row every N steps
    snapshot_cadence: int = 0   # 0 = off
    profile_cadence: int = 0    # 0 = off
    threads: int = 1            # accepted for parity; the device ignores it

    # (key, attribute, kind) in echo order (config.cpp:111-137, 196-224)
    KEYS = (("scenario", "scenario", "s"), ("L", "L", "d"), ("dt", "dt", "d"), ("k", "k", "i"),
            ("mu", "mu", "d"), ("t_final", "t_final", "d"), ("sigma", "sigma", "d"),
            ("t0", "t0", "d"), ("vmax_e", "vmax_e", "d"), ("vmax_i", "vmax_i", "d"),
            ("mesh.fine_block_cells", "fine_block_cells", "i"),
            ("mesh.coarse_block_cells", "coarse_block_cells", "i"),
            ("mesh.refinement_ratio", "refinement_ratio", "i"), ("v_cells", "v_cells", "i"),
            ("limiter", "limiter", "s"), ("limiter.threshold", "limiter_threshold", "d"),
            ("adaptivity.v_adjust", "v_adjust", "b"), ("adaptivity.p", "adapt_p", "d"),
            ("adaptivity.gamma", "adapt_gamma", "d"), ("adaptivity.tol", "adapt_tol", "d"),
            ("poisson.penalty_scale", "penalty_scale", "d"), ("output.dir", "out_dir", "s"),
            ("output.cadence", "cadence", "i"), ("output.snapshot_cadence", "snapshot_cadence", "i"),
            ("output.profile_cadence", "profile_cadence", "i"), ("threads", "threads", "i"))
    # name -> (scenario, fine, coarse, m, v_cells or None to keep the defaults, t_final)
    PRESETS = {"blob-desk": ("blob", None, 400.0), "injection-desk": ("injection", None, 400.0),
               "blob-paper": ("blob", (100, 100, 1, 150), 4000.0),
               "injection-paper": ("injection", (100, 100, 8, 150), 8000.0)}

    @staticmethod
    def preset(name: str) -> "RunConfig":
        """config.cpp:58-86"""
        if name not in RunConfig.PRESETS:
            raise RuntimeError(f"unknown preset '{name}' (expected blob-paper, injection-paper, "
                               "blob-desk, injection-desk)")
        scenario, mesh, t_final = RunConfig.PRESETS[name]
        c = RunConfig(scenario=scenario, t_final=t_final)
        if mesh:
            c.fine_block_cells, c.coarse_block_cells, c.refinement_ratio, c.v_cells = mesh
        return c

    @staticmethod
    def from_file(path: str) -> "RunConfig":
        c = RunConfig()
        c.apply_file(path)
        return c

    def apply_file(self, path: str) -> None:
        """flat key = value lines with '#' comments (config.cpp:93-109)"""
        try:
            with open(path, "rb") as fh:
                data = fh.read().decode("utf-8", "surrogateescape")
        except OSError:
            raise RuntimeError(f"cannot read config file '{path}'") from None
        for lineno, line in enumerate(data.split("\n")[: data.count("\n") + (not data.endswith("\n"))], 1):
            line = RC.trim(line.split("#", 1)[0])
            if not line:
                continue
            if "=" not in line:
                raise RuntimeError(f"{path}:{lineno}: expected key = value")
            key, value = line.split("=", 1)
            self.apply_kv(RC.trim(key), RC.trim(value))

    def apply_kv(self, key: str, value: str) -> None:
        """config.cpp:111-138"""
        for name, attr, kind in self.KEYS:
            if name != key:
                continue
            if kind == "d":
                setattr(self, attr, RC.stod_full(key, value))
            elif kind == "i":
                setattr(self, attr, RC.stoi_full(key, value))
            elif kind == "b":
                setattr(self, attr, RC.onoff(key, value))
            else:
                setattr(self, attr, value)
            return
        raise RuntimeError(f"unknown config key '{key}'")

    def resolve(self) -> None:
        """sigma < 0 -> 0.1 L (config.cpp:140-142)"""
        if self.sigma < 0:
            self.sigma = 0.1 * self.L

    def violations(self) -> list:
        """'key: message' lines in the reference's order (config.cpp:144-185)"""
        out = []

        def need(ok, key, msg):
            if not ok:
                out.append(f"{key}: {msg}")

        need(self.scenario in ("blob", "injection"), "scenario", "must be blob or injection")
        need(self.L > 0, "L", "must be positive")
        need(self.dt > 0, "dt", "must be positive")
        need(0 <= self.k <= 6, "k", "must be in 0..6")
        need(self.mu > 0, "mu", "must be positive")
        need(not self.t_final < 0, "t_final", "must be >= 0")
        need(self.sigma > 0, "sigma", "must be positive (call resolve() to default to 0.1*L)")
        need(self.t0 > 0, "t0", "must be positive")
        need(self.vmax_e > 0, "vmax_e", "must be positive")
        need(self.vmax_i > 0, "vmax_i", "must be positive")
        need(self.fine_block_cells >= 1, "mesh.fine_block_cells", "must be >= 1")
        need(self.coarse_block_cells >= 1, "mesh.coarse_block_cells", "must be >= 1")
        need(self.refinement_ratio >= 1, "mesh.refinement_ratio", "must be >= 1")
        need(self.v_cells >= 1, "v_cells", "must be >= 1")
        try:
            LimiterConfig.parse(self.limiter)
            ok = True
        except RuntimeError:
            ok = False
        need(ok, "limiter", "must be one of " + ", ".join(LimiterConfig.MODES))
        need(self.limiter_threshold > 0, "limiter.threshold", "must be positive")
        need(self.adapt_p > 0 and not self.adapt_gamma < 0 and not self.adapt_p + self.adapt_gamma >= 1,
             "adaptivity.p/gamma", "need 0 < p, 0 <= gamma, p + gamma < 1")
        need(self.adapt_tol > 0, "adaptivity.tol", "must be positive")
        need(self.penalty_scale > 0, "poisson.penalty_scale", "must be positive")
        need(self.cadence >= 1, "output.cadence", "must be >= 1")
        need(self.snapshot_cadence >= 0, "output.snapshot_cadence", "must be >= 0")
        need(self.profile_cadence >= 0, "output.profile_cadence", "must be >= 0")
        need(self.threads >= 1, "threads", "must be >= 1")
        return out

    def validate(self) -> None:
        v = self.violations()
        if v:
            raise RuntimeError("invalid configuration:" + "".join("\n  " + s for s in v))

    def echo(self) -> str:
        """re-ingestible key = value echo (config.cpp:187-218)"""
        fmt = {"d": RC.g17, "i": str, "b": lambda b: "on" if b else "off", "s": str}
        return "".join(f"{name} = {fmt[kind](getattr(self, attr))}\n" for name, attr, kind in self.KEYS)

    def nsteps(self) -> int:
        """std::lround(t_final / dt) (config.cpp:220)"""
        return RC.lround(self.t_final / self.dt)

    @property
    def nx(self) -> int:
        return 2 * self.fine_block_cells + self.coarse_block_cells

    @property
    def dof_total(self) -> int:
        """phase-space DoF of both species: 2*(nx*p)*(nv*p)"""
        p = self.k + 1
        return 2 * self.nx * p * self.v_cells * p

    def oracle_kwargs(self) -> dict:
        return dict(L=self.L, dt=self.dt, k=self.k, mu=self.mu, sigma=self.sigma,
                    vmax_e=self.vmax_e, vmax_i=self.vmax_i, nf=self.fine_block_cells,
                    nc=self.coarse_block_cells, m=self.refinement_ratio, nv=self.v_cells,
                    limiter=self.limiter, limiter_threshold=self.limiter_threshold,
                    v_adjust=int(self.v_adjust), adapt_p=self.adapt_p,
                    adapt_gamma=self.adapt_gamma, adapt_tol=self.adapt_tol,
                    penalty_scale=self.penalty_scale, scenario=self.scenario, t0=self.t0)

    def to_c(self) -> N.sk_run_config:
        if self.scenario not in ("blob", "injection"):
            raise RuntimeError("RunConfig: scenario must be blob or injection")
        lim = LimiterConfig.parse(self.limiter)
        lim.threshold = self.limiter_threshold
        c = N.sk_run_config()
        c.L, c.dt, c.mu, c.sigma = self.L, self.dt, self.mu, self.sigma
        c.vmax_e, c.vmax_i, c.k = self.vmax_e, self.vmax_i, self.k
        c.fine_block_cells, c.coarse_block_cells = self.fine_block_cells, self.coarse_block_cells
        c.refinement_ratio, c.v_cells = self.refinement_ratio, self.v_cells
        c.limiter = lim.to_c()
        c.v_adjust = int(self.v_adjust)
        c.policy = N.sk_vadjust(self.adapt_p, self.adapt_gamma, self.adapt_tol)
        c.penalty_scale = self.penalty_scale
        c.scenario = 1 if self.scenario == "injection" else 0
        c.t0 = self.t0
        return c


# SURVEY.md §8(d) config shapes (BASELINE.json configs[0..4]).
NAMED_CONFIGS = {
    "C1": RunConfig(k=2, fine_block_cells=32, coarse_block_cells=64, refinement_ratio=1,
                    v_cells=128, limiter="none"),
    "C2": RunConfig(k=2, fine_block_cells=128, coarse_block_cells=256, refinement_ratio=8,
                    v_cells=512, limiter="sldg"),
    "C3": RunConfig(k=3, mu=1836.0, fine_block_cells=512, coarse_block_cells=1024,
                    refinement_ratio=1, v_cells=4096, limiter="sldg"),
    "C5": RunConfig(k=3, mu=1836.0, fine_block_cells=4096, coarse_block_cells=8192,
                    refinement_ratio=1, v_cells=16384, limiter="sldg"),
    "C5k2": RunConfig(k=2, mu=1836.0, fine_block_cells=4096, coarse_block_cells=8192,
                      refinement_ratio=1, v_cells=16384, limiter="sldg"),
}


def named_config(name: str, **overrides) -> RunConfig:
    import dataclasses

    return dataclasses.replace(NAMED_CONFIGS[name], **overrides)


# ----------------------------------------------------------------------------
# grid / context / field
# ----------------------------------------------------------------------------
@dataclass
class Grid1D:
    """grid.hpp:18-49 (block list)."""

    left: list = field(default_factory=list)
    cells: list = field(default_factory=list)
    dx: list = field(default_factory=list)

    @staticmethod
    def uniform(left: float, right: float, cells: int) -> "Grid1D":
        if not (right > left and cells >= 1):
            raise RuntimeError("Grid1D::uniform: invalid extent or cell count")
        return Grid1D([left], [cells], [(right - left) / cells])

    @staticmethod
    def three_block(left, right, fine_cells, coarse_cells, m) -> "Grid1D":
        bl = (C.c_double * 3)()
        bc = (C.c_int * 3)()
        bd = (C.c_double * 3)()
        _check(N.lib().sk_grid_three_block(left, right, fine_cells, coarse_cells, m, bl, bc, bd))
        return Grid1D(list(bl), list(bc), list(bd))

    @property
    def ncells(self) -> int:
        return int(sum(self.cells))

    def right(self) -> float:
        return self.left[-1] + self.cells[-1] * self.dx[-1]


class Context:
    """One GPU: x grid, degree k, the Poisson operator (factorised once)."""

    def __init__(self, grid: Grid1D, k: int, penalty_scale: float = 10.0, device: int = 0,
                 use_torch_stream: bool = True):
        L = N.lib()
        nb = len(grid.cells)
        h = C.c_void_p()
        _check(L.sk_ctx_create(device, k, nb, (C.c_double * nb)(*grid.left),
                               (C.c_int * nb)(*grid.cells), (C.c_double * nb)(*grid.dx),
                               penalty_scale, C.byref(h)))
        self.h = h
        self.grid, self.k, self.p, self.device = grid, k, k + 1, device
        self.nx = grid.ncells
        self.stream = None
        if use_torch_stream:
            # the library runs on a dedicated (non-default, capturable) torch
            # stream; fence() orders it against torch's current stream
            import torch

            torch.cuda.set_device(device)
            self.stream = torch.cuda.Stream(device=device)
            _check(L.sk_ctx_set_stream(h, C.c_void_p(self.stream.cuda_stream)))

    def enter(self):
        """library work must see torch work already queued on the current stream"""
        if self.stream is not None:
            import torch

            self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def leave(self):
        """torch work queued after this point must see the library's results"""
        if self.stream is not None:
            import torch

            torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def close(self):
        if getattr(self, "h", None):
            N.lib().sk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_eager_errors(self, on: bool):
        _check(N.lib().sk_ctx_set_eager_errors(self.h, int(on)))

    def set_exact_reductions(self, on: bool):
        """exact (parity) mode: reference rounding sequence in the sweeps (no FMA),
        reference-order charge density, sequential dpbtrs solve"""
        _check(N.lib().sk_ctx_set_exact_reductions(self.h, int(on)))

    EXACT_ARITH, EXACT_RHO, EXACT_POISSON = 1, 2, 4

    def set_exact_parts(self, mask: int):
        """exact mode per part (OR of EXACT_ARITH / EXACT_RHO / EXACT_POISSON),
        to attribute a fast-mode deviation to one of them"""
        _check(N.lib().sk_ctx_set_exact_parts(self.h, int(mask)))

    def check_guards(self) -> int:
        """guard words overwritten around the state buffers (needs SK_GUARD=1)"""
        bad = C.c_longlong()
        _check(N.lib().sk_ctx_check_guards(self.h, C.byref(bad)))
        return bad.value

    def set_step_fusion(self, on):
        """fuse step n's second and step n+1's first x half sweep in run_steps
        (True / False; None: auto, the default -- fused for states >= 2^32 DoF)"""
        _check(N.lib().sk_ctx_set_step_fusion(self.h, -1 if on is None else int(bool(on))))

    def set_post_fusion(self, on: bool):
        """decide the post limiter V's flags inside the v sweep (default on)"""
        _check(N.lib().sk_ctx_set_post_fusion(self.h, int(on)))

    def synchronize(self):
        _check(N.lib().sk_ctx_synchronize(self.h))

    def stats(self) -> dict:
        s = N.sk_stats()
        _check(N.lib().sk_stats_get(self.h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in N.sk_stats._fields_}

    def reset_stats(self):
        _check(N.lib().sk_stats_reset(self.h))

    def dev_zeros(self, n: int):
        import torch

        return torch.zeros(n, dtype=torch.float64, device=f"cuda:{self.device}")


class NodalField:
    """NodalField on the device (field.hpp:21-80), reference layout."""

    def __init__(self, ctx: Context, species: int, v: Grid1D, _handle=None, _owner=None):
        self.ctx, self.species = ctx, species
        self._owner = _owner
        if _handle is not None:
            self.h = _handle
            self._owns = False
        else:
            if len(v.cells) != 1:
                raise RuntimeError("NodalField: v grid must be a single uniform block")
            h = C.c_void_p()
            _check(N.lib().sk_field_create(ctx.h, species, v.left[0], v.right(), v.cells[0],
                                           C.byref(h)))
            self.h = h
            self._owns = True
        self.nv = self.size // (ctx.p * ctx.nx * ctx.p)  # cells held (a v shard may hold fewer)

    def close(self):
        if self._owns and getattr(self, "h", None):
            N.lib().sk_field_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def size(self) -> int:
        return int(N.lib().sk_field_size(self.h))

    @property
    def shape(self):
        p = self.ctx.p
        return (self.nv, p, self.ctx.nx, p)

    def data_ptr(self) -> int:
        return N.lib().sk_field_data_dev(self.h)

    def v_grid(self):
        left, dx, cells = C.c_double(), C.c_double(), C.c_int()
        _check(N.lib().sk_field_v_grid(self.h, C.byref(left), C.byref(dx), C.byref(cells)))
        return left.value, dx.value, cells.value

    def vmax(self) -> float:
        left, dx, cells = self.v_grid()
        return left + cells * dx  # Grid1D::right (grid.cpp:48-51)

    def upload(self, data: np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.float64).ravel()
        _check(N.lib().sk_field_upload(self.h, a.ctypes.data_as(C.POINTER(C.c_double)), a.size))

    def download_2d(self, offset: int, width: int, height: int, pitch: int) -> np.ndarray:
        """height runs of width doubles, pitch apart, from element offset (an x
        line: width = nx*p; a v line: width 1, pitch nx*p) -> [height, width]"""
        out = np.empty((height, width))
        _check(N.lib().sk_field_download_2d(self.h, out.ctypes.data_as(C.POINTER(C.c_double)), offset, width,
                                            height, pitch))
        return out

    def download(self) -> np.ndarray:
        out = np.empty(self.size)
        _check(N.lib().sk_field_download(self.h, out.ctypes.data_as(C.POINTER(C.c_double)),
                                         out.size))
        return out

    def perturb(self, seed: int = 20240817, amp: float = 0.01):
        """benchmark stress variant: f *= 1 + amp * xi, xi uniform in [-1, 1) (device hash RNG)"""
        _check(N.lib().sk_field_perturb(self.h, int(seed), float(amp)))

    def fill_blob(self, sigma: float):
        _check(N.lib().sk_field_fill_blob(self.h, sigma))

    def moments(self) -> dict:
        out = (C.c_double * 4)()
        _check(N.lib().sk_field_moments(self.h, out))
        return dict(mass=out[0], l2=out[1], momentum=out[2], kinetic=out[3])

    def mass(self) -> float:
        return self.moments()["mass"]

    def l2_norm(self) -> float:
        return self.moments()["l2"]


@dataclass
class SweepOptions:
    """advection.hpp:72-79"""

    bc: int = 0  # 0 ZeroInflow, 1 Periodic
    limiter: LimiterConfig = field(default_factory=LimiterConfig)
    max_ghost: int = -1
    step_index: int = 0


def advect_x(f: NodalField, tau: float, sp: SpeciesParams, opt: SweepOptions = SweepOptions()):
    """advect_x (advection.cpp:144-207)"""
    lim = opt.limiter.to_c()
    _check(N.lib().sk_advect_x(f.h, tau, sp.sqrt_mu, opt.bc, C.byref(lim), opt.max_ghost,
                               opt.step_index))


def _device_array(ctx: Context, a):
    import torch

    if isinstance(a, torch.Tensor):
        return a
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64),
                           device=f"cuda:{ctx.device}")


def advect_v(f: NodalField, tau: float, E_nodes, sp: SpeciesParams,
             opt: SweepOptions = SweepOptions()):
    """advect_v (advection.cpp:209-238); E_nodes: nx*(k+1) values (numpy or CUDA tensor)."""
    E = _device_array(f.ctx, E_nodes)
    if E.numel() != f.ctx.nx * f.ctx.p:
        raise RuntimeError("advect_v: E node array size mismatch")
    lim = opt.limiter.to_c()
    f.ctx.enter()
    _check(N.lib().sk_advect_v(f.h, tau, C.c_void_p(_dptr(E)), sp.charge_sign, sp.sqrt_mu, opt.bc,
                               C.byref(lim)))
    f.ctx.leave()


def apply_post_limiter(f: NodalField, direction: int, cfg: LimiterConfig, bc: int = 0):
    """apply_post_limiter (limiters.cpp:280-345); direction 0 = X, 1 = V."""
    lim = cfg.to_c()
    _check(N.lib().sk_post_limit(f.h, direction, C.byref(lim), bc))


def charge_density(fe: NodalField, fi: NodalField, out=None):
    """charge_density (poisson.cpp:194-216) -> CUDA tensor nx*(k+1)."""
    rho = out if out is not None else fe.ctx.dev_zeros(fe.ctx.nx * fe.ctx.p)
    fe.ctx.enter()
    _check(N.lib().sk_charge_density(fe.h, fi.h, C.c_void_p(_dptr(rho))))
    fe.ctx.leave()
    return rho


@dataclass
class FieldPair:
    E: object
    phi: object


class PoissonOperator:
    """PoissonOperator (poisson.hpp:24-57): assembled + reduced in the Context."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def solve(self, rho) -> FieldPair:
        rho = _device_array(self.ctx, rho)
        E = self.ctx.dev_zeros(self.ctx.nx * self.ctx.p)
        phi = self.ctx.dev_zeros(self.ctx.nx * (self.ctx.p + 1))
        self.ctx.enter()
        _check(N.lib().sk_poisson_solve(self.ctx.h, C.c_void_p(_dptr(rho)), C.c_void_p(_dptr(E)),
                                        C.c_void_p(_dptr(phi))))
        self.ctx.leave()
        return FieldPair(E, phi)


def check_velocity_shrink(f: NodalField, policy: VAdjustPolicy = VAdjustPolicy()) -> bool:
    """check_velocity_shrink (adaptivity.cpp:16-38)"""
    pol = policy.to_c()
    out = C.c_int()
    _check(N.lib().sk_check_velocity_shrink(f.h, C.byref(pol), C.byref(out)))
    return bool(out.value)


def shrink_velocity_domain(f: NodalField, policy: VAdjustPolicy = VAdjustPolicy()) -> dict:
    """shrink_velocity_domain (adaptivity.cpp:94-130) -> ShrinkResult fields"""
    pol = policy.to_c()
    r = N.sk_shrink_result()
    _check(N.lib().sk_shrink_velocity_domain(f.h, C.byref(pol), C.byref(r)))
    return dict(vmax_before=r.vmax_before, vmax_after=r.vmax_after,
                mass_before=r.mass_before, mass_after=r.mass_after)


def electric_energy(ctx: Context, E) -> float:
    out = C.c_double()
    ctx.enter()
    _check(N.lib().sk_electric_energy(ctx.h, C.c_void_p(_dptr(E)), C.byref(out)))
    return out.value


# ----------------------------------------------------------------------------
# state + step
# ----------------------------------------------------------------------------
class SimulationState:
    """build_initial_state (run.cpp:26-58) on the device; the step API of
    stepper.cpp:44-103 and the run() loop body of run.cpp:124-131."""

    def __init__(self, cfg: RunConfig, device: int = 0, ctx: Context | None = None,
                 exact: bool = False):
        self.cfg = cfg
        if ctx is None:
            grid = Grid1D.three_block(-cfg.L, cfg.L, cfg.fine_block_cells, cfg.coarse_block_cells,
                                      cfg.refinement_ratio)
            ctx = Context(grid, cfg.k, cfg.penalty_scale, device)
        if exact is True:
            ctx.set_exact_reductions(True)
        elif exact:  # a mask of Context.EXACT_* parts
            ctx.set_exact_parts(int(exact))
        self.ctx = ctx
        h = C.c_void_p()
        ccfg = cfg.to_c()
        _check(N.lib().sk_state_create(ctx.h, C.byref(ccfg), C.byref(h)))
        self.h = h
        L = N.lib()
        self.f_e = NodalField(ctx, 0, None, _handle=L.sk_state_field(h, 0), _owner=self)
        self.f_i = NodalField(ctx, 1, None, _handle=L.sk_state_field(h, 1), _owner=self)
        self.steps_enqueued = 0

    def close(self):
        if getattr(self, "h", None):
            N.lib().sk_state_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def field(self, species: int) -> NodalField:
        return self.f_e if species == 0 else self.f_i

    def E_ptr(self) -> int:
        return N.lib().sk_state_E_dev(self.h)

    def rho(self) -> np.ndarray:
        """the charge density of the last step (the Poisson right-hand side)"""
        out = np.empty(self.ctx.nx * self.ctx.p)
        _check(N.lib().sk_state_download_rho(self.h, out.ctypes.data_as(C.POINTER(C.c_double)), out.size))
        return out

    def E(self) -> np.ndarray:
        """state.field.E (stepper.hpp:48) downloaded to the host."""
        out = np.empty(self.ctx.nx * self.ctx.p)
        _check(N.lib().sk_state_download_E(self.h, out.ctypes.data_as(C.POINTER(C.c_double)),
                                           out.size))
        return out

    def strang_step(self):
        _check(N.lib().sk_strang_step(self.h))
        self.steps_enqueued += 1

    def run_step(self):
        _check(N.lib().sk_run_step(self.h))
        self.steps_enqueued += 1

    def run_steps(self, n: int):
        _check(N.lib().sk_run_steps(self.h, n))
        self.steps_enqueued += n

    def prepare_steps(self, n: int):
        """capture the graphs run_steps(n) will replay (no work is run)"""
        _check(N.lib().sk_state_prepare_steps(self.h, n))

    def run_step_host(self, fe: np.ndarray, fi: np.ndarray):
        """drop-in strang_step + shrink over host arrays (updated in place)."""
        pd = C.POINTER(C.c_double)
        _check(N.lib().sk_run_step_host(self.h, fe.ctypes.data_as(pd), fi.ctypes.data_as(pd),
                                        fe.size))
        self.steps_enqueued += 1

    def run_steps_host(self, n: int, fe: np.ndarray, fi: np.ndarray):
        """n drop-in steps over host arrays (updated in place), copies pipelined across steps."""
        pd = C.POINTER(C.c_double)
        _check(N.lib().sk_run_steps_host(self.h, int(n), fe.ctypes.data_as(pd), fi.ctypes.data_as(pd),
                                         fe.size))
        self.steps_enqueued += n

    def set_phase_timing(self, on: bool):
        _check(N.lib().sk_state_set_phase_timing(self.h, int(on)))

    def phase_times(self) -> dict:
        """accumulated ms per phase since the last call (CUDA events on the step stream)"""
        n = len(N.PHASES)
        ms = (C.c_double * n)()
        cnt = (C.c_long * n)()
        _check(N.lib().sk_state_phase_times(self.h, ms, cnt, n))
        return {name: (ms[i], cnt[i]) for i, name in enumerate(N.PHASES)}

    def launches(self) -> int:
        return int(N.lib().sk_ctx_launch_count(self.ctx.h))

    def step_fusion(self) -> bool:
        """whether run_steps fuses this state's step boundaries"""
        on = C.c_int()
        _check(N.lib().sk_state_step_fusion(self.h, C.byref(on)))
        return bool(on.value)

    def step_index(self) -> int:
        s = C.c_long()
        _check(N.lib().sk_state_step_index(self.h, C.byref(s)))
        return s.value

    def shrinks(self, species: int):
        cnt, last = C.c_int(), C.c_long()
        _check(N.lib().sk_state_shrinks(self.h, species, C.byref(cnt), C.byref(last)))
        return cnt.value, last.value

    # ---- diagnostics + output (diagnostics.cpp) ----
    def time(self) -> float:
        """state.time (stepper.cpp:98)"""
        t = C.c_double()
        _check(N.lib().sk_state_time(self.h, C.byref(t)))
        return t.value

    def wall_flux(self, species: int, side: int) -> tuple:
        """wall_flux (diagnostics.cpp:24-69): (outflow, naive); side 0 left, 1 right"""
        o, n = C.c_double(), C.c_double()
        _check(N.lib().sk_state_wall_flux(self.h, species, side, C.byref(o), C.byref(n)))
        return o.value, n.value

    def sample_fluxes(self) -> dict:
        """sample_fluxes (diagnostics.cpp:98-116)"""
        out = N.sk_flux_sample()
        _check(N.lib().sk_state_sample_fluxes(self.h, C.byref(out)))
        return {k: getattr(out, k) for k, _ in out._fields_}

    def summarize(self) -> dict:
        """summarize (diagnostics.cpp:85-96)"""
        out = N.sk_summary()
        _check(N.lib().sk_state_summarize(self.h, C.byref(out)))
        return {k: getattr(out, k) for k, _ in out._fields_}

    def write_snapshot(self, directory: str):
        """OutputWriter::write_snapshot: <dir>/snapshot_<step>.bin (SOLKSNP1) + .meta"""
        _check(N.lib().sk_state_write_snapshot(self.h, str(directory).encode()))

    def write_profiles(self, directory: str):
        """OutputWriter::write_profiles: <dir>/profiles_<step>.csv"""
        _check(N.lib().sk_state_write_profiles(self.h, str(directory).encode()))

    def stats(self) -> dict:
        s = self.ctx.stats()
        p = self.ctx.p
        s["outputs"] = self.steps_enqueued * 2 * 3 * self.ctx.nx * self.cfg.v_cells * p
        return s

    def summary(self) -> dict:
        me, mi = self.f_e.moments(), self.f_i.moments()
        import torch

        E = torch.as_tensor(self.E(), device=f"cuda:{self.ctx.device}")
        return dict(mass_e=me["mass"], mass_i=mi["mass"], l2_e=me["l2"], l2_i=mi["l2"],
                    e_energy=electric_energy(self.ctx, E), vmax_e=self.f_e.vmax(),
                    vmax_i=self.f_i.vmax(), mom_e=me["momentum"], mom_i=mi["momentum"],
                    ekin_e=me["kinetic"], ekin_i=mi["kinetic"])


def strang_step(state: SimulationState):
    state.strang_step()


def run_step(state: SimulationState):
    state.run_step()


_FROM_CFG = object()


def run(cfg: RunConfig, nsteps: int | None = None, cadence: int | None = None,
        snapshot_cadence: int | None = None, profile_cadence: int | None = None,
        out_dir=_FROM_CFG, device: int = 0, exact: bool = False) -> dict:
    """run() (run.cpp:60-169): nsteps (default cfg.nsteps(), config.cpp:220) run()
    loop bodies with flux.csv rows every `cadence` steps, snapshots / profiles
    at their cadences, run.log -- into out_dir (None: no files). Cadences and
    out_dir default to the config's output.* keys."""
    import dataclasses

    cfg = dataclasses.replace(cfg)  # run.cpp:61-63: resolve + validate a copy
    cfg.resolve()
    cfg.validate()
    if nsteps is None:
        nsteps = cfg.nsteps()
    cadence = cfg.cadence if cadence is None else cadence
    snapshot_cadence = cfg.snapshot_cadence if snapshot_cadence is None else snapshot_cadence
    profile_cadence = cfg.profile_cadence if profile_cadence is None else profile_cadence
    if out_dir is _FROM_CFG:
        out_dir = cfg.out_dir
    if out_dir is not None:  # run.cpp:70-73
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "config_resolved.cfg"), "w") as f:
            f.write(cfg.echo())
    grid = Grid1D.three_block(-cfg.L, cfg.L, cfg.fine_block_cells, cfg.coarse_block_cells,
                              cfg.refinement_ratio)
    ctx = Context(grid, cfg.k, cfg.penalty_scale, device)
    if exact:
        ctx.set_exact_reductions(True)
    try:
        res = N.sk_run_result()
        ccfg = cfg.to_c()
        rc = N.lib().sk_run(ctx.h, C.byref(ccfg), int(nsteps), int(cadence), int(snapshot_cadence),
                            int(profile_cadence), None if out_dir is None else str(out_dir).encode(),
                            C.byref(res))
        _check(rc)
        return dict(exit_code=res.exit_code, steps_done=res.steps_done, shrinks_e=res.shrinks_e,
                    shrinks_i=res.shrinks_i, wall_seconds=res.wall_seconds,
                    error=N.lib().sk_last_error().decode() if res.exit_code else "")
    finally:
        ctx.close()


# ----------------------------------------------------------------------------
# shift matrices / the `solkin matrices` table
# ----------------------------------------------------------------------------
def build_shift_matrices(k: int, alpha: float):
    """build_shift_matrices(ReferenceBasis::get(k), alpha) (advection.cpp:27-66):
    (A, B) as p x p arrays from the library's host constants. No GPU needed."""
    p = k + 1
    A = np.zeros((max(p, 1), max(p, 1)))
    B = np.zeros_like(A)
    _check(N.lib().sk_shift_matrices(int(k), float(alpha), A.ctypes.data_as(N._dp),
                                     B.ctypes.data_as(N._dp)))
    return A, B


def matrices_text(alpha: float, order: int) -> str:
    """the text `solkin matrices --alpha a --order k` prints (tools/solkin_main.cpp:43-57)"""
    A, B = build_shift_matrices(order, alpha)
    out = []
    for name, mat in (("A", A), ("B", B)):
        out.append(f"{name}(alpha={RC.g17(alpha)}), order {order}:\n")
        for row in mat:
            out.append("".join(RC.e17(x) for x in row) + "\n")
    return "".join(out)
