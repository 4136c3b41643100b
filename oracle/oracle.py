"""ctypes front-end for the CPU checkers (test / baseline infrastructure only).

Two libraries with the same shape:
  * libsk_oracle.so  -- plain-C restatement (oracle/sk_oracle.c), always built;
  * libsolkin_ref.so -- the reference sources compiled in place (oracle/Makefile),
                        present when built in a container that has /root/reference.
Both expose a "state" (blob initial data, run() loop body of
core/src/run.cpp:124-131) and unit-level operator entry points.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsk_oracle.so")
ORACLE_FMA_SO = os.path.join(HERE, "_build", "libsk_oracle_fma.so")  # envelope: FMA build
REF_SO = os.path.join(HERE, "_ref", "libsolkin_ref.so")

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_long)


def build(ref: bool | None = None) -> None:
    """make the oracle (and oracle/_ref when /root/reference exists)."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/core/src")
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def oracle_available() -> bool:
    return os.path.exists(ORACLE_SO)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _arr(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run oracle.build())")
        self.lib = C.CDLL(path)


# ----------------------------------------------------------------------------
class Oracle(_Lib):
    """plain-C restatement."""

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.sko_last_error.restype = C.c_char_p
        L.sko_state_new.restype = C.c_void_p
        L.sko_state_set_injection.argtypes = [C.c_void_p, C.c_double]
        L.sko_state_set_injection.restype = C.c_int
        L.sko_state_new.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_char_p, C.c_double, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_double]
        for n in ("sko_state_field", "sko_state_E", "sko_state_phi"):
            getattr(L, n).restype = _dp
        for n in ("sko_state_field", "sko_state_field_size", "sko_state_vmax", "sko_state_shrinks",
                  "sko_state_last_shrink", "sko_state_check_shrink"):
            getattr(L, n).argtypes = [C.c_void_p, C.c_int]
        L.sko_state_field_size.restype = C.c_long
        L.sko_state_vmax.restype = C.c_double
        L.sko_state_last_shrink.restype = C.c_long
        L.sko_state_step_index.restype = C.c_long
        for n in ("sko_state_E", "sko_state_phi", "sko_state_step_index", "sko_state_delete",
                  "sko_run_step"):
            getattr(L, n).argtypes = [C.c_void_p]
        L.sko_state_stats.argtypes = [C.c_void_p, _lp]
        L.sko_state_advect_x.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int]
        L.sko_state_advect_v.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, C.c_int]
        L.sko_state_post_limit.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p]
        L.sko_state_charge_density.argtypes = [C.c_void_p, _dp]
        L.sko_state_poisson_solve.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.sko_set_lapack.argtypes = [C.c_void_p, C.c_void_p]
        L.sko_state_shrink.argtypes = [C.c_void_p, C.c_int, _dp]
        L.sko_state_summary.argtypes = [C.c_void_p, _dp]
        L.sko_lagrange.restype = C.c_double
        L.sko_evaluate.restype = C.c_double
        L.sko_max_on.restype = C.c_double
        L.sko_min_on.restype = C.c_double
        L.sko_smoothness_beta.restype = C.c_double
        L.sko_max_on.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double]
        L.sko_min_on.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double]
        L.sko_inline_init.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double]
        L.sko_decompose_shift.argtypes = [C.c_double, C.c_double, C.c_double,
                                          C.POINTER(C.c_int), _dp]
        L.sko_shift_matrices.argtypes = [C.c_void_p, C.c_double, _dp, _dp]
        L.sko_required_ghost_width.argtypes = [C.c_double] * 4
        L.sko_minmod.restype = C.c_double
        L.sko_minmod.argtypes = [C.c_double] * 3
        L.sko_indicator_meanerr.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_double]
        L.sko_advect_v_lines.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                         C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_void_p, C.c_void_p]
        L.sko_limiter_parse.argtypes = [C.c_char_p, C.c_void_p]
        L.sko_dpbtrf_lower.argtypes = [C.c_int, C.c_int, _dp, C.c_int]
        L.sko_dpbtrs_lower.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp]
        self._basis = {}

    def last_error(self) -> str:
        return self.lib.sko_last_error().decode()

    # sko_basis is ~1.2 KB; keep opaque buffers per degree
    def basis(self, k):
        if k not in self._basis:
            buf = C.create_string_buffer(4096)
            rc = self.lib.sko_basis_init(buf, k)
            if rc:
                raise RuntimeError(self.last_error())
            self._basis[k] = buf
        return self._basis[k]

    def gauss_legendre(self, k):
        n = np.zeros(k + 1)
        w = np.zeros(k + 1)
        self.lib.sko_gauss_legendre(k, n.ctypes.data_as(_dp), w.ctypes.data_as(_dp))
        return n, w

    def decompose_shift(self, speed, dt, dx):
        i = C.c_int()
        a = C.c_double()
        self.lib.sko_decompose_shift(speed, dt, dx, C.byref(i), C.byref(a))
        return i.value, a.value

    def shift_matrices(self, k, alpha):
        p = k + 1
        A = np.zeros(p * p)
        B = np.zeros(p * p)
        rc = self.lib.sko_shift_matrices(self.basis(k), alpha, A.ctypes.data_as(_dp),
                                         B.ctypes.data_as(_dp))
        if rc:
            raise RuntimeError(self.last_error())
        return A.reshape(p, p), B.reshape(p, p)

    def max_on(self, k, u, a, b):
        u, pu = _arr(u)
        return self.lib.sko_max_on(self.basis(k), pu, a, b)

    def min_on(self, k, u, a, b):
        u, pu = _arr(u)
        return self.lib.sko_min_on(self.basis(k), pu, a, b)

    def inline_apply(self, k, alpha, thr, ul, ur, up):
        lim = C.create_string_buffer(512)
        self.lib.sko_inline_init(lim, self.basis(k), alpha, thr)
        ul, pl = _arr(ul)
        ur, pr = _arr(ur)
        up = np.array(up, dtype=np.float64)
        flags = self.lib.sko_inline_apply(lim, self.basis(k), pl, pr, up.ctypes.data_as(_dp))
        return flags, up

    def post_indicator(self, k, kind, thr, um, u0, up):
        um, a = _arr(um)
        u0, b = _arr(u0)
        up, c = _arr(up)
        if kind == 1:
            return self.lib.sko_indicator_minmod(self.basis(k), a, b, c)
        return self.lib.sko_indicator_meanerr(self.basis(k), a, b, c, thr)

    def post_modify(self, k, kind, um, u0, up):
        um, a = _arr(um)
        u0, b = _arr(u0)
        up, c = _arr(up)
        out = np.zeros(k + 1)
        cfg = C.create_string_buffer(256)
        self.lib.sko_limiter_parse(b"minmod+simple", cfg)
        fn = self.lib.sko_modify_simple_weno if kind == 1 else self.lib.sko_modify_line_weno
        fn(self.basis(k), a, b, c, cfg, out.ctypes.data_as(_dp))
        return out

    def smoothness_beta(self, k, u):
        u, pu = _arr(u)
        return self.lib.sko_smoothness_beta(self.basis(k), pu)

    def fine_to_coarse(self, k, fine, m):
        fine, pf = _arr(fine)
        out = np.zeros(k + 1)
        self.lib.sko_fine_to_coarse(self.basis(k), pf, m, out.ctypes.data_as(_dp))
        return out

    def coarse_to_fine(self, k, coarse, m):
        coarse, pc = _arr(coarse)
        out = np.zeros(m * (k + 1))
        self.lib.sko_coarse_to_fine(self.basis(k), pc, m, out.ctypes.data_as(_dp))
        return out

    def required_ghost_width(self, vmax, dt, sqrt_mu_min, dx):
        return self.lib.sko_required_ghost_width(vmax, dt, sqrt_mu_min, dx)

    def advect_v_lines(self, k, lines_in, gl, n, gr, E, charge_sign, sqrt_mu, tau, dv,
                       limiter: str = "none"):
        """v sweep of gathered lines [nlines, (gl+n+gr)*p] -> [nlines, n*p]."""
        p = k + 1
        lines_in = np.ascontiguousarray(lines_in, dtype=np.float64)
        nl = lines_in.shape[0]
        out = np.zeros((nl, n * p))
        E = np.ascontiguousarray(E, dtype=np.float64)
        cfg = C.create_string_buffer(256)
        self.lib.sko_limiter_parse(limiter.encode(), cfg)
        lim_ptr = cfg if limiter == "sldg" else None
        rc = self.lib.sko_advect_v_lines(self.basis(k), nl, lines_in.shape[1],
                                         lines_in.ctypes.data_as(_dp), gl, n, gr,
                                         out.ctypes.data_as(_dp), E.ctypes.data_as(_dp),
                                         charge_sign, sqrt_mu, tau, dv, lim_ptr, None)
        if rc:
            raise RuntimeError(self.last_error())
        return out

    def advect_x_line(self, k, grid_left, grid_cells, grid_dx, speed, tau, line,
                      inline_sldg=False, threshold=0.5, max_ghost=-1):
        nb = len(grid_cells)
        line = np.ascontiguousarray(line, dtype=np.float64)
        out = np.zeros_like(line)
        self.lib.sko_advect_x_line.argtypes = [C.c_int, C.c_int, _dp, C.POINTER(C.c_int), _dp,
                                               C.c_double, C.c_double, C.c_int, C.c_double,
                                               C.c_int, _dp, _dp]
        rc = self.lib.sko_advect_x_line(k, nb, (C.c_double * nb)(*grid_left),
                                        (C.c_int * nb)(*grid_cells), (C.c_double * nb)(*grid_dx),
                                        speed, tau, int(inline_sldg), threshold, max_ghost,
                                        line.ctypes.data_as(_dp), out.ctypes.data_as(_dp))
        if rc:
            raise RuntimeError(self.last_error())
        return out

    def set_rho_order(self, mode: int):
        """0 = reference order; 1 = electrons first (rounding-noise envelope)"""
        self.lib.sko_set_rho_order(int(mode))

    def set_lapack(self, lib=None):
        """Poisson operators created from now on factor and solve with
        ``lib``'s dpbtrf_/dpbtrs_ (a ctypes CDLL, e.g. openblas()); None = the
        reference-LAPACK restatement. Rounding-noise envelope only."""
        if lib is None:
            self.lib.sko_set_lapack(None, None)
        elif isinstance(lib, tuple):  # raw (dpbtrf, dpbtrs) function addresses
            self.lib.sko_set_lapack(C.c_void_p(lib[0]), C.c_void_p(lib[1]))
        else:
            self.lib.sko_set_lapack(C.cast(lib.dpbtrf_, C.c_void_p), C.cast(lib.dpbtrs_, C.c_void_p))

    def state(self, **cfg) -> "OracleState":
        return OracleState(self, **cfg)


def _cfg_args(cfg):
    c = dict(L=200.0, dt=0.1, k=3, mu=400.0, sigma=-1.0, vmax_e=12.0, vmax_i=12.0, nf=50, nc=50,
             m=1, nv=40, limiter="none", limiter_threshold=0.5, v_adjust=1, adapt_p=0.05,
             adapt_gamma=0.05, adapt_tol=1e-14, penalty_scale=10.0, scenario="blob", t0=2000.0)
    unknown = set(cfg) - set(c) - {"threads"}
    if unknown:
        raise KeyError(f"unknown oracle config keys {unknown}")
    c.update({k: v for k, v in cfg.items() if k in c})
    return c


def openblas():
    """The OpenBLAS 0.3.15 shipped in this image (opencv wheel), or None."""
    import glob

    d = "/opt/prime-rl/.venv/lib/python3.12/site-packages/opencv_python_headless.libs/"
    libs = glob.glob(d + "libopenblas*.so")
    if not libs:
        return None
    for dep in glob.glob(d + "libquadmath*") + glob.glob(d + "libgfortran*"):
        C.CDLL(dep, mode=C.RTLD_GLOBAL)
    return C.CDLL(libs[0])


def scipy_lapack():
    """(dpbtrf, dpbtrs) addresses of the LAPACK scipy links (scipy-openblas,
    a different build from openblas()), or None."""
    try:
        from scipy.linalg import cython_lapack
    except Exception:
        return None
    get = C.pythonapi.PyCapsule_GetPointer
    get.restype, get.argtypes = C.c_void_p, [C.py_object, C.c_char_p]
    name = C.pythonapi.PyCapsule_GetName
    name.restype, name.argtypes = C.c_char_p, [C.py_object]
    caps = cython_lapack.__pyx_capi__
    return tuple(get(caps[f], name(caps[f])) for f in ("dpbtrf", "dpbtrs"))


class _StateBase:
    P = ""

    def _fn(self, name):
        return getattr(self.lib, self.P + name)

    @property
    def k(self):
        return self.cfg["k"]

    @property
    def nx(self):
        return 2 * self.cfg["nf"] + self.cfg["nc"]

    @property
    def nv(self):
        return self.cfg["nv"]

    def shape(self):
        p = self.k + 1
        return (self.nv, p, self.nx, p)


class OracleState(_StateBase):
    P = "sko_state_"

    def __init__(self, owner: Oracle, **cfg):
        self.owner = owner
        self.lib = owner.lib
        self.cfg = _cfg_args(cfg)
        c = self.cfg
        self.h = self.lib.sko_state_new(c["L"], c["dt"], c["k"], c["mu"], c["sigma"], c["vmax_e"],
                                        c["vmax_i"], c["nf"], c["nc"], c["m"], c["nv"],
                                        c["limiter"].encode(), c["limiter_threshold"],
                                        int(c["v_adjust"]), c["adapt_p"], c["adapt_gamma"],
                                        c["adapt_tol"], c["penalty_scale"])
        if not self.h:
            raise RuntimeError(owner.last_error())
        if c["scenario"] == "injection":
            if self.lib.sko_state_set_injection(self.h, c["t0"]):
                raise RuntimeError(owner.last_error())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.sko_state_delete(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"oracle rc={rc}: {self.owner.last_error()}")

    def step(self):
        self._check(self.lib.sko_run_step(self.h))

    def field(self, species) -> np.ndarray:
        n = self.lib.sko_state_field_size(self.h, species)
        ptr = self.lib.sko_state_field(self.h, species)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy()

    def set_field(self, species, data):
        n = self.lib.sko_state_field_size(self.h, species)
        ptr = self.lib.sko_state_field(self.h, species)
        np.ctypeslib.as_array(ptr, shape=(n,))[:] = np.asarray(data, dtype=np.float64).ravel()

    def E(self):
        ptr = self.lib.sko_state_E(self.h)
        return np.ctypeslib.as_array(ptr, shape=(self.nx * (self.k + 1),)).copy()

    def vmax(self, species):
        return self.lib.sko_state_vmax(self.h, species)

    def step_index(self):
        return self.lib.sko_state_step_index(self.h)

    def shrinks(self, species):
        return self.lib.sko_state_shrinks(self.h, species)

    def last_shrink(self, species):
        return self.lib.sko_state_last_shrink(self.h, species)

    def stats(self):
        out = (C.c_long * 6)()
        self.lib.sko_state_stats(self.h, out)
        return dict(zip(("outputs", "inline_troubled", "inline_clamped", "inline_mean_outside",
                         "post_checked", "post_troubled"), list(out)))

    def advect_x(self, species, tau, limited=True, max_ghost=-1):
        self._check(self.lib.sko_state_advect_x(self.h, species, tau, int(limited), max_ghost))

    def advect_v(self, species, tau, E, limited=True):
        E, pE = _arr(E)
        self._check(self.lib.sko_state_advect_v(self.h, species, tau, pE, int(limited)))

    def post_limit(self, species, direction, mode):
        self._check(self.lib.sko_state_post_limit(self.h, species, direction, mode.encode()))

    def charge_density(self):
        rho = np.zeros(self.nx * (self.k + 1))
        self.lib.sko_state_charge_density(self.h, rho.ctypes.data_as(_dp))
        return rho

    def poisson_solve(self, rho):
        rho, pr = _arr(rho)
        E = np.zeros(self.nx * (self.k + 1))
        phi = np.zeros(self.nx * (self.k + 2))
        self._check(self.lib.sko_state_poisson_solve(self.h, pr, E.ctypes.data_as(_dp),
                                                     phi.ctypes.data_as(_dp)))
        return E, phi

    def poisson_band(self):
        """the assembled SIPG band (kd+1 rows per column, lower, column-major)"""
        n, kd = C.c_int(), C.c_int()
        f = self.lib.sko_state_poisson_band
        f.restype, f.argtypes = _dp, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        ptr = f(self.h, C.byref(n), C.byref(kd))
        return np.ctypeslib.as_array(ptr, shape=(n.value, kd.value + 1)).copy()

    def poisson_load(self, rho):
        rho, pr = _arr(rho)
        out = np.zeros(self.nx * (self.k + 2))
        self.lib.sko_state_poisson_load.argtypes = [C.c_void_p, _dp, _dp]
        self._check(self.lib.sko_state_poisson_load(self.h, pr, out.ctypes.data_as(_dp)))
        return out

    def check_shrink(self, species):
        r = self.lib.sko_state_check_shrink(self.h, species)
        if r < 0:
            raise RuntimeError(self.owner.last_error())
        return bool(r)

    def shrink(self, species):
        out = np.zeros(4)
        self._check(self.lib.sko_state_shrink(self.h, species, out.ctypes.data_as(_dp)))
        return dict(zip(("vmax_before", "vmax_after", "mass_before", "mass_after"), out))

    def summary(self):
        out = np.zeros(11)
        self.lib.sko_state_summary(self.h, out.ctypes.data_as(_dp))
        keys = ("mass_e", "mass_i", "l2_e", "l2_i", "e_energy", "vmax_e", "vmax_i", "mom_e",
                "mom_i", "ekin_e", "ekin_i")
        return dict(zip(keys, out))


# ----------------------------------------------------------------------------
class Ref(_Lib):
    """the reference (core/src/*.cpp) compiled in place + oracle/ref_driver.cpp."""

    def __init__(self, path=REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_state_create.restype = C.c_void_p
        L.ref_state_set_injection.argtypes = [C.c_void_p, C.c_double]
        L.ref_state_set_injection.restype = C.c_int
        L.ref_state_wall_flux.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.ref_state_wall_flux.restype = C.c_int
        L.ref_state_time.argtypes = [C.c_void_p]
        L.ref_state_time.restype = C.c_double
        L.ref_state_write_snapshot.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_state_write_snapshot.restype = C.c_int
        L.ref_run_files.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int, C.c_char_p]
        L.ref_run_files.restype = C.c_int
        L.ref_state_create.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_char_p, C.c_double, C.c_int, C.c_double,
                                       C.c_double, C.c_double, C.c_double, C.c_int]
        for n in ("ref_state_free", "ref_state_step", "ref_state_step_index"):
            getattr(L, n).argtypes = [C.c_void_p]
        L.ref_state_step_index.restype = C.c_long
        L.ref_state_run.argtypes = [C.c_void_p, C.c_int]
        L.ref_state_run.restype = C.c_double
        for n in ("ref_state_field_size", "ref_state_vmax", "ref_state_shrinks",
                  "ref_state_last_shrink", "ref_state_check_shrink"):
            getattr(L, n).argtypes = [C.c_void_p, C.c_int]
        L.ref_state_field_size.restype = C.c_long
        L.ref_state_vmax.restype = C.c_double
        L.ref_state_last_shrink.restype = C.c_long
        L.ref_state_get_field.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_state_set_field.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_state_get_E.argtypes = [C.c_void_p, _dp]
        L.ref_state_get_phi.argtypes = [C.c_void_p, _dp]
        L.ref_state_get_stats.argtypes = [C.c_void_p, _lp]
        L.ref_state_get_timers.argtypes = [C.c_void_p, _dp]
        L.ref_state_summary.argtypes = [C.c_void_p, _dp]
        L.ref_state_advect_x.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int]
        L.ref_state_advect_v.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, C.c_int]
        L.ref_state_post_limit.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p]
        L.ref_state_charge_density.argtypes = [C.c_void_p, _dp]
        L.ref_state_poisson_solve.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_state_shrink.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_decompose_shift.argtypes = [C.c_double, C.c_double, C.c_double,
                                          C.POINTER(C.c_int), _dp]
        L.ref_shift_matrices.argtypes = [C.c_int, C.c_double, _dp, _dp]
        L.ref_max_on.restype = C.c_double
        L.ref_min_on.restype = C.c_double
        L.ref_max_on.argtypes = [C.c_int, _dp, C.c_double, C.c_double]
        L.ref_min_on.argtypes = [C.c_int, _dp, C.c_double, C.c_double]
        L.ref_inline_apply.argtypes = [C.c_int, C.c_double, C.c_double, _dp, _dp, _dp]
        L.ref_post_indicator.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp, _dp]
        L.ref_post_modify.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_smoothness_beta.restype = C.c_double
        L.ref_smoothness_beta.argtypes = [C.c_int, _dp]
        L.ref_fine_to_coarse.argtypes = [C.c_int, _dp, C.c_int, _dp]
        L.ref_coarse_to_fine.argtypes = [C.c_int, _dp, C.c_int, _dp]

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def self_checks(self):
        fails = self.lib.ref_self_checks()
        return fails, self.last_error()

    def config_eval(self, preset="", file="", kv=(), resolve=False):
        """RunConfig layered as cmd_run does (solkin_main.cpp:20-28): returns
        ("ok", echo, [violations], nsteps) or ("error", message)."""
        L = self.lib
        L.ref_config_eval.restype = C.c_int
        L.ref_config_eval.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_char_p,
                                      C.c_long, C.c_char_p, C.c_long, C.POINTER(C.c_long)]
        echo = C.create_string_buffer(1 << 14)
        viol = C.create_string_buffer(1 << 14)
        n = C.c_long(0)
        kvs = "".join(f"{k}\t{v}\n" for k, v in kv).encode()
        rc = L.ref_config_eval(preset.encode(), str(file).encode(), kvs, int(resolve), echo,
                               len(echo), viol, len(viol), C.byref(n))
        if rc:
            return ("error", self.last_error())
        lines = viol.value.decode().split("\n")
        return ("ok", echo.value.decode(), [x for x in lines if x], n.value)

    def matrices_text(self, alpha, order):
        """the `solkin matrices` table (solkin_main.cpp:43-57)"""
        L = self.lib
        L.ref_matrices_text.restype = C.c_int
        L.ref_matrices_text.argtypes = [C.c_double, C.c_int, C.c_char_p, C.c_long]
        out = C.create_string_buffer(1 << 14)
        if L.ref_matrices_text(float(alpha), int(order), out, len(out)):
            raise RuntimeError(self.last_error())
        return out.value.decode()

    def gauss_legendre(self, k):
        n = np.zeros(k + 1)
        w = np.zeros(k + 1)
        self.lib.ref_gauss_legendre(k, n.ctypes.data_as(_dp), w.ctypes.data_as(_dp))
        return n, w

    def decompose_shift(self, speed, dt, dx):
        i = C.c_int()
        a = C.c_double()
        self.lib.ref_decompose_shift(speed, dt, dx, C.byref(i), C.byref(a))
        return i.value, a.value

    def shift_matrices(self, k, alpha):
        p = k + 1
        A = np.zeros(p * p)
        B = np.zeros(p * p)
        if self.lib.ref_shift_matrices(k, alpha, A.ctypes.data_as(_dp), B.ctypes.data_as(_dp)):
            raise RuntimeError(self.last_error())
        return A.reshape(p, p), B.reshape(p, p)

    def max_on(self, k, u, a, b):
        u, pu = _arr(u)
        return self.lib.ref_max_on(k, pu, a, b)

    def min_on(self, k, u, a, b):
        u, pu = _arr(u)
        return self.lib.ref_min_on(k, pu, a, b)

    def inline_apply(self, k, alpha, thr, ul, ur, up):
        ul, pl = _arr(ul)
        ur, pr = _arr(ur)
        up = np.array(up, dtype=np.float64)
        flags = self.lib.ref_inline_apply(k, alpha, thr, pl, pr, up.ctypes.data_as(_dp))
        return flags, up

    def post_indicator(self, k, kind, thr, um, u0, up):
        um, a = _arr(um)
        u0, b = _arr(u0)
        up, c = _arr(up)
        return self.lib.ref_post_indicator(k, kind, thr, a, b, c)

    def post_modify(self, k, kind, um, u0, up):
        um, a = _arr(um)
        u0, b = _arr(u0)
        up, c = _arr(up)
        out = np.zeros(k + 1)
        self.lib.ref_post_modify(k, kind, a, b, c, out.ctypes.data_as(_dp))
        return out

    def smoothness_beta(self, k, u):
        u, pu = _arr(u)
        return self.lib.ref_smoothness_beta(k, pu)

    def fine_to_coarse(self, k, fine, m):
        fine, pf = _arr(fine)
        out = np.zeros(k + 1)
        self.lib.ref_fine_to_coarse(k, pf, m, out.ctypes.data_as(_dp))
        return out

    def coarse_to_fine(self, k, coarse, m):
        coarse, pc = _arr(coarse)
        out = np.zeros(m * (k + 1))
        self.lib.ref_coarse_to_fine(k, pc, m, out.ctypes.data_as(_dp))
        return out

    def state(self, **cfg) -> "RefState":
        return RefState(self, **cfg)


class RefState(_StateBase):
    def __init__(self, owner: Ref, threads: int = 1, **cfg):
        self.owner = owner
        self.lib = owner.lib
        self.cfg = _cfg_args(cfg)
        c = self.cfg
        self.h = self.lib.ref_state_create(c["L"], c["dt"], c["k"], c["mu"], c["sigma"],
                                           c["vmax_e"], c["vmax_i"], c["nf"], c["nc"], c["m"],
                                           c["nv"], c["limiter"].encode(),
                                           c["limiter_threshold"], int(c["v_adjust"]),
                                           c["adapt_p"], c["adapt_gamma"], c["adapt_tol"],
                                           c["penalty_scale"], int(threads))
        if not self.h:
            raise RuntimeError(owner.last_error())
        if c["scenario"] == "injection":
            if self.lib.ref_state_set_injection(self.h, c["t0"]):
                raise RuntimeError(owner.last_error())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_state_free(self.h)
            self.h = None

    def wall_flux(self, species, side):
        out = (C.c_double * 2)()
        if self.lib.ref_state_wall_flux(self.h, species, side, out):
            raise RuntimeError(self.owner.last_error())
        return out[0], out[1]

    def time(self):
        return self.lib.ref_state_time(self.h)

    def write_snapshot(self, directory):
        if self.lib.ref_state_write_snapshot(self.h, str(directory).encode()):
            raise RuntimeError(self.owner.last_error())

    def run_files(self, t_final, cadence, snapshot_cadence, profile_cadence, directory):
        """the reference's run() with files for this configuration (fresh state)"""
        if self.lib.ref_run_files(self.h, t_final, cadence, snapshot_cadence, profile_cadence,
                                  str(directory).encode()):
            raise RuntimeError(self.owner.last_error())

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"reference rc={rc}: {self.owner.last_error()}")

    def step(self):
        self._check(self.lib.ref_state_step(self.h))

    def run(self, n) -> float:
        t = self.lib.ref_state_run(self.h, n)
        if t < 0:
            raise RuntimeError(self.owner.last_error())
        return t

    def field(self, species):
        n = self.lib.ref_state_field_size(self.h, species)
        out = np.zeros(n)
        self.lib.ref_state_get_field(self.h, species, out.ctypes.data_as(_dp))
        return out

    def set_field(self, species, data):
        data, pd = _arr(np.asarray(data).ravel())
        self.lib.ref_state_set_field(self.h, species, pd)

    def E(self):
        out = np.zeros(self.nx * (self.k + 1))
        self.lib.ref_state_get_E(self.h, out.ctypes.data_as(_dp))
        return out

    def vmax(self, species):
        return self.lib.ref_state_vmax(self.h, species)

    def step_index(self):
        return self.lib.ref_state_step_index(self.h)

    def shrinks(self, species):
        return self.lib.ref_state_shrinks(self.h, species)

    def last_shrink(self, species):
        return self.lib.ref_state_last_shrink(self.h, species)

    def stats(self):
        out = (C.c_long * 6)()
        self.lib.ref_state_get_stats(self.h, out)
        return dict(zip(("outputs", "inline_troubled", "inline_clamped", "inline_mean_outside",
                         "post_checked", "post_troubled"), list(out)))

    def timers(self):
        out = np.zeros(5)
        self.lib.ref_state_get_timers(self.h, out.ctypes.data_as(_dp))
        return dict(zip(("source", "advect_x", "advect_v", "poisson", "post_limiter"), out))

    def advect_x(self, species, tau, limited=True, max_ghost=-1):
        self._check(self.lib.ref_state_advect_x(self.h, species, tau, int(limited), max_ghost))

    def advect_v(self, species, tau, E, limited=True):
        E, pE = _arr(E)
        self._check(self.lib.ref_state_advect_v(self.h, species, tau, pE, int(limited)))

    def post_limit(self, species, direction, mode):
        self._check(self.lib.ref_state_post_limit(self.h, species, direction, mode.encode()))

    def charge_density(self):
        rho = np.zeros(self.nx * (self.k + 1))
        self._check(self.lib.ref_state_charge_density(self.h, rho.ctypes.data_as(_dp)))
        return rho

    def poisson_solve(self, rho):
        rho, pr = _arr(rho)
        E = np.zeros(self.nx * (self.k + 1))
        phi = np.zeros(self.nx * (self.k + 2))
        self._check(self.lib.ref_state_poisson_solve(self.h, pr, E.ctypes.data_as(_dp),
                                                     phi.ctypes.data_as(_dp)))
        return E, phi

    def check_shrink(self, species):
        r = self.lib.ref_state_check_shrink(self.h, species)
        if r < 0:
            raise RuntimeError(self.owner.last_error())
        return bool(r)

    def shrink(self, species):
        out = np.zeros(4)
        self._check(self.lib.ref_state_shrink(self.h, species, out.ctypes.data_as(_dp)))
        return dict(zip(("vmax_before", "vmax_after", "mass_before", "mass_after"), out))

    def summary(self):
        out = np.zeros(7)
        self.lib.ref_state_summary(self.h, out.ctypes.data_as(_dp))
        return dict(zip(("mass_e", "mass_i", "l2_e", "l2_i", "e_energy", "vmax_e", "vmax_i"), out))
