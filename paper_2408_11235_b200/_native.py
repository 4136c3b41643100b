"""ctypes binding of include/sk_b200.h (libsk_b200.so). No CPU fallback:
loading fails loudly when the library is missing, and every compute entry
point raises when no CUDA device is present."""
from __future__ import annotations

import ctypes as C
import os
import re

from .build import LIB

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "sk_b200.h")

SK_OK, SK_ERR_RUNTIME, SK_ERR_SIMULATION, SK_ERR_CUDA = 0, 1, 2, 3


class sk_limiter(C.Structure):
    _fields_ = [("indicator", C.c_int), ("modifier", C.c_int), ("inline_sldg", C.c_int),
                ("threshold", C.c_double), ("gamma_simple", C.c_double * 3),
                ("gamma_line", C.c_double * 3), ("epsilon", C.c_double)]


class sk_stats(C.Structure):
    _fields_ = [(n, C.c_longlong) for n in ("outputs", "inline_troubled", "inline_clamped",
                                            "inline_mean_outside", "post_checked",
                                            "post_troubled")]


class sk_run_result(C.Structure):
    _fields_ = [("exit_code", C.c_int), ("steps_done", C.c_long), ("shrinks_e", C.c_long),
                ("shrinks_i", C.c_long), ("wall_seconds", C.c_double), ("stats", sk_stats)]


class sk_vadjust(C.Structure):
    _fields_ = [("p", C.c_double), ("gamma", C.c_double), ("tol", C.c_double)]


class sk_shrink_result(C.Structure):
    _fields_ = [("vmax_before", C.c_double), ("vmax_after", C.c_double),
                ("mass_before", C.c_double), ("mass_after", C.c_double)]


class sk_flux_sample(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t", "je_plus", "je_minus", "ji_plus", "ji_minus", "je_naive",
                                          "ji_naive", "mass_e", "mass_i", "e_energy", "vmax_e", "vmax_i")]


class sk_summary(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mass_e", "mass_i", "charge", "l2_e", "l2_i", "e_energy",
                                          "vmax_e", "vmax_i")]


class sk_run_config(C.Structure):
    _fields_ = [("L", C.c_double), ("dt", C.c_double), ("mu", C.c_double), ("sigma", C.c_double),
                ("vmax_e", C.c_double), ("vmax_i", C.c_double), ("k", C.c_int),
                ("fine_block_cells", C.c_int), ("coarse_block_cells", C.c_int),
                ("refinement_ratio", C.c_int), ("v_cells", C.c_int), ("limiter", sk_limiter),
                ("v_adjust", C.c_int), ("policy", sk_vadjust), ("penalty_scale", C.c_double),
                ("scenario", C.c_int), ("t0", C.c_double)]


_vp, _dp, _ip, _lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_long)
_i, _d, _sz = C.c_int, C.c_double, C.c_size_t

SIGNATURES = {
    "sk_last_error": (C.c_char_p, []),
    "sk_last_error_step": (C.c_long, []),
    "sk_version": (C.c_char_p, []),
    "sk_grid_three_block": (_i, [_d, _d, _i, _i, _i, _dp, _ip, _dp]),
    "sk_shift_matrices": (_i, [_i, _d, _dp, _dp]),
    "sk_ctx_create": (_i, [_i, _i, _i, _dp, _ip, _dp, _d, C.POINTER(_vp)]),
    "sk_ctx_destroy": (_i, [_vp]),
    "sk_ctx_set_stream": (_i, [_vp, _vp]),
    "sk_ctx_set_eager_errors": (_i, [_vp, _i]),
    "sk_ctx_set_exact_reductions": (_i, [_vp, _i]),
    "sk_ctx_set_exact_parts": (_i, [_vp, _i]),
    "sk_ctx_set_step_fusion": (_i, [_vp, _i]),
    "sk_state_step_fusion": (_i, [_vp, C.POINTER(_i)]),
    "sk_ctx_set_post_fusion": (_i, [_vp, _i]),
    "sk_ctx_check_guards": (_i, [_vp, C.POINTER(C.c_longlong)]),
    "sk_ctx_set_fix_capacity": (_i, [_vp, C.c_uint]),
    "sk_ctx_synchronize": (_i, [_vp]),
    "sk_stats_get": (_i, [_vp, C.POINTER(sk_stats)]),
    "sk_stats_reset": (_i, [_vp]),
    "sk_field_create": (_i, [_vp, _i, _d, _d, _i, C.POINTER(_vp)]),
    "sk_field_destroy": (_i, [_vp]),
    "sk_field_size": (_sz, [_vp]),
    "sk_field_data_dev": (_vp, [_vp]),
    "sk_field_upload": (_i, [_vp, _dp, _sz]),
    "sk_field_download": (_i, [_vp, _dp, _sz]),
    "sk_field_perturb": (_i, [_vp, C.c_ulonglong, _d]),
    "sk_field_download_2d": (_i, [_vp, _dp, _sz, _sz, _sz, _sz]),
    "sk_field_upload_async": (_i, [_vp, _dp, _sz]),
    "sk_field_download_async": (_i, [_vp, _dp, _sz]),
    "sk_field_v_grid": (_i, [_vp, _dp, _dp, _ip]),
    "sk_field_create_shard": (_i, [_vp, _i, _d, _d, _i, _i, _i, _i, C.POINTER(_vp)]),
    "sk_field_halo": (_i, [_vp, _i, _i, C.POINTER(_vp), C.POINTER(_sz)]),
    "sk_field_halo_n": (_i, [_vp, _i, _i, _i, C.POINTER(_vp), C.POINTER(_sz)]),
    "sk_state_create_shard": (_i, [_vp, C.POINTER(sk_run_config), _i, _i, _i, C.POINTER(_vp)]),
    "sk_state_rho_dev": (_vp, [_vp]),
    "sk_state_shrink_flags_dev": (_vp, [_vp]),
    "sk_state_shrink_halo": (_i, [_vp]),
    "sk_state_vhalo_need": (_i, [_vp, C.POINTER(C.c_int)]),
    "sk_state_set_vhalo": (_i, [_vp, _i, _i]),
    "sk_state_vhalo_capacity": (_i, [_vp]),
    "sk_state_phase": (_i, [_vp, _i]),
    "sk_field_fill_blob": (_i, [_vp, _d]),
    "sk_advect_x": (_i, [_vp, _d, _d, _i, C.POINTER(sk_limiter), _i, C.c_long]),
    "sk_advect_v": (_i, [_vp, _d, _vp, _d, _d, _i, C.POINTER(sk_limiter)]),
    "sk_post_limit": (_i, [_vp, _i, C.POINTER(sk_limiter), _i]),
    "sk_charge_density": (_i, [_vp, _vp, _vp]),
    "sk_poisson_solve": (_i, [_vp, _vp, _vp, _vp]),
    "sk_check_velocity_shrink": (_i, [_vp, C.POINTER(sk_vadjust), _ip]),
    "sk_shrink_velocity_domain": (_i, [_vp, C.POINTER(sk_vadjust), C.POINTER(sk_shrink_result)]),
    "sk_field_moments": (_i, [_vp, _dp]),
    "sk_electric_energy": (_i, [_vp, _vp, _dp]),
    "sk_state_create": (_i, [_vp, C.POINTER(sk_run_config), C.POINTER(_vp)]),
    "sk_state_destroy": (_i, [_vp]),
    "sk_state_field": (_vp, [_vp, _i]),
    "sk_state_E_dev": (_vp, [_vp]),
    "sk_state_download_E": (_i, [_vp, _dp, _sz]),
    "sk_state_download_rho": (_i, [_vp, _dp, _sz]),
    "sk_strang_step": (_i, [_vp]),
    "sk_run_step": (_i, [_vp]),
    "sk_run_steps": (_i, [_vp, _i]),
    "sk_state_prepare_steps": (_i, [_vp, _i]),
    "sk_state_step_index": (_i, [_vp, _lp]),
    "sk_state_shrinks": (_i, [_vp, _i, _ip, _lp]),
    "sk_run_step_host": (_i, [_vp, _dp, _dp, _sz]),
    "sk_run_steps_host": (_i, [_vp, _i, _dp, _dp, _sz]),
    "sk_state_time": (_i, [_vp, _dp]),
    "sk_state_wall_flux": (_i, [_vp, _i, _i, _dp, _dp]),
    "sk_state_sample_fluxes": (_i, [_vp, C.POINTER(sk_flux_sample)]),
    "sk_state_summarize": (_i, [_vp, C.POINTER(sk_summary)]),
    "sk_state_write_snapshot": (_i, [_vp, C.c_char_p]),
    "sk_state_write_profiles": (_i, [_vp, C.c_char_p]),
    "sk_run": (_i, [_vp, C.POINTER(sk_run_config), C.c_long, _i, _i, _i, C.c_char_p, C.POINTER(sk_run_result)]),
    "sk_state_set_phase_timing": (_i, [_vp, _i]),
    "sk_state_phase_times": (_i, [_vp, _dp, _lp, _i]),
    "sk_ctx_launch_count": (C.c_longlong, [_vp]),
}

PHASES = ("x_tables", "x_sweep_1", "post_x_1", "charge_density", "poisson", "v_tables",
          "v_sweep", "post_v", "x_sweep_2", "post_x_2", "step_end_cutoff",
          "x_fix_1", "v_fix", "x_fix_2")


def header_symbols() -> list[str]:
    """Function names declared in include/sk_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sk_[A-Za-z0-9_]+)\s*\(", text)))


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.environ.get("SK_B200_LIB") or LIB  # (another build of the same ABI, for A/B timing)
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is not built: run __graft_entry__.build() "
                               "(the sLdG step has no CPU fallback)")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
