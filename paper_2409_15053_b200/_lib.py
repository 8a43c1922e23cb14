"""ctypes binding of the C ABI in include/flz.h (libflz.so, built in-tree by csrc/Makefile).

The library is the product; this module only declares signatures.  It fails loudly when
libflz.so is missing — there is no Python/NumPy fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLZ_LIB", os.path.join(PKG_DIR, "libflz.so"))  # FLZ_LIB: kernel-variant A/B runs
CSRC = os.path.join(PKG_DIR, "csrc")

FLZ_OK = 0
ERROR_NAMES = {-1: "EINVAL", -2: "EDIM", -3: "EINTERVAL", -4: "ECUDA", -5: "ENODEV", -6: "ENCCL",
               -7: "ENOMEM", -8: "EPARSE", -9: "ENUMERIC"}

f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
vp, d, i64, i32, u64, sz = C.c_void_p, C.c_double, C.c_int64, C.c_int, C.c_uint64, C.c_size_t
dP, iP, i64P, szP = C.POINTER(d), C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(sz)


class FlzError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"flz error {ERROR_NAMES.get(code, code)}: {message}")
        self.code = code


class FlzConfig(C.Structure):
    """Mirror of ``flz_config`` (include/flz.h) / ``speig::LanczosConfig`` (lanczos.hpp:14-29)."""

    _fields_ = [
        ("block_size", C.c_int32), ("tol", C.c_double), ("max_dim", C.c_int32),
        ("check_every", C.c_int32), ("seed", C.c_uint64), ("extra_ritz", C.c_int32),
        ("bounds_steps", C.c_int32), ("degree", C.c_int32), ("epsilon", C.c_double),
        ("max_degree", C.c_int32), ("collect_diagnostics", C.c_int32),
        ("return_vectors", C.c_int32), ("jackson_damping", C.c_int32),
    ]


class FlzStats(C.Structure):
    """Mirror of ``flz_stats`` / ``speig::SolveStats`` (lanczos.hpp:136-155) + device extras."""

    _fields_ = [
        ("block_steps", C.c_int32), ("basis_vectors", C.c_int32), ("degree", C.c_int32),
        ("mv_iteration", C.c_uint64), ("mv_bounds", C.c_uint64), ("mv_total", C.c_uint64),
        ("time_total_s", C.c_double), ("time_preproc_s", C.c_double), ("time_orth_s", C.c_double),
        ("time_mv_s", C.c_double), ("checks", C.c_int32), ("converged", C.c_int32),
        ("breakdown_replacements", C.c_int32), ("degree_clamped", C.c_int32),
        ("norm_estimate", C.c_double), ("lambda_min_est", C.c_double),
        ("lambda_max_est", C.c_double), ("ortho_error", C.c_double),
        ("time_check_s", C.c_double), ("time_recover_s", C.c_double),
        ("time_upload_s", C.c_double), ("gpu_launches", C.c_uint64),
    ]


_SIGS = {
    "flz_last_error": (C.c_char_p, []),
    "flz_version": (C.c_char_p, []),
    "flz_ctx_create": (i32, [i32, C.POINTER(vp)]),
    "flz_ctx_create_dist": (i32, [i32, i32, i32, vp, C.POINTER(vp)]),
    "flz_nccl_unique_id": (i32, [vp]),
    "flz_loop_hub_create": (i32, [i32, C.POINTER(vp)]),
    "flz_loop_hub_destroy": (None, [vp]),
    "flz_ctx_create_loopback": (i32, [i32, i32, i32, vp, C.POINTER(vp)]),
    "flz_ctx_destroy": (None, [vp]),
    "flz_ctx_sync": (i32, [vp]),
    "flz_ctx_make_current": (i32, [vp]),
    "flz_ctx_rank": (i32, [vp]),
    "flz_ctx_nranks": (i32, [vp]),
    "flz_ctx_launch_count": (u64, [vp]),
    "flz_timer_start": (i32, [vp, i32]),
    "flz_timer_stop": (i32, [vp, i32, dP]),
    "flz_flush_l2": (i32, [vp, sz]),
    "flz_ctx_set_exact": (i32, [vp, i32]),
    "flz_host_alloc": (i32, [sz, C.POINTER(vp)]),
    "flz_host_free": (None, [vp]),
    "flz_mem_info": (i32, [vp, szP, szP]),
    "flz_matrix_upload": (i32, [vp, i64, i64, i64, i64p, i32p, f64p, i32, C.POINTER(vp)]),
    "flz_matrix_destroy": (None, [vp]),
    "flz_matrix_rows_local": (i64, [vp]),
    "flz_matrix_nnz_local": (i64, [vp]),
    "flz_matrix_stats": (i32, [vp, i64P, i64P, i64P, i64P]),
    "flz_matrix_layout": (i32, [vp, i64P, i64P]),
    "flz_ctx_set_tuning": (i32, [vp, i32, i32, i32]),
    "flz_plan_create": (i32, [i64, i32, i32, i64p, i64p, i32p, f64p, i32, C.POINTER(vp)]),
    "flz_plan_destroy": (None, [vp]),
    "flz_matrix_upload_plan": (i32, [vp, vp, C.POINTER(vp)]),
    "flz_plan_info": (i32, [vp, i64p]),
    "flz_plan_need": (i64, [vp, i32, vp]),
    "flz_plan_set_give": (i32, [vp, i32, i64, i64p]),
    "flz_plan_arrays": (i32, [vp] + [vp] * 12),
    "flz_plan_ug": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "flz_plan_p2": (i32, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "flz_plan_hy": (i32, [vp] * 11),
    "flz_matrix_k1_info": (i32, [vp, i32, vp, vp, i32]),
    "flz_plan_tiles": (i32, [vp, vp, vp]),
    "flz_plan_tile_slab": (i32, [vp, vp]),
    "flz_matvec_count": (u64, []),
    "flz_reset_matvec_count": (None, []),
    "flz_matvec_sub": (None, [u64]),
    "flz_basis_truncate": (i32, [vp, vp, i64, d]),
    "flz_spmm": (i32, [vp, vp, vp, i32, vp, i32]),
    "flz_filter_apply": (i32, [vp, vp, f64p, i32, d, d, vp, i32, vp]),
    "flz_filter_bench": (i32, [vp, vp, f64p, i32, d, d, vp, i32, i32, i32, dP, vp]),
    "flz_dot": (i32, [vp, f64p, f64p, i64, dP]),
    "flz_axpy": (i32, [vp, d, f64p, f64p, i64]),
    "flz_clenshaw_combine": (i32, [vp, i64, d, d, d, f64p, f64p, f64p, f64p, f64p]),
    "flz_basis_create": (i32, [vp, vp, i64, i32, f64p, C.POINTER(vp)]),
    "flz_basis_destroy": (None, [vp]),
    "flz_basis_blocks": (i64, [vp]),
    "flz_basis_get": (i32, [vp, vp, i64, i64, f64p]),
    "flz_basis_set": (i32, [vp, vp, i64, f64p]),
    "flz_lanczos_step": (i32, [vp, vp, vp, vp, i32, d, d, f64p, f64p, dP, u8p]),
    "flz_orthogonalize_column": (i32, [vp, vp, i64, i32, f64p, dP]),
    "flz_basis_ortho_error": (i32, [vp, vp, vp, dP]),
    "flz_basis_times": (i32, [vp, dP, dP]),
    "flz_ritz_lift": (i32, [vp, vp, vp, i64, f64p, i32, f64p, u8p, iP, f64p]),
    "flz_ritz_rotate": (i32, [vp, vp, f64p, f64p, i32, d, f64p, vp]),
    "flz_ritz_plain": (i32, [vp, vp, vp, f64p, i32, d, f64p, vp]),
    "flz_bounds_lanczos": (i32, [vp, vp, i32, f64p, f64p, f64p, dP, iP]),
}

# host-side solver entry points (include/flz_solver.h, csrc/host/capi_solver.cpp)
_SOLVER_SIGS = {
    "flz_config_default": (None, [C.POINTER(FlzConfig)]),
    "flz_set_default_ctx": (i32, [vp]),
    "flz_set_thread_ctx": (i32, [vp]),
    "flz_default_ctx": (i32, [C.POINTER(vp)]),
    "flz_hostmatrix_from_triplets": (i32, [i64, i64, i64p, i64p, f64p, C.POINTER(vp)]),
    "flz_hostmatrix_from_csr": (i32, [i64, i64p, i32p, f64p, i32, C.POINTER(vp)]),
    "flz_hostmatrix_from_local_rows": (i32, [i64, i64, i64, i64p, i32p, f64p, C.POINTER(vp)]),
    "flz_hostmatrix_load_mm": (i32, [C.c_char_p, C.POINTER(vp)]),
    "flz_hostmatrix_save_bin": (i32, [vp, C.c_char_p]),
    "flz_hostmatrix_load_bin": (i32, [C.c_char_p, C.POINTER(vp)]),
    "flz_hostmatrix_save_mm": (i32, [vp, C.c_char_p]),
    "flz_hostmatrix_free": (None, [vp]),
    "flz_hostmatrix_dims": (i32, [vp, i64P, i64P]),
    "flz_hostmatrix_layout": (i32, [vp, i64P, i64P]),
    "flz_hostmatrix_k1_info": (i32, [vp, i32, vp, vp, i32]),
    "flz_hostmatrix_csr": (i32, [vp, i64p, i32p, f64p]),
    "flz_hostmatrix_spmm": (i32, [vp, f64p, i64, i32, f64p]),
    "flz_hostmatrix_filter_apply": (i32, [vp, f64p, i32, d, d, f64p, i64, i32, f64p]),
    "flz_indicator_coefficients": (i32, [d, d, i32, f64p]),
    "flz_jackson_factors": (i32, [i32, f64p]),
    "flz_select_degree": (i32, [d, d, d, i32, iP]),
    "flz_clenshaw": (d, [f64p, i32, d]),
    "flz_build_filter": (i32, [d, d, d, d, i32, d, i32, vp, i32, dP, dP, iP]),
    "flz_init_block": (i32, [i64, i32, u64, f64p]),
    "flz_estimate_bounds": (i32, [vp, i32, u64, dP, dP]),
    "flz_sym_band_eig": (i32, [i64, i64, f64p, f64p, vp]),
    "flz_band_ritz_rows": (i32, [i64, i64, f64p, i64, i64p, f64p, vp]),
    "flz_band_eigenvectors": (i32, [i64, i64, f64p, f64p, i64, i64p, f64p, dP, dP]),
    "flz_fact_create": (i32, [vp, f64p, i32, d, d, d, d, f64p, i32, i64, C.POINTER(vp)]),
    "flz_fact_free": (None, [vp]),
    "flz_fact_expand": (i32, [vp, i32]),
    "flz_fact_block_count": (i64, [vp]),
    "flz_fact_get": (i32, [vp, vp, vp, vp, vp]),
    "flz_fact_ortho_error": (i32, [vp, dP]),
    "flz_fact_flags": (i32, [vp]),
    "flz_fact_check": (i32, [vp, d, d, d, i32, f64p, f64p, u8p, u8p]),
    "flz_solve": (i32, [vp, d, d, C.POINTER(FlzConfig), i32, C.POINTER(vp)]),
    "flz_result_free": (None, [vp]),
    "flz_result_count": (i64, [vp]),
    "flz_result_get": (i32, [vp, vp, vp, vp, C.POINTER(FlzStats)]),
    "flz_result_vectors": (vp, [vp]),
    "flz_result_rows": (i64, [vp]),
}


def build(verbose: bool = False) -> str:
    """Compile libflz.so for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-C", CSRC, "-j8"], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    return LIB_PATH


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FlzError(-5, f"{LIB_PATH} is not built; run "
                               "`python -c 'import __graft_entry__ as g; g.build()'` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        for name, (res, args) in _SOLVER_SIGS.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def check(code: int):
    if code != FLZ_OK:
        raise FlzError(code, lib().flz_last_error().decode())


def exported_symbols():
    """Every symbol include/flz.h declares (used by the boundary test)."""
    return list(_SIGS) + list(_SOLVER_SIGS)
