"""ctypes binding of libhykkt.so (the C ABI in include/hykkt.h).

The product path has no CPU fallback: if the CUDA library is missing or a
call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libhykkt.so"

I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)


class Config(C.Structure):
    _fields_ = [
        ("gamma", C.c_double),
        ("delta_min", C.c_double),
        ("delta_max", C.c_double),
        ("delta2", C.c_double),
        ("cg_tol", C.c_double),
        ("cg_max_iter", C.c_int64),
        ("small_quadratic_threshold", C.c_double),
        ("pivot_floor", C.c_double),
        ("ruiz_tol", C.c_double),
        ("ruiz_max_iters", C.c_int64),
    ]


class Values(C.Structure):
    _fields_ = [(n, F64P) for n in ("h_val", "j_val", "jd_val", "d_x", "d_s",
                                    "r_tilde_x", "r_s", "r_y", "r_yd")]


class Report(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("symbolic_reused", C.c_int32),
        ("delta1_final", C.c_double),
        ("delta2_used", C.c_double),
        ("cg_iterations", C.c_int64),
        ("factorization_attempts", C.c_int64),
        ("be_4x4", C.c_double), ("rr_4x4", C.c_double),
        ("be_2x2", C.c_double), ("rr_2x2", C.c_double),
        ("be_2x2_scaled", C.c_double), ("rr_2x2_scaled", C.c_double),
        ("ruiz_iterations", C.c_int64),
        ("nnz_op", C.c_int64), ("nnz_fac", C.c_int64),
        ("density_ratio", C.c_double), ("rho_c", C.c_double),
        ("cg_relative_residual", C.c_double),
        ("failed_column", C.c_int64),
    ]


class Analysis(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("nnz_h_tilde", C.c_int64), ("nnz_h_gamma", C.c_int64),
        ("nnz_l", C.c_int64), ("n_supernodes", C.c_int64), ("n_levels", C.c_int64),
        ("etree_height", C.c_int64), ("max_sn_width", C.c_int64), ("max_sn_rows", C.c_int64),
        ("panel_slots", C.c_int64), ("factor_flops", C.c_double),
        ("nnz_j", C.c_int64), ("nnz_jd", C.c_int64), ("m_c", C.c_int64), ("m_d", C.c_int64),
        ("explicit_zeros", C.c_int64),
    ]


class Timing(C.Structure):
    _fields_ = [
        ("assemble_ms", C.c_double), ("factor_ms", C.c_double), ("solve_w_ms", C.c_double),
        ("cg_ms", C.c_double), ("solve_dx_ms", C.c_double), ("total_ms", C.c_double),
        ("kernel_launches", C.c_int64), ("cg_kernel_launches", C.c_int64),
    ]


FLAG_METRICS = 1
FLAG_TIMING = 2

# Every symbol include/hykkt.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "hykkt_config_default", "hykkt_last_error", "hykkt_create", "hykkt_destroy",
    "hykkt_analyze", "hykkt_analysis_info", "hykkt_host_analyze", "hykkt_get_perm", "hykkt_solve_full",
    "hykkt_upload_values", "hykkt_solve_resident", "hykkt_download_solution",
    "hykkt_last_timing", "hykkt_chol_analyze", "hykkt_chol_factor", "hykkt_chol_solve",
    "hykkt_chol_get_factor", "hykkt_batch_solve", "hykkt_batch_upload",
    "hykkt_batch_solve_resident", "hykkt_batch_download",
    "hykkt_upload_values_device", "hykkt_batch_upload_device", "hykkt_solution_device",
    "hykkt_batch_solution_device", "hykkt_analyze_reduced", "hykkt_upload_reduced",
    "hykkt_upload_reduced_device", "hykkt_solve_reduced", "hykkt_assemble", "hykkt_hgamma_pattern",
    "hykkt_factor_ladder", "hykkt_chol_set_factor", "hykkt_chol_set_j", "hykkt_cg_schur",
    "hykkt_set_option", "hykkt_batch_upload_async", "hykkt_batch_download_async", "hykkt_batch_sync",
]


class HykktError(RuntimeError):
    """A non-zero status from the C ABI (the reference raises
    InvalidMatrixError for the argument class, csc_matrix.hpp:29-33)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"hykkt error {code}: {msg}")
        self.code = code


class InvalidMatrixError(HykktError, ValueError):
    pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(str(LIB_PATH))
    vp = C.c_void_p
    L.hykkt_last_error.restype = C.c_char_p
    L.hykkt_config_default.argtypes = [C.POINTER(Config)]
    L.hykkt_config_default.restype = None
    L.hykkt_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.hykkt_destroy.argtypes = [vp]
    L.hykkt_destroy.restype = None
    L.hykkt_analyze.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, I64P, I64P, I64P, I64P,
                                I64P, I64P, I64P]
    L.hykkt_analysis_info.argtypes = [vp, C.POINTER(Analysis)]
    L.hykkt_get_perm.argtypes = [vp, I64P]
    L.hykkt_host_analyze.argtypes = [C.c_int64, C.c_int64, C.c_int64, I64P, I64P, I64P, I64P,
                                     I64P, I64P, I64P, I64P, C.POINTER(Analysis)]
    L.hykkt_solve_full.argtypes = [vp, C.POINTER(Config), C.POINTER(Values), F64P, C.c_int,
                                   C.POINTER(Report), F64P, F64P, F64P, F64P]
    L.hykkt_upload_values.argtypes = [vp, C.POINTER(Values)]
    L.hykkt_solve_resident.argtypes = [vp, C.POINTER(Config), F64P, C.c_int, C.POINTER(Report)]
    L.hykkt_download_solution.argtypes = [vp, F64P, F64P, F64P, F64P]
    L.hykkt_last_timing.argtypes = [vp, C.POINTER(Timing)]
    L.hykkt_chol_analyze.argtypes = [vp, C.c_int64, I64P, I64P, I64P]
    L.hykkt_chol_factor.argtypes = [vp, F64P, C.c_double, I64P, F64P]
    L.hykkt_chol_solve.argtypes = [vp, F64P, F64P]
    L.hykkt_chol_get_factor.argtypes = [vp, I64P, I64P, F64P, I64P]
    L.hykkt_batch_solve.argtypes = [vp, C.POINTER(Config), C.c_int64, C.POINTER(Values), C.c_int,
                                    C.POINTER(Report), F64P, F64P, F64P, F64P]
    L.hykkt_batch_upload.argtypes = [vp, C.c_int64, C.POINTER(Values)]
    L.hykkt_batch_solve_resident.argtypes = [vp, C.POINTER(Config), C.c_int, C.POINTER(Report)]
    L.hykkt_batch_download.argtypes = [vp, F64P, F64P, F64P, F64P]
    L.hykkt_batch_upload_async.argtypes = [vp, C.c_int64, C.POINTER(Values)]
    L.hykkt_batch_download_async.argtypes = [vp, F64P, F64P, F64P, F64P]
    L.hykkt_batch_sync.argtypes = [vp]
    VPP = C.POINTER(C.c_void_p)
    I32P = C.POINTER(C.c_int32)
    L.hykkt_upload_values_device.argtypes = [vp, C.POINTER(Values)]
    L.hykkt_batch_upload_device.argtypes = [vp, C.c_int64, C.POINTER(Values)]
    L.hykkt_solution_device.argtypes = [vp, VPP, VPP, VPP, VPP]
    L.hykkt_batch_solution_device.argtypes = [vp, VPP, VPP, VPP, VPP]
    L.hykkt_analyze_reduced.argtypes = [vp, C.c_int64, C.c_int64, I64P, I64P, I64P, I64P, I64P]
    L.hykkt_upload_reduced.argtypes = [vp, F64P, F64P, F64P, F64P]
    L.hykkt_upload_reduced_device.argtypes = [vp, vp, vp, vp, vp]
    L.hykkt_solve_reduced.argtypes = [vp, C.POINTER(Config), F64P, F64P, F64P, F64P, F64P, C.c_int,
                                      C.POINTER(Report), F64P, F64P]
    L.hykkt_assemble.argtypes = [vp, C.POINTER(Config), F64P, F64P]
    L.hykkt_hgamma_pattern.argtypes = [vp, I64P, I64P]
    L.hykkt_factor_ladder.argtypes = [vp, C.POINTER(Config), F64P, F64P, I64P, F64P, I64P]
    L.hykkt_chol_set_factor.argtypes = [vp, F64P]
    L.hykkt_chol_set_j.argtypes = [vp, C.c_int64, I64P, I64P, F64P]
    L.hykkt_cg_schur.argtypes = [vp, C.POINTER(Config), F64P, C.c_double, F64P, I64P, F64P, I32P, I32P]
    L.hykkt_set_option.argtypes = [vp, C.c_char_p, C.c_int64]
    for name in EXPORTS:
        fn = getattr(L, name)
        if name not in ("hykkt_last_error", "hykkt_destroy", "hykkt_config_default"):
            fn.restype = C.c_int
    _lib = L
    return L


def check(code: int) -> None:
    if code != 0:
        msg = lib().hykkt_last_error().decode(errors="replace")
        if code == -1:
            raise InvalidMatrixError(code, msg)
        raise HykktError(code, msg)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def ip(a):
    return None if a is None else a.ctypes.data_as(I64P)


def dp(a):
    return None if a is None else a.ctypes.data_as(F64P)
