"""ORACLE / TEST INFRASTRUCTURE ONLY: ctypes driver of the plain-C
restatement (oracle/hykkt_oracle.c -> oracle/_ref/libhkkt_oracle.so).

Used by tests/ to pin the restatement bit-for-bit against the compiled
reference, and as a second, independently written checker."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import ref as _ref

SO = Path(__file__).resolve().parent / "_ref" / "libhkkt_oracle.so"
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)


class OConfig(C.Structure):
    _fields_ = _ref.RefConfig._fields_


class OReport(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_int32), ("delta1_final", C.c_double),
                ("delta2_used", C.c_double), ("cg_iterations", C.c_int64),
                ("factorization_attempts", C.c_int64), ("ruiz_iterations", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not SO.exists():
            _ref.build()
        L = C.CDLL(str(SO))
        L.oracle_solve_full.argtypes = ([C.c_int64] * 3 + [I64P, I64P, F64P] * 3 + [F64P] * 6 +
                                        [I64P, C.POINTER(OConfig), F64P, C.POINTER(OReport)] + [F64P] * 4)
        L.oracle_solve_full.restype = C.c_int
        L.oracle_cholesky.argtypes = [C.c_int64, I64P, I64P, F64P, I64P, C.c_double, I64P, F64P, C.c_int64,
                                      F64P, F64P, F64P]
        L.oracle_cholesky.restype = C.c_int64
        _lib = L
    return _lib


def _i(a):
    return np.ascontiguousarray(a, np.int64)


def _f(a):
    return np.ascontiguousarray(a, np.float64)


def solve_full(sys, cfg, perm, delta_min_current: float = 0.0):
    rc = _ref.config(cfg)
    oc = OConfig(*[getattr(rc, n) for n, _ in OConfig._fields_])
    keep = [_i(sys.h.colptr), _i(sys.h.rowidx), _f(sys.h.values), _i(sys.j.colptr), _i(sys.j.rowidx),
            _f(sys.j.values), _i(sys.j_d.colptr), _i(sys.j_d.rowidx), _f(sys.j_d.values),
            _f(sys.d_x), _f(sys.d_s), _f(sys.r_tilde_x), _f(sys.r_s), _f(sys.r_y), _f(sys.r_yd), _i(perm)]
    ptrs = [a.ctypes.data_as(I64P if a.dtype == np.int64 else F64P) for a in keep]
    rep = OReport()
    dm = C.c_double(delta_min_current)
    dx, ds, dy, dyd = np.zeros(sys.n_x), np.zeros(sys.m_d), np.zeros(sys.m_c), np.zeros(sys.m_d)
    lib().oracle_solve_full(sys.n_x, sys.m_c, sys.m_d, *ptrs[:15], ptrs[15], C.byref(oc), C.byref(dm),
                            C.byref(rep), *[a.ctypes.data_as(F64P) for a in (dx, ds, dy, dyd)])
    r = {n: getattr(rep, n) for n, _ in OReport._fields_ if n != "pad"}
    return r, dx, ds, dy, dyd, dm.value


def cholesky(a, perm, floor_abs=0.0, b=None):
    n = a.ncols
    cp, ri, v, p = _i(a.colptr), _i(a.rowidx), _f(a.values), _i(perm)
    lnnz = C.c_int64(0)
    fp = C.c_double(0.0)
    lib().oracle_cholesky(n, cp.ctypes.data_as(I64P), ri.ctypes.data_as(I64P), v.ctypes.data_as(F64P),
                          p.ctypes.data_as(I64P), floor_abs, C.byref(lnnz), None, 0, C.byref(fp), None, None)
    lv = np.zeros(lnnz.value)
    bb = _f(b) if b is not None else None
    x = np.zeros(n) if b is not None else None
    failed = lib().oracle_cholesky(n, cp.ctypes.data_as(I64P), ri.ctypes.data_as(I64P), v.ctypes.data_as(F64P),
                                   p.ctypes.data_as(I64P), floor_abs, C.byref(lnnz), lv.ctypes.data_as(F64P),
                                   lnnz.value, C.byref(fp),
                                   None if bb is None else bb.ctypes.data_as(F64P),
                                   None if x is None else x.ctypes.data_as(F64P))
    return dict(failed_column=int(failed), failed_pivot=fp.value, l_values=lv, x=x)
