"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes driver for oracle/_ref/libhkkt_ref.so: the UNMODIFIED reference
library (compiled from /root/reference/proj/core/src by oracle/Makefile)
plus the thin extern "C" shim oracle/ref_shim.cpp.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module, and only as the checker or the timed CPU baseline —
never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libhkkt_ref.so"
ORACLE_SO = HERE / "_ref" / "libhkkt_oracle.so"
REFERENCE_SRC = Path("/root/reference/proj")

I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)


class RefConfig(C.Structure):
    _fields_ = [("gamma", C.c_double), ("delta_min", C.c_double), ("delta_max", C.c_double),
                ("delta2", C.c_double), ("cg_tol", C.c_double), ("cg_max_iter", C.c_int64),
                ("small_quadratic_threshold", C.c_double), ("pivot_floor", C.c_double),
                ("ruiz_tol", C.c_double), ("ruiz_max_iters", C.c_int64)]


class RefSystem(C.Structure):
    _fields_ = [("n_x", C.c_int64), ("m_c", C.c_int64), ("m_d", C.c_int64),
                ("h_colptr", I64P), ("h_rowidx", I64P), ("h_val", F64P),
                ("j_colptr", I64P), ("j_rowidx", I64P), ("j_val", F64P),
                ("jd_colptr", I64P), ("jd_rowidx", I64P), ("jd_val", F64P),
                ("d_x", F64P), ("d_s", F64P), ("r_tilde_x", F64P), ("r_s", F64P),
                ("r_y", F64P), ("r_yd", F64P)]


class RefReport(C.Structure):
    _fields_ = [("status", C.c_int32), ("symbolic_reused", C.c_int32),
                ("delta1_final", C.c_double), ("delta2_used", C.c_double),
                ("cg_iterations", C.c_int64), ("factorization_attempts", C.c_int64),
                ("be_4x4", C.c_double), ("rr_4x4", C.c_double), ("be_2x2", C.c_double),
                ("rr_2x2", C.c_double), ("be_2x2_scaled", C.c_double),
                ("rr_2x2_scaled", C.c_double), ("ruiz_iterations", C.c_int64),
                ("nnz_op", C.c_int64), ("nnz_fac", C.c_int64), ("density_ratio", C.c_double),
                ("rho_c", C.c_double)]


def build(quiet: bool = True) -> bool:
    """Build oracle/_ref from the reference sources (only where
    /root/reference exists — on the GPU box the prebuilt .so is used)."""
    if not REFERENCE_SRC.exists():
        return REF_SO.exists()
    r = subprocess.run(["make", "-C", str(HERE), "-j8", "all"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + r.stdout[-2000:] + r.stderr[-4000:])
    return True


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not REF_SO.exists():
        build()
    L = C.CDLL(str(REF_SO))
    vp = C.c_void_p
    L.ref_last_error.restype = C.c_char_p
    L.ref_solve_full.argtypes = [C.POINTER(RefSystem), C.POINTER(RefConfig), I64P, F64P,
                                 C.POINTER(RefReport), F64P, F64P, F64P, F64P]
    L.ref_hgamma_amd.argtypes = [C.POINTER(RefSystem), C.POINTER(RefConfig), I64P]
    L.ref_assemble.argtypes = [C.POINTER(RefSystem), C.POINTER(RefConfig), I64P, I64P, I64P,
                               F64P, F64P, F64P, I64P, F64P, F64P]
    L.ref_pattern_stats.argtypes = [C.POINTER(RefSystem), C.POINTER(RefConfig), I64P, I64P]
    L.ref_time_phases.argtypes = [C.POINTER(RefSystem), C.POINTER(RefConfig), I64P, C.c_int,
                                  F64P, I64P]
    L.ref_batch_new.argtypes = [C.c_int64, C.POINTER(RefSystem)]
    L.ref_batch_new.restype = vp
    L.ref_batch_free.argtypes = [vp]
    L.ref_batch_free.restype = None
    L.ref_batch_run.argtypes = [vp, C.POINTER(RefConfig), I64P, C.c_int64, C.c_int64, C.c_int,
                                F64P, I64P, I32P]
    L.ref_chol_new.argtypes = [C.c_int64, I64P, I64P, F64P, I64P, C.c_double, I64P, F64P, I64P]
    L.ref_chol_new.restype = vp
    L.ref_chol_get.argtypes = [vp, I64P, I64P, I64P, I64P, F64P]
    L.ref_chol_solve.argtypes = [vp, F64P, F64P]
    L.ref_chol_free.argtypes = [vp]
    L.ref_chol_free.restype = None
    L.ref_ladder.argtypes = [C.c_int64, I64P, I64P, F64P, I64P, C.POINTER(RefConfig), F64P,
                             I32P, I64P, F64P, I64P]
    L.ref_gen_new.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                              C.c_double, C.c_uint64]
    L.ref_gen_new.restype = vp
    L.ref_gen_free.argtypes = [vp]
    L.ref_gen_free.restype = None
    L.ref_gen_dims.argtypes = [vp, C.c_int64, I64P]
    L.ref_gen_get.argtypes = [vp, C.c_int64] + [I64P, I64P, F64P] * 3 + [F64P] * 6
    L.ref_cg_schur.argtypes = [C.c_int64, I64P, I64P, F64P, C.c_int64, I64P, I64P, F64P, I64P,
                               C.POINTER(RefConfig), C.c_double, F64P, F64P, I64P, F64P, I32P]
    L.ref_reduce.argtypes = [C.POINTER(RefSystem), I64P, I64P, I64P, F64P, F64P]
    L.ref_solve_reduced.argtypes = [C.c_int64, C.c_int64, I64P, I64P, F64P, I64P, I64P, F64P, F64P,
                                    F64P, C.POINTER(RefConfig), I64P, F64P, C.POINTER(RefReport),
                                    F64P, F64P]
    L.ref_solve_sequence.argtypes = [C.c_int64, C.POINTER(RefSystem), C.POINTER(RefConfig),
                                     C.POINTER(RefReport), F64P, I64P]
    _lib = L
    return L


def _chk(code):
    if code != 0:
        raise RuntimeError("reference error: " + lib().ref_last_error().decode())


def _ip(a):
    return None if a is None else np.ascontiguousarray(a, np.int64).ctypes.data_as(I64P)


def _dp(a):
    return None if a is None else a.ctypes.data_as(F64P)


def config(cfg=None) -> RefConfig:
    """RefConfig from any object with SolverConfig attribute names."""
    c = RefConfig(1e4, 1e-9, 1e-6, 1e-9, 1e-12, 500, 1e-12, 1e-13, 0.01, 20)
    if cfg is not None:
        for name, _ in RefConfig._fields_:
            if hasattr(cfg, name):
                setattr(c, name, getattr(cfg, name))
    return c


class _SysHolder:
    """Keeps the numpy buffers alive while the reference reads them."""

    def __init__(self, sys):
        f = lambda a: np.ascontiguousarray(a, np.float64)
        i = lambda a: np.ascontiguousarray(a, np.int64)
        self.keep = [i(sys.h.colptr), i(sys.h.rowidx), f(sys.h.values),
                     i(sys.j.colptr), i(sys.j.rowidx), f(sys.j.values),
                     i(sys.j_d.colptr), i(sys.j_d.rowidx), f(sys.j_d.values),
                     f(sys.d_x), f(sys.d_s), f(sys.r_tilde_x), f(sys.r_s), f(sys.r_y), f(sys.r_yd)]
        k = self.keep
        self.s = RefSystem(sys.n_x, sys.m_c, sys.m_d,
                           k[0].ctypes.data_as(I64P), k[1].ctypes.data_as(I64P), k[2].ctypes.data_as(F64P),
                           k[3].ctypes.data_as(I64P), k[4].ctypes.data_as(I64P), k[5].ctypes.data_as(F64P),
                           k[6].ctypes.data_as(I64P), k[7].ctypes.data_as(I64P), k[8].ctypes.data_as(F64P),
                           *[a.ctypes.data_as(F64P) for a in k[9:]])


@dataclass
class RefSolve:
    report: dict
    dx: np.ndarray
    ds: np.ndarray
    dy: np.ndarray
    dyd: np.ndarray
    delta_min_current: float

    def stacked(self):
        return np.concatenate([self.dx, self.ds, self.dy, self.dyd])


def solve_full(sys, cfg=None, perm=None, delta_min_current: float = 0.0) -> RefSolve:
    """hkkt::solve_full (solver.cpp:295-328).  perm=None: reference AMD."""
    L = lib()
    h = _SysHolder(sys)
    rc = config(cfg)
    rep = RefReport()
    dm = C.c_double(delta_min_current)
    dx, ds = np.zeros(sys.n_x), np.zeros(sys.m_d)
    dy, dyd = np.zeros(sys.m_c), np.zeros(sys.m_d)
    p = None if perm is None else np.ascontiguousarray(perm, np.int64)
    _chk(L.ref_solve_full(C.byref(h.s), C.byref(rc), _ip(p), C.byref(dm), C.byref(rep),
                          _dp(dx), _dp(ds), _dp(dy), _dp(dyd)))
    r = {name: getattr(rep, name) for name, _ in RefReport._fields_}
    return RefSolve(r, dx, ds, dy, dyd, dm.value)


def hgamma_amd(sys, cfg=None) -> np.ndarray:
    """amd_order of the H_gamma pattern that solve_reduced factors."""
    h = _SysHolder(sys)
    rc = config(cfg)
    perm = np.zeros(sys.n_x, np.int64)
    _chk(lib().ref_hgamma_amd(C.byref(h.s), C.byref(rc), perm.ctypes.data_as(I64P)))
    return perm


def assemble(sys, cfg=None) -> dict:
    """reduce -> ruiz_scale -> assemble_h_gamma outputs."""
    L = lib()
    h = _SysHolder(sys)
    rc = config(cfg)
    nnz = C.c_int64(0)
    _chk(L.ref_assemble(C.byref(h.s), C.byref(rc), C.byref(nnz), None, None, None, None, None,
                        None, None, None))
    n = sys.n_x
    cp = np.zeros(n + 1, np.int64)
    ri = np.zeros(nnz.value, np.int64)
    v = np.zeros(nnz.value)
    rhat = np.zeros(n)
    d = np.zeros(n + sys.m_c)
    it = C.c_int64(0)
    js = np.zeros(sys.j.nnz)
    _chk(L.ref_assemble(C.byref(h.s), C.byref(rc), C.byref(nnz), cp.ctypes.data_as(I64P),
                        ri.ctypes.data_as(I64P), _dp(v), _dp(rhat), _dp(d), C.byref(it), None,
                        _dp(js)))
    return dict(colptr=cp, rowidx=ri, values=v, r_hat_x=rhat, d=d, ruiz_iterations=it.value,
                j_scaled=js)


def pattern_stats(sys, cfg=None, perm=None) -> dict:
    h = _SysHolder(sys)
    rc = config(cfg)
    out = np.zeros(4, np.int64)
    p = None if perm is None else np.ascontiguousarray(perm, np.int64)
    _chk(lib().ref_pattern_stats(C.byref(h.s), C.byref(rc), _ip(p), out.ctypes.data_as(I64P)))
    return dict(nnz_h_tilde=int(out[0]), nnz_h_gamma=int(out[1]), nnz_l=int(out[2]),
                etree_height=int(out[3]))


def time_phases(sys, cfg=None, perm=None, reps: int = 3):
    """(assembly_s, factor_s, cg_s, cg_iterations), median of reps, 1 thread."""
    h = _SysHolder(sys)
    rc = config(cfg)
    out = np.zeros(3)
    it = C.c_int64(0)
    p = None if perm is None else np.ascontiguousarray(perm, np.int64)
    _chk(lib().ref_time_phases(C.byref(h.s), C.byref(rc), _ip(p), reps, _dp(out), C.byref(it)))
    return float(out[0]), float(out[1]), float(out[2]), int(it.value)


class Batch:
    """Prebuilt reference systems for the std::thread throughput baseline."""

    def __init__(self, systems):
        self.holders = [_SysHolder(s) for s in systems]
        arr = (RefSystem * len(systems))(*[h.s for h in self.holders])
        self.h = lib().ref_batch_new(len(systems), arr)
        if not self.h:
            _chk(-1)
        self.n = len(systems)

    def run(self, cfg=None, perm=None, first=0, count=None, threads=None):
        count = self.n - first if count is None else count
        threads = threads or os.cpu_count() or 1
        sec = C.c_double(0)
        its = np.zeros(count, np.int64)
        st = np.zeros(count, np.int32)
        rc = config(cfg)
        p = None if perm is None else np.ascontiguousarray(perm, np.int64)
        _chk(lib().ref_batch_run(self.h, C.byref(rc), _ip(p), first, count, threads,
                                 C.byref(sec), its.ctypes.data_as(I64P), st.ctypes.data_as(I32P)))
        return sec.value, its, st

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_batch_free(self.h)
            self.h = None


def numeric_cholesky(a, perm=None, floor: float = 0.0) -> dict:
    """symbolic_cholesky + numeric_cholesky on a lower CSC matrix."""
    L = lib()
    cp = np.ascontiguousarray(a.colptr, np.int64)
    ri = np.ascontiguousarray(a.rowidx, np.int64)
    v = np.ascontiguousarray(a.values, np.float64)
    fc, fp, lnnz = C.c_int64(0), C.c_double(0), C.c_int64(0)
    p = None if perm is None else np.ascontiguousarray(perm, np.int64)
    hnd = L.ref_chol_new(a.ncols, cp.ctypes.data_as(I64P), ri.ctypes.data_as(I64P), _dp(v), _ip(p),
                         floor, C.byref(fc), C.byref(fp), C.byref(lnnz))
    if not hnd:
        _chk(-1)
    n = a.ncols
    out = dict(failed_column=int(fc.value), failed_pivot=float(fp.value))
    permo = np.zeros(n, np.int64)
    parent = np.zeros(n, np.int64)
    lcp = np.zeros(n + 1, np.int64)
    lri = np.zeros(lnnz.value, np.int64)
    lv = np.zeros(lnnz.value) if fc.value < 0 else None
    _chk(L.ref_chol_get(hnd, permo.ctypes.data_as(I64P), parent.ctypes.data_as(I64P),
                        lcp.ctypes.data_as(I64P), lri.ctypes.data_as(I64P), _dp(lv)))
    out.update(perm=permo, parent=parent, l_colptr=lcp, l_rowidx=lri, l_values=lv, handle=hnd)
    return out


def factor_solve(chol: dict, b) -> np.ndarray:
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros_like(b)
    _chk(lib().ref_chol_solve(chol["handle"], _dp(b), _dp(x)))
    return x


def free_chol(chol: dict) -> None:
    if chol.get("handle"):
        lib().ref_chol_free(chol["handle"])
        chol["handle"] = None


def ladder(h_gamma, cfg=None, perm=None, delta_min_current: float = 0.0) -> dict:
    """factorize_with_ladder on an explicit lower H_gamma."""
    rc = config(cfg)
    dm = C.c_double(delta_min_current)
    ok, att, d1, fcol = C.c_int32(0), C.c_int64(0), C.c_double(0), C.c_int64(0)
    p = None if perm is None else np.ascontiguousarray(perm, np.int64)
    _chk(lib().ref_ladder(h_gamma.ncols, _ip(h_gamma.colptr), _ip(h_gamma.rowidx),
                          _dp(np.ascontiguousarray(h_gamma.values, np.float64)), _ip(p),
                          C.byref(rc), C.byref(dm), C.byref(ok), C.byref(att), C.byref(d1),
                          C.byref(fcol)))
    return dict(ok=bool(ok.value), attempts=att.value, delta1=d1.value, failed_column=fcol.value,
                delta_min_current=dm.value)


def generate(n_x, m_c, m_d, degree=4, klass=0, length=1, drift=0.01, seed=1):
    """Reference generator (generator.cpp:289-406) -> list of BlockKkt4x4."""
    from paper_2110_03636_b200.kkt import BlockKkt4x4, CscMatrix
    L = lib()
    hnd = L.ref_gen_new(n_x, m_c, m_d, degree, klass, length, drift, seed)
    if not hnd:
        _chk(-1)
    out = []
    try:
        for k in range(length):
            dims = np.zeros(6, np.int64)
            _chk(L.ref_gen_dims(hnd, k, dims.ctypes.data_as(I64P)))
            nx, mc, md, nh, nj, njd = map(int, dims)
            arrs = dict(h_cp=np.zeros(nx + 1, np.int64), h_ri=np.zeros(nh, np.int64), h_v=np.zeros(nh),
                        j_cp=np.zeros(nx + 1, np.int64), j_ri=np.zeros(nj, np.int64), j_v=np.zeros(nj),
                        jd_cp=np.zeros(nx + 1, np.int64), jd_ri=np.zeros(njd, np.int64),
                        jd_v=np.zeros(njd), d_x=np.zeros(nx), d_s=np.zeros(md), rtx=np.zeros(nx),
                        r_s=np.zeros(md), r_y=np.zeros(mc), r_yd=np.zeros(md))
            ptrs = [a.ctypes.data_as(I64P if a.dtype == np.int64 else F64P) for a in arrs.values()]
            _chk(L.ref_gen_get(hnd, k, *ptrs))
            a = arrs
            out.append(BlockKkt4x4(
                h=CscMatrix(nx, nx, a["h_cp"], a["h_ri"], a["h_v"]),
                j=CscMatrix(mc, nx, a["j_cp"], a["j_ri"], a["j_v"]),
                j_d=CscMatrix(md, nx, a["jd_cp"], a["jd_ri"], a["jd_v"]),
                d_x=a["d_x"], d_s=a["d_s"], r_tilde_x=a["rtx"], r_s=a["r_s"], r_y=a["r_y"],
                r_yd=a["r_yd"]))
    finally:
        L.ref_gen_free(hnd)
    return out


def cg_schur(h_lower, j, rhs, cfg=None, perm=None, delta2=0.0) -> dict:
    rc = config(cfg)
    rhs = np.ascontiguousarray(rhs, np.float64)
    x = np.zeros_like(rhs)
    it, rr, fl = C.c_int64(0), C.c_double(0), C.c_int32(0)
    p = None if perm is None else np.ascontiguousarray(perm, np.int64)
    _chk(lib().ref_cg_schur(h_lower.ncols, _ip(h_lower.colptr), _ip(h_lower.rowidx),
                            _dp(np.ascontiguousarray(h_lower.values, np.float64)), j.nrows,
                            _ip(j.colptr), _ip(j.rowidx), _dp(np.ascontiguousarray(j.values, np.float64)),
                            _ip(p), C.byref(rc), delta2, _dp(rhs), _dp(x), C.byref(it), C.byref(rr),
                            C.byref(fl)))
    return dict(x=x, iterations=it.value, relative_residual=rr.value,
                converged=bool(fl.value & 1), small_quadratic=bool(fl.value & 2))


def reduce(sys):
    """hkkt::reduce (kkt_system.cpp:66-87) -> Reduced2x2."""
    from paper_2110_03636_b200.kkt import CscMatrix, Reduced2x2
    L = lib()
    h = _SysHolder(sys)
    nnz = C.c_int64(0)
    _chk(L.ref_reduce(C.byref(h.s), C.byref(nnz), None, None, None, None))
    n = sys.n_x
    cp, ri, v, rx = np.zeros(n + 1, np.int64), np.zeros(nnz.value, np.int64), np.zeros(nnz.value), np.zeros(n)
    _chk(L.ref_reduce(C.byref(h.s), C.byref(nnz), _ip(cp), _ip(ri), _dp(v), _dp(rx)))
    return Reduced2x2(CscMatrix(n, n, cp, ri, v), sys.j, rx, np.array(sys.r_y, np.float64))


def solve_reduced(red, cfg=None, perm=None, delta_min_current: float = 0.0) -> dict:
    """hkkt::solve_reduced (solver.cpp:222-293).  perm=None: reference AMD."""
    rc = config(cfg)
    rep = RefReport()
    dm = C.c_double(delta_min_current)
    f = lambda a: np.ascontiguousarray(a, np.float64)
    i = lambda a: np.ascontiguousarray(a, np.int64)
    keep = [i(red.h_tilde.colptr), i(red.h_tilde.rowidx), f(red.h_tilde.values), i(red.j.colptr),
            i(red.j.rowidx), f(red.j.values), f(red.r_x), f(red.r_y)]
    dx, dy = np.zeros(red.n_x), np.zeros(red.m_c)
    p = None if perm is None else i(perm)
    _chk(lib().ref_solve_reduced(red.n_x, red.m_c, _ip(keep[0]), _ip(keep[1]), _dp(keep[2]), _ip(keep[3]),
                                 _ip(keep[4]), _dp(keep[5]), _dp(keep[6]), _dp(keep[7]), C.byref(rc), _ip(p),
                                 C.byref(dm), C.byref(rep), _dp(dx), _dp(dy)))
    r = {name: getattr(rep, name) for name, _ in RefReport._fields_}
    return dict(report=r, dx=dx, dy=dy, delta_min_current=dm.value)


def solve_sequence(systems, cfg=None) -> dict:
    """hkkt::solve_sequence (solver.cpp:352-412), sequential mode."""
    rc = config(cfg)
    holders = [_SysHolder(s) for s in systems]
    arr = (RefSystem * len(systems))(*[h.s for h in holders])
    reps = (RefReport * len(systems))()
    N = systems[0].total_size
    sols = np.zeros(len(systems) * N)
    stats = np.zeros(4, np.int64)
    _chk(lib().ref_solve_sequence(len(systems), arr, C.byref(rc), reps, _dp(sols), _ip(stats)))
    return dict(reports=[{name: getattr(r, name) for name, _ in RefReport._fields_} for r in reps],
                solutions=sols.reshape(len(systems), N),
                stats=dict(symbolic_analyses=int(stats[0]), numeric_factorizations=int(stats[1]),
                           factorization_attempts=int(stats[2]), pattern_uniform=bool(stats[3])))
