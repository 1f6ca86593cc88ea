"""Host-side mirror of the reference solver API over the B200 C ABI.

Names, argument meaning, defaults and outcomes follow
/root/reference/proj/core/include/hkkt/solver.hpp and cholesky.hpp:

  SolverConfig / RegularizationState / SolveStatus / SolveReport   solver.hpp:29-150
  solve_full / solve_sequence / SequenceResult                     solver.hpp:172-205
  solve_reduced / ReducedSolveResult                               solver.hpp:152-170
  assemble_h_gamma / factorize_with_ladder / LadderFailure          solver.hpp:75-94
  cg_schur / CgResult                                              solver.hpp:110-122
  symbolic_cholesky / numeric_cholesky / factor_solve              cholesky.hpp:41-83
  NotSpdFailure                                                    cholesky.hpp:47-50

Every numeric step runs in libhykkt.so on the GPU; there is no CPU fallback
(a missing library or a CUDA failure raises).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field, fields
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, dp, f64, i64, ip
from .kkt import BlockKkt4x4, CscMatrix, FullSolution, HGammaSystem, Reduced2x2


@dataclass
class SolverConfig:
    gamma: float = 1e4
    delta_min: float = 1e-9
    delta_max: float = 1e-6
    delta2: float = 1e-9
    cg_tol: float = 1e-12
    cg_max_iter: int = 500
    small_quadratic_threshold: float = 1e-12
    pivot_floor: float = 1e-13
    ruiz_tol: float = 0.01
    ruiz_max_iters: int = 20

    def c(self) -> _lib.Config:
        return _lib.Config(*[getattr(self, f.name) for f in fields(self)])


class SolveStatus(enum.IntEnum):
    kSolved = 0
    kSolvedWithDelta2 = 1
    kFailedDeltaMaxExceeded = 2
    kFailedCgNoConvergence = 3


def is_success(s) -> bool:
    return SolveStatus(s) in (SolveStatus.kSolved, SolveStatus.kSolvedWithDelta2)


@dataclass
class RegularizationState:
    delta1: float = 0.0
    delta_min_current: float = 0.0
    attempts: int = 0

    @staticmethod
    def initial(cfg: SolverConfig) -> "RegularizationState":
        return RegularizationState(0.0, cfg.delta_min, 0)


@dataclass
class SolveReport:
    status: SolveStatus = SolveStatus.kSolved
    delta1_final: float = 0.0
    delta2_used: float = 0.0
    cg_iterations: int = 0
    factorization_attempts: int = 0
    be_4x4: float = 0.0
    rr_4x4: float = 0.0
    be_2x2: float = 0.0
    rr_2x2: float = 0.0
    be_2x2_scaled: float = 0.0
    rr_2x2_scaled: float = 0.0
    symbolic_reused: bool = False
    nnz_op: int = 0
    nnz_fac: int = 0
    density_ratio: float = 0.0
    rho_c: float = 0.0
    ruiz_iterations: int = 0
    cg_relative_residual: float = 0.0
    failure_detail: str = ""

    @staticmethod
    def from_c(r: _lib.Report) -> "SolveReport":
        rep = SolveReport(
            status=SolveStatus(r.status), delta1_final=r.delta1_final, delta2_used=r.delta2_used,
            cg_iterations=r.cg_iterations, factorization_attempts=r.factorization_attempts,
            be_4x4=r.be_4x4, rr_4x4=r.rr_4x4, be_2x2=r.be_2x2, rr_2x2=r.rr_2x2,
            be_2x2_scaled=r.be_2x2_scaled, rr_2x2_scaled=r.rr_2x2_scaled,
            symbolic_reused=bool(r.symbolic_reused), nnz_op=r.nnz_op, nnz_fac=r.nnz_fac,
            density_ratio=r.density_ratio, rho_c=r.rho_c, ruiz_iterations=r.ruiz_iterations,
            cg_relative_residual=r.cg_relative_residual)
        if rep.status == SolveStatus.kFailedDeltaMaxExceeded:
            rep.failure_detail = (f"factorization failed up to delta1 = {rep.delta1_final:f} "
                                  f"at column {r.failed_column}")
        elif rep.status == SolveStatus.kFailedCgNoConvergence:
            rep.failure_detail = f"CG stalled at relative residual {rep.cg_relative_residual:f}"
        return rep


@dataclass
class FullSolveResult:
    solution: Optional[FullSolution]
    report: SolveReport
    symbolic_created: bool = False


@dataclass
class SequenceStats:
    symbolic_analyses: int = 0
    numeric_factorizations: int = 0
    factorization_attempts: int = 0


@dataclass
class SequenceResult:
    reports: list = field(default_factory=list)
    solutions: list = field(default_factory=list)
    stats: SequenceStats = field(default_factory=SequenceStats)
    pattern_uniform: bool = True

    def all_successful(self) -> bool:
        return all(is_success(r.status) for r in self.reports)


@dataclass
class NotSpdFailure:
    column: int
    pivot: float


@dataclass
class LadderFailure:
    attempts: int
    last_delta1: float
    failed_column: int


@dataclass
class CgResult:
    x: np.ndarray
    iterations: int = 0
    relative_residual: float = 0.0
    converged: bool = False
    small_quadratic_detected: bool = False


@dataclass
class ReducedSolveResult:
    dx: Optional[np.ndarray]
    dy: Optional[np.ndarray]
    report: SolveReport
    symbolic_created: bool = False

    def ok(self) -> bool:
        return is_success(self.report.status)


def check_dims(sys: BlockKkt4x4) -> None:
    """BlockKkt4x4::validate (kkt_system.cpp:33-54), dimension part."""
    nx, mc, md = sys.n_x, sys.m_c, sys.m_d
    bad = None
    if sys.h.nrows != nx:
        bad = "H must be square"
    elif sys.j.ncols != nx:
        bad = "J column count must be n_x"
    elif sys.j_d.ncols != nx:
        bad = "J_d column count must be n_x"
    elif len(sys.d_x) != nx or len(sys.r_tilde_x) != nx:
        bad = "D_x and r_tilde_x must have length n_x"
    elif len(sys.d_s) != md or len(sys.r_s) != md or len(sys.r_yd) != md:
        bad = "D_s, r_s, r_yd must have length m_d"
    elif len(sys.r_y) != mc:
        bad = "r_y must have length m_c"
    elif (np.asarray(sys.d_x) < 0).any() or (np.asarray(sys.d_s) < 0).any() or not (
            np.isfinite(sys.d_x).all() and np.isfinite(sys.d_s).all()):
        bad = "D_x and D_s must be nonnegative and finite"
    if bad:
        raise _lib.InvalidMatrixError(-1, bad)


class Device:
    """One libhykkt handle: a device, a stream and one analysed pattern."""

    def __init__(self, device: int = 0):
        L = _lib.lib()
        h = C.c_void_p()
        check(L.hykkt_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self._pattern = None  # the BlockKkt4x4 whose pattern was analysed
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().hykkt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- analysis ----------------------------------------------------------
    def analyze(self, sys: BlockKkt4x4, perm=None) -> None:
        """Per-pattern half of solve_reduced (solver.cpp:230-235), once."""
        check_dims(sys)
        L = _lib.lib()
        a = [i64(x) for x in (sys.h.colptr, sys.h.rowidx, sys.j.colptr, sys.j.rowidx,
                              sys.j_d.colptr, sys.j_d.rowidx)]
        p = None if perm is None else i64(perm)
        check(L.hykkt_analyze(self.h, sys.n_x, sys.m_c, sys.m_d, *[ip(x) for x in a], ip(p)))
        self._pattern = sys

    def info(self) -> dict:
        a = _lib.Analysis()
        check(_lib.lib().hykkt_analysis_info(self.h, C.byref(a)))
        return {n: getattr(a, n) for n, _ in a._fields_}

    def perm(self) -> np.ndarray:
        n = self.info()["n"]
        out = np.zeros(n, np.int64)
        check(_lib.lib().hykkt_get_perm(self.h, ip(out)))
        return out

    def analyze_reduced(self, red: Reduced2x2, perm=None) -> None:
        """Per-pattern half of solve_reduced (solver.cpp:230-235) for a
        Reduced2x2 caller."""
        L = _lib.lib()
        a = [i64(x) for x in (red.h_tilde.colptr, red.h_tilde.rowidx, red.j.colptr, red.j.rowidx)]
        p = None if perm is None else i64(perm)
        check(L.hykkt_analyze_reduced(self.h, red.n_x, red.m_c, *[ip(x) for x in a], ip(p)))
        self._pattern = red

    def solve_reduced(self, red: Reduced2x2, cfg: SolverConfig | None = None,
                      state: RegularizationState | None = None,
                      metrics: bool = True) -> ReducedSolveResult:
        """hkkt::solve_reduced (solver.cpp:222-293): assemble H_gamma, ladder,
        w solve, CG with the delta2 restart, dx solve; no Ruiz, no recovery."""
        cfg = cfg or SolverConfig()
        created = False
        if not isinstance(self._pattern, Reduced2x2) or not self._pattern.same_pattern_as(red):
            self.analyze_reduced(red)
            created = True
        if state is None:
            state = RegularizationState.initial(cfg)
        arrs = [f64(x) for x in (red.h_tilde.values, red.j.values, red.r_x, red.r_y)]
        dx, dy = np.zeros(red.n_x), np.zeros(red.m_c)
        rep = _lib.Report()
        dm = C.c_double(state.delta_min_current)
        check(_lib.lib().hykkt_solve_reduced(self.h, C.byref(cfg.c()), *[dp(a) for a in arrs], C.byref(dm),
                                             _lib.FLAG_METRICS if metrics else 0, C.byref(rep), dp(dx),
                                             dp(dy)))
        state.delta_min_current = dm.value
        state.delta1 = rep.delta1_final
        state.attempts = rep.factorization_attempts
        report = SolveReport.from_c(rep)
        ok = is_success(report.status)
        return ReducedSolveResult(dx if ok else None, dy if ok else None, report, created)

    def assemble(self, cfg: SolverConfig | None = None) -> HGammaSystem:
        """assemble_h_gamma (solver.cpp:66-84) on the uploaded values (a
        reduced handle: the Reduced2x2 as given; a block-4x4 handle: the
        Ruiz-scaled reduction of the system)."""
        cfg = cfg or SolverConfig()
        info = self.info()
        n, nnz = info["n"], info["nnz_h_gamma"]
        cp, ri = np.zeros(n + 1, np.int64), np.zeros(nnz, np.int64)
        vals, rhat = np.zeros(nnz), np.zeros(n)
        L = _lib.lib()
        check(L.hykkt_assemble(self.h, C.byref(cfg.c()), dp(vals), dp(rhat)))
        check(L.hykkt_hgamma_pattern(self.h, ip(cp), ip(ri)))
        return HGammaSystem(CscMatrix(n, n, cp, ri, vals), rhat, cfg.gamma)

    def factorize_with_ladder(self, cfg: SolverConfig, state: RegularizationState):
        """factorize_with_ladder (solver.cpp:108-142) on the H_gamma of the
        last assemble(); returns None on success or a LadderFailure."""
        return _ladder(self.h, cfg, None, state)

    def upload_reduced(self, red: Reduced2x2) -> None:
        arrs = [f64(x) for x in (red.h_tilde.values, red.j.values, red.r_x, red.r_y)]
        self._keep = arrs
        check(_lib.lib().hykkt_upload_reduced(self.h, *[dp(a) for a in arrs]))

    def cg_schur(self, rhs, cfg: SolverConfig | None = None, delta2: float = 0.0) -> CgResult:
        return _cg_schur(self.h, rhs, cfg or SolverConfig(), delta2)

    def factor_solve(self, b) -> np.ndarray:
        b = f64(b)
        x = np.zeros(b.shape[0])
        check(_lib.lib().hykkt_chol_solve(self.h, dp(b), dp(x)))
        return x

    # ---- values ------------------------------------------------------------
    def _values(self, sys: BlockKkt4x4):
        arrs = [f64(x) for x in (sys.h.values, sys.j.values, sys.j_d.values, sys.d_x, sys.d_s,
                                 sys.r_tilde_x, sys.r_s, sys.r_y, sys.r_yd)]
        self._keep = arrs
        return _lib.Values(*[dp(x) for x in arrs])

    def upload(self, sys: BlockKkt4x4) -> None:
        v = self._values(sys)
        check(_lib.lib().hykkt_upload_values(self.h, C.byref(v)))

    def solve_resident(self, cfg: SolverConfig, state: RegularizationState | None = None,
                       metrics: bool = False, timing: bool = False) -> SolveReport:
        rep = _lib.Report()
        dm = C.c_double(state.delta_min_current if state else 0.0)
        flags = (_lib.FLAG_METRICS if metrics else 0) | (_lib.FLAG_TIMING if timing else 0)
        check(_lib.lib().hykkt_solve_resident(self.h, C.byref(cfg.c()), C.byref(dm), flags,
                                              C.byref(rep)))
        if state is not None:
            state.delta_min_current = dm.value
            state.delta1 = rep.delta1_final
            state.attempts = rep.factorization_attempts
        return SolveReport.from_c(rep)

    def download(self) -> FullSolution:
        s = self._pattern
        out = FullSolution(np.zeros(s.n_x), np.zeros(s.m_d), np.zeros(s.m_c), np.zeros(s.m_d))
        check(_lib.lib().hykkt_download_solution(self.h, dp(out.dx), dp(out.ds), dp(out.dy),
                                                 dp(out.dyd)))
        return out

    def set_option(self, name: str, value: int) -> None:
        """Scheduling knobs (hykkt_set_option), e.g. ("ks_lpt", 0)."""
        check(_lib.lib().hykkt_set_option(self.h, name.encode(), int(value)))

    def timing(self) -> dict:
        t = _lib.Timing()
        check(_lib.lib().hykkt_last_timing(self.h, C.byref(t)))
        return {n: getattr(t, n) for n, _ in t._fields_}

    def solve_full(self, sys: BlockKkt4x4, cfg: SolverConfig | None = None,
                   state: RegularizationState | None = None,
                   metrics: bool = True) -> FullSolveResult:
        """hkkt::solve_full (solver.cpp:295-328) with this handle's symbolic
        analysis (analysed on first use, like a null `shared`)."""
        cfg = cfg or SolverConfig()
        check_dims(sys)
        created = False
        if not isinstance(self._pattern, BlockKkt4x4) or not self._pattern.same_pattern_as(sys):
            self.analyze(sys)
            created = True
        if state is None:
            state = RegularizationState.initial(cfg)
        v = self._values(sys)
        rep = _lib.Report()
        dm = C.c_double(state.delta_min_current)
        sol = FullSolution(np.zeros(sys.n_x), np.zeros(sys.m_d), np.zeros(sys.m_c),
                           np.zeros(sys.m_d))
        flags = _lib.FLAG_METRICS if metrics else 0
        check(_lib.lib().hykkt_solve_full(self.h, C.byref(cfg.c()), C.byref(v), C.byref(dm),
                                          flags, C.byref(rep), dp(sol.dx), dp(sol.ds),
                                          dp(sol.dy), dp(sol.dyd)))
        state.delta_min_current = dm.value
        state.delta1 = rep.delta1_final
        state.attempts = rep.factorization_attempts
        report = SolveReport.from_c(rep)
        return FullSolveResult(sol if is_success(report.status) else None, report, created)


def solve_full(sys: BlockKkt4x4, cfg: SolverConfig | None = None, shared: Device | None = None,
               state: RegularizationState | None = None) -> FullSolveResult:
    dev = shared or Device()
    return dev.solve_full(sys, cfg, state)


def _ladder(h, cfg: SolverConfig, values, state: RegularizationState):
    dm = C.c_double(state.delta_min_current)
    att, d1, fc = C.c_int64(0), C.c_double(0.0), C.c_int64(-1)
    v = None if values is None else f64(values)
    check(_lib.lib().hykkt_factor_ladder(h, C.byref(cfg.c()), dp(v), C.byref(dm), C.byref(att),
                                         C.byref(d1), C.byref(fc)))
    state.delta_min_current = dm.value
    state.delta1 = d1.value
    state.attempts = att.value
    return None if fc.value < 0 else LadderFailure(att.value, d1.value, fc.value)


def _cg_schur(h, rhs, cfg: SolverConfig, delta2: float) -> CgResult:
    rhs = f64(rhs)
    x = np.zeros(rhs.shape[0])
    it, rr = C.c_int64(0), C.c_double(0.0)
    conv, sq = C.c_int32(0), C.c_int32(0)
    check(_lib.lib().hykkt_cg_schur(h, C.byref(cfg.c()), dp(rhs), delta2, dp(x), C.byref(it),
                                    C.byref(rr), C.byref(conv), C.byref(sq)))
    return CgResult(x, it.value, rr.value, bool(conv.value), bool(sq.value))


def solve_sequence(systems: Sequence[BlockKkt4x4], cfg: SolverConfig | None = None,
                   device: int = 0, perm=None) -> SequenceResult:
    """hkkt::solve_sequence (solver.cpp:352-412): one symbolic analysis when
    the patterns are uniform, delta_min carried across, failures recorded
    and the sequence continued.  `perm` (optional) is the ordering of the
    shared symbolic analysis (the reference computes amd_order there)."""
    if len(systems) == 0:
        raise _lib.InvalidMatrixError(-1, "solve_sequence: empty sequence")
    cfg = cfg or SolverConfig()
    res = SequenceResult()
    res.pattern_uniform = all(s.same_pattern_as(systems[0]) for s in systems[1:])
    dev = Device(device)
    state = RegularizationState.initial(cfg)
    for k, sys in enumerate(systems):
        if not res.pattern_uniform:
            dev._pattern = None
        if dev._pattern is None and perm is not None and (res.pattern_uniform or k == 0):
            dev.analyze(sys, perm)
            res.stats.symbolic_analyses += 1
        r = dev.solve_full(sys, cfg, state)
        r.report.symbolic_reused = res.pattern_uniform and k > 0
        if r.symbolic_created:
            res.stats.symbolic_analyses += 1
        res.stats.factorization_attempts += r.report.factorization_attempts
        if r.report.status != SolveStatus.kFailedDeltaMaxExceeded:
            res.stats.numeric_factorizations += 1
        res.reports.append(r.report)
        res.solutions.append(r.solution)
    dev.close()
    return res


class CholeskyFactor:
    """symbolic_cholesky + numeric_cholesky + factor_solve on the device
    (cholesky.hpp:41-83) for a general SPD matrix in lower CSC storage."""

    def __init__(self, a_lower: CscMatrix, perm=None, device: int = 0):
        self.dev = Device(device)
        self.n = a_lower.ncols
        self._cp, self._ri = i64(a_lower.colptr), i64(a_lower.rowidx)
        p = None if perm is None else i64(perm)
        check(_lib.lib().hykkt_chol_analyze(self.dev.h, self.n, ip(self._cp), ip(self._ri), ip(p)))
        self.ok = False

    def factorize(self, values, pivot_floor: float = 0.0):
        """Returns None on success or NotSpdFailure (a value, as in the
        reference)."""
        v = f64(values)
        fc, fp = C.c_int64(0), C.c_double(0)
        check(_lib.lib().hykkt_chol_factor(self.dev.h, dp(v), pivot_floor, C.byref(fc),
                                           C.byref(fp)))
        self.ok = fc.value < 0
        return None if self.ok else NotSpdFailure(int(fc.value), float(fp.value))

    def solve(self, b) -> np.ndarray:
        b = f64(b)
        if b.shape[0] != self.n:
            raise _lib.InvalidMatrixError(-1, f"factor_solve: rhs has length {b.shape[0]}, "
                                              f"expected {self.n}")
        x = np.zeros(self.n)
        check(_lib.lib().hykkt_chol_solve(self.dev.h, dp(b), dp(x)))
        return x

    def factorize_with_ladder(self, values, cfg: SolverConfig, state: RegularizationState):
        """factorize_with_ladder (solver.cpp:108-142) on a matrix in this
        factor's pattern (an HGammaSystem's h_gamma values); None on
        success or a LadderFailure."""
        r = _ladder(self.dev.h, cfg, values, state)
        self.ok = r is None
        return r

    def set_factor(self, l_values) -> None:
        """Load reference-layout L values (NumericCholesky::l_values)."""
        v = f64(l_values)
        check(_lib.lib().hykkt_chol_set_factor(self.dev.h, dp(v)))
        self.ok = True

    def set_j(self, j: CscMatrix) -> None:
        """The J of SchurOperator (solver.hpp:97-103) for cg_schur."""
        self._j = [i64(j.colptr), i64(j.rowidx), f64(j.values)]
        check(_lib.lib().hykkt_chol_set_j(self.dev.h, j.nrows, ip(self._j[0]), ip(self._j[1]),
                                          dp(self._j[2])))

    def cg_schur(self, rhs, cfg: SolverConfig | None = None, delta2: float = 0.0) -> CgResult:
        """cg_schur (solver.cpp:154-201) on S = J H^-1 J^T + delta2 I."""
        return _cg_schur(self.dev.h, rhs, cfg or SolverConfig(), delta2)

    def factor(self) -> dict:
        info = self.dev.info()
        n, nnz = info["n"], info["nnz_l"]
        cp, ri, par = np.zeros(n + 1, np.int64), np.zeros(nnz, np.int64), np.zeros(n, np.int64)
        lv = np.zeros(nnz) if self.ok else None
        check(_lib.lib().hykkt_chol_get_factor(self.dev.h, ip(cp), ip(ri), dp(lv), ip(par)))
        return dict(l_colptr=cp, l_rowidx=ri, l_values=lv, parent=par, perm=self.dev.perm())


def host_analyze(sys: BlockKkt4x4, perm=None):
    """Host-only symbolic analysis (no GPU): returns (stats dict, ordering)."""
    check_dims(sys)
    a = [i64(x) for x in (sys.h.colptr, sys.h.rowidx, sys.j.colptr, sys.j.rowidx,
                          sys.j_d.colptr, sys.j_d.rowidx)]
    p = None if perm is None else i64(perm)
    out = np.zeros(sys.n_x, np.int64)
    st = _lib.Analysis()
    check(_lib.lib().hykkt_host_analyze(sys.n_x, sys.m_c, sys.m_d, *[ip(x) for x in a], ip(p),
                                        ip(out), C.byref(st)))
    return {n: getattr(st, n) for n, _ in st._fields_}, out


def sysplan_check(sys: BlockKkt4x4, perm=None, nchunk: int = 8) -> dict:
    """Host-only: builds the system-per-CTA stream program of the batched
    solve for this pattern (rings of nchunk x 1024 entries) and runs its host
    emulation of J^T -> forward -> backward -> J: max relative error vs a
    plain reference plus program statistics.  Raises when a step would read
    outside its ring windows."""
    check_dims(sys)
    a = [i64(x) for x in (sys.h.colptr, sys.h.rowidx, sys.j.colptr, sys.j.rowidx,
                          sys.j_d.colptr, sys.j_d.rowidx)]
    p = None if perm is None else i64(perm)
    out = np.zeros(8)
    L = _lib.lib()
    L.hykkt_debug_sysplan_check.argtypes = [C.c_int64] * 3 + [C.c_void_p] * 7 + [C.c_int, C.c_void_p]
    check(L.hykkt_debug_sysplan_check(sys.n_x, sys.m_c, sys.m_d, *[ip(x) for x in a], ip(p),
                                      nchunk, out.ctypes.data))
    keys = ("max_rel_err", "value_len", "index_len", "steps", "tasks", "segments",
            "max_segs_per_step", "value_entries")
    return dict(zip(keys, out.tolist()))


VALUE_FIELDS = ("h_val", "j_val", "jd_val", "d_x", "d_s", "r_tilde_x", "r_s", "r_y", "r_yd")


def system_values(sys: BlockKkt4x4) -> tuple:
    return (sys.h.values, sys.j.values, sys.j_d.values, sys.d_x, sys.d_s, sys.r_tilde_x,
            sys.r_s, sys.r_y, sys.r_yd)


def stack_values(systems: Sequence[BlockKkt4x4], out: dict | None = None) -> dict:
    """[system][entry] arrays per value field (the batch C-ABI layout).  With
    `out` (e.g. pinned host buffers) the arrays are filled in place."""
    cols = list(zip(*[system_values(s) for s in systems]))
    res = {}
    for name, parts in zip(VALUE_FIELDS, cols):
        if out is not None:
            np.stack(parts, out=out[name])
            res[name] = out[name]
        else:
            res[name] = np.ascontiguousarray(np.stack(parts), np.float64)
    return res


class Batch:
    """B independent systems on the pattern analysed by `dev` (device-side
    replacement of solve_sequence's parallel mode, solver.cpp:374-398)."""

    def __init__(self, dev: Device):
        self.dev = dev
        self.count = 0

    def upload(self, values: dict) -> None:
        arrs = [values[n] for n in VALUE_FIELDS]
        for a in arrs:
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise _lib.InvalidMatrixError(-1, "batch values must be C-contiguous float64")
        self.count = arrs[0].shape[0]
        self._keep = arrs
        v = _lib.Values(*[dp(a) for a in arrs])
        check(_lib.lib().hykkt_batch_upload(self.dev.h, self.count, C.byref(v)))

    def upload_async(self, values: dict) -> None:
        """Starts the host-to-device copy of the next batch
        (hykkt_batch_upload_async); the next solve_resident consumes the
        oldest pending upload.  The arrays must stay alive (and unchanged)
        until that solve: they are kept referenced here."""
        arrs = [values[n] for n in VALUE_FIELDS]
        for a in arrs:
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise _lib.InvalidMatrixError(-1, "batch values must be C-contiguous float64")
        self._pending = getattr(self, "_pending", [])[-1:] + [arrs]
        v = _lib.Values(*[dp(a) for a in arrs])
        check(_lib.lib().hykkt_batch_upload_async(self.dev.h, arrs[0].shape[0], C.byref(v)))
        if not self.count:
            self.count = arrs[0].shape[0]

    def download_async(self, out: dict) -> dict:
        """Starts the device-to-host copy of the last solve's outputs
        (hykkt_batch_download_async); `out` is complete after sync()."""
        check(_lib.lib().hykkt_batch_download_async(self.dev.h, dp(out["dx"]), dp(out["ds"]),
                                                    dp(out["dy"]), dp(out["dyd"])))
        return out

    def sync(self) -> None:
        check(_lib.lib().hykkt_batch_sync(self.dev.h))

    def upload_device(self, ptrs: dict, count: int) -> None:
        """Values already in device memory (hykkt_batch_upload_device):
        `ptrs` maps each VALUE_FIELDS name to a device address of a
        [system][entry] float64 array; copied device-to-device."""
        self.count = int(count)
        v = _lib.Values(*[C.cast(C.c_void_p(int(ptrs[n])), _lib.F64P) for n in VALUE_FIELDS])
        check(_lib.lib().hykkt_batch_upload_device(self.dev.h, self.count, C.byref(v)))

    def solve_resident(self, cfg: SolverConfig, metrics: bool = False, timing: bool = False):
        reps = (_lib.Report * self.count)()
        flags = (_lib.FLAG_METRICS if metrics else 0) | (_lib.FLAG_TIMING if timing else 0)
        check(_lib.lib().hykkt_batch_solve_resident(self.dev.h, C.byref(cfg.c()), flags, reps))
        return [SolveReport.from_c(r) for r in reps]

    def download(self, out: dict | None = None) -> dict:
        s = self.dev._pattern
        B = self.count
        if out is None:
            out = dict(dx=np.zeros((B, s.n_x)), ds=np.zeros((B, s.m_d)), dy=np.zeros((B, s.m_c)),
                       dyd=np.zeros((B, s.m_d)))
        check(_lib.lib().hykkt_batch_download(self.dev.h, dp(out["dx"]), dp(out["ds"]),
                                              dp(out["dy"]), dp(out["dyd"])))
        return out
