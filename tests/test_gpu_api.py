"""GPU: the split reference API through the C ABI — solve_reduced,
assemble_h_gamma, factorize_with_ladder, cg_schur, factor_solve on a
reference-layout factor, device-pointer values — against the compiled
reference (oracle/_ref) and restatements of the reference's own known-answer
tests (proj/tests/test_hybrid_solver.cpp, cited per test).

Tolerances: identical status / delta1 / delta2 / attempts; CG iterations
within +-1; solutions <= 1e-8 relative (north_star)."""
import numpy as np
import pytest

from paper_2110_03636_b200 import (CholeskyFactor, Device, LadderFailure, RegularizationState,
                                   SolverConfig, SolveStatus, acopf)
from paper_2110_03636_b200.kkt import CscMatrix, Reduced2x2

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def diagonal_h_gamma(n, eps):
    """test_hybrid_solver.cpp:31-42: diag(1 + 0.1 i), last entry -eps."""
    d = np.array([-eps if i == n - 1 else 1.0 + 0.1 * i for i in range(n)])
    return CscMatrix.from_triplets(n, n, np.arange(n), np.arange(n), d)


def spd_lower(n, per_col, margin, rng):
    """Same construction as test_support.hpp:62-82 (random_spd_lower)."""
    rows, cols, vals = [], [], []
    absr = np.zeros(n)
    for j in range(n - 1):
        seen = set()
        for _ in range(per_col):
            i = int(rng.integers(j + 1, n))
            if i in seen:
                continue
            seen.add(i)
            v = rng.uniform(-1, 1)
            rows.append(i); cols.append(j); vals.append(v)
            absr[i] += abs(v); absr[j] += abs(v)
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(absr[i] + margin + rng.uniform(0, 1))
    return CscMatrix.from_triplets(n, n, rows, cols, vals)


# ---- factorize_with_ladder KATs ----------------------------------------------
@pytest.mark.parametrize("j", range(7))
def test_ladder_minimal_level_within_factor_two(j):
    """test_hybrid_solver.cpp:157-179: success at delta_min 2^(j+1) after j+3
    attempts; half of that level still fails."""
    cfg = SolverConfig()
    eps = 1.5 * cfg.delta_min * 2.0 ** j
    hg = diagonal_h_gamma(12, eps)
    f = CholeskyFactor(hg)
    st = RegularizationState.initial(cfg)
    assert f.factorize_with_ladder(hg.values, cfg, st) is None
    assert st.delta1 == pytest.approx(cfg.delta_min * 2.0 ** (j + 1), rel=1e-12)
    assert st.attempts == j + 3
    half = hg.values.copy()
    half[np.flatnonzero(hg.rowidx == hg.col_of_entries())] += st.delta1 / 2.0
    assert f.factorize(half, cfg.pivot_floor * 1.0) is not None


def test_ladder_failure_exhausts_attempt_bound():
    """test_hybrid_solver.cpp:181-192: lambda_min = -1 -> LadderFailure after
    ceil(log2(delta_max / delta_min)) + 1 attempts."""
    cfg = SolverConfig()
    hg = diagonal_h_gamma(10, 1.0)
    f = CholeskyFactor(hg)
    st = RegularizationState.initial(cfg)
    r = f.factorize_with_ladder(hg.values, cfg, st)
    assert isinstance(r, LadderFailure)
    bound = int(np.ceil(np.log2(cfg.delta_max / cfg.delta_min))) + 1
    assert r.attempts == bound
    assert r.failed_column >= 0


def test_ladder_delta_min_carries_across_matrices():
    """test_hybrid_solver.cpp:194-212: the second matrix restarts at 0 and
    jumps straight back to the carried level (2 attempts)."""
    cfg = SolverConfig()
    hg = diagonal_h_gamma(12, 1.5 * cfg.delta_min * 16.0)
    f = CholeskyFactor(hg)
    st = RegularizationState.initial(cfg)
    assert f.factorize_with_ladder(hg.values, cfg, st) is None
    level = st.delta1
    assert level == pytest.approx(32.0 * cfg.delta_min, rel=1e-12)
    assert f.factorize_with_ladder(hg.values, cfg, st) is None
    assert st.attempts == 2
    assert st.delta1 == pytest.approx(level, rel=1e-12)


def test_ladder_pivot_just_below_floor_rescued_at_first_rung():
    """test_hybrid_solver.cpp:498-509."""
    cfg = SolverConfig()
    hg = diagonal_h_gamma(8, 2e-13)
    f = CholeskyFactor(hg)
    st = RegularizationState.initial(cfg)
    assert f.factorize_with_ladder(hg.values, cfg, st) is None
    assert st.delta1 == cfg.delta_min
    assert st.attempts == 2


@pytest.mark.parametrize("seed", [44, 45])
def test_ladder_matches_reference_on_indefinite_h_gamma(ref, seed):
    """An indefinite generator instance (kIndefinite) through the device
    ladder vs the reference's factorize_with_ladder on the same H_gamma."""
    s = ref.generate(60, 15, 12, klass=1, seed=seed)[0]
    cfg = SolverConfig()
    a = ref.assemble(s, cfg)
    hg = CscMatrix(s.n_x, s.n_x, a["colptr"], a["rowidx"], a["values"])
    perm = ref.hgamma_amd(s, cfg)
    want = ref.ladder(hg, cfg, perm)
    f = CholeskyFactor(hg, perm=perm)
    st = RegularizationState.initial(cfg)
    got = f.factorize_with_ladder(hg.values, cfg, st)
    assert (got is None) == want["ok"]
    assert st.attempts == want["attempts"]
    assert st.delta1 == want["delta1"]
    assert st.delta_min_current == want["delta_min_current"]


# ---- cg_schur ------------------------------------------------------------------
def test_cg_schur_zero_rhs_takes_no_iterations():
    """test_hybrid_solver.cpp:214-227."""
    rng = np.random.default_rng(5)
    h = spd_lower(10, 2, 0.5, rng)
    f = CholeskyFactor(h)
    assert f.factorize(h.values, 0.0) is None
    j = CscMatrix.from_triplets(4, 10, [0, 1, 2, 3, 0], [0, 3, 5, 9, 7], [1.0, -0.5, 2.0, 0.3, 0.7])
    f.set_j(j)
    r = f.cg_schur(np.zeros(4))
    assert r.converged and r.iterations == 0
    assert (r.x == 0.0).all()


def test_cg_schur_identity_converges_in_one_iteration():
    """test_hybrid_solver.cpp:229-244: H = I, J orthonormal rows -> S = I."""
    nx, mc = 6, 3
    h = CscMatrix.from_triplets(nx, nx, np.arange(nx), np.arange(nx), np.ones(nx))
    f = CholeskyFactor(h)
    assert f.factorize(h.values, 0.0) is None
    f.set_j(CscMatrix.from_triplets(mc, nx, np.arange(mc), 2 * np.arange(mc), np.ones(mc)))
    r = f.cg_schur([1.0, -2.0, 0.5])
    assert r.converged and r.iterations == 1


@pytest.mark.parametrize("delta2", [0.0, 1e-9])
def test_cg_schur_matches_reference(ref, delta2):
    rng = np.random.default_rng(11)
    h = spd_lower(300, 3, 0.5, rng)
    jr, jc = rng.integers(0, 80, 600), rng.integers(0, 300, 600)
    j = CscMatrix.from_triplets(80, 300, jr, jc, rng.uniform(-1, 1, 600))
    rhs = rng.uniform(-1, 1, 80)
    cfg = SolverConfig()
    want = ref.numeric_cholesky(h, None, 0.0)
    perm = want["perm"]
    wcg = ref.cg_schur(h, j, rhs, cfg, perm, delta2)
    f = CholeskyFactor(h, perm=perm)
    assert f.factorize(h.values, 0.0) is None
    f.set_j(j)
    got = f.cg_schur(rhs, cfg, delta2)
    assert got.converged == wcg["converged"]
    assert abs(got.iterations - wcg["iterations"]) <= 1
    assert rel(got.x, wcg["x"]) <= 1e-10
    # the same CG on a factor loaded from the reference layout
    g = CholeskyFactor(h, perm=perm)
    g.set_factor(want["l_values"])
    g.set_j(j)
    got2 = g.cg_schur(rhs, cfg, delta2)
    assert abs(got2.iterations - wcg["iterations"]) <= 1
    assert rel(got2.x, wcg["x"]) <= 1e-10
    b = rng.uniform(-1, 1, 300)
    assert rel(g.solve(b), ref.factor_solve(want, b)) <= 1e-12
    ref.free_chol(want)


# ---- assemble_h_gamma ------------------------------------------------------------
@pytest.mark.parametrize("gamma", [0.0, 1e4, 1e8])
def test_assemble_matches_reference(ref, gamma):
    s = acopf.generate(120, 7, 7)
    cfg = SolverConfig(gamma=gamma)
    want = ref.assemble(s, cfg)
    dev = Device(0)
    dev.analyze(s)
    dev.upload(s)
    hg = dev.assemble(cfg)
    assert np.array_equal(hg.h_gamma.colptr, want["colptr"])
    assert np.array_equal(hg.h_gamma.rowidx, want["rowidx"])
    assert rel(hg.h_gamma.values, want["values"]) <= 1e-15
    assert rel(hg.r_hat_x, want["r_hat_x"]) <= 1e-15
    # the split path: ladder + w solve + cg_schur on the same handle
    st = RegularizationState.initial(cfg)
    if gamma > 0.0:
        assert dev.factorize_with_ladder(cfg, st) is None
        w = dev.factor_solve(hg.r_hat_x)
        assert np.isfinite(w).all()
    dev.close()


# ---- solve_reduced ---------------------------------------------------------------
def test_solve_reduced_matches_dense_block_solve():
    """test_hybrid_solver.cpp:246-275: J square nonsingular, H_tilde SPD ->
    dense solve of [[H, J^T], [J, 0]] to 1e-9."""
    rng = np.random.default_rng(13)
    n = 14
    ht = spd_lower(n, 3, 0.5, rng)
    rows = list(range(n)) + list(range(n - 1))
    cols = list(range(n)) + list(range(1, n))
    vals = [1.0 + 0.1 * i for i in range(n)] + [0.3] * (n - 1)
    j = CscMatrix.from_triplets(n, n, rows, cols, vals)
    red = Reduced2x2(ht, j, rng.uniform(-1, 1, n), rng.uniform(-1, 1, n))
    dev = Device(0)
    r = dev.solve_reduced(red, SolverConfig())
    assert r.ok() and r.report.status == SolveStatus.kSolved and r.report.delta1_final == 0.0
    H = ht.to_dense(symmetric_lower=True)
    J = j.to_dense()
    K = np.block([[H, J.T], [J, np.zeros((n, n))]])
    z = np.linalg.solve(K, np.concatenate([red.r_x, red.r_y]))
    assert rel(np.concatenate([r.dx, r.dy]), z) <= 1e-9
    dev.close()


@pytest.mark.parametrize("klass,seed,status", [(2, 7, SolveStatus.kSolved),
                                               (3, 8, SolveStatus.kSolvedWithDelta2)])
def test_solve_reduced_rank_deficient(ref, klass, seed, status):
    """test_hybrid_solver.cpp:277-315: consistent rank-deficient J solves
    without delta2, the inconsistent one restarts with delta2."""
    s = ref.generate(30, 8, 6, klass=klass, seed=seed)[0]
    red = ref.reduce(s)
    cfg = SolverConfig()
    perm = ref.hgamma_amd(s, cfg)
    want = ref.solve_reduced(red, cfg, perm)
    dev = Device(0)
    dev.analyze_reduced(red, perm)
    r = dev.solve_reduced(red, cfg)
    assert r.report.status == status == SolveStatus(want["report"]["status"])
    assert r.report.delta2_used == want["report"]["delta2_used"]
    assert abs(r.report.cg_iterations - want["report"]["cg_iterations"]) <= 1
    assert rel(np.concatenate([r.dx, r.dy]), np.concatenate([want["dx"], want["dy"]])) <= 1e-8
    dev.close()


@pytest.mark.parametrize("nb", [60, 500, 2000])
def test_solve_reduced_matches_reference_acopf(ref, nb):
    s = acopf.generate(nb, 7, 7)
    red = ref.reduce(s)
    cfg = SolverConfig()
    perm = ref.hgamma_amd(s, cfg)
    want = ref.solve_reduced(red, cfg, perm)
    dev = Device(0)
    dev.analyze_reduced(red, perm)
    r = dev.solve_reduced(red, cfg)
    w = want["report"]
    assert int(r.report.status) == w["status"]
    assert r.report.delta1_final == w["delta1_final"]
    assert r.report.factorization_attempts == w["factorization_attempts"]
    assert abs(r.report.cg_iterations - w["cg_iterations"]) <= 1
    assert rel(np.concatenate([r.dx, r.dy]), np.concatenate([want["dx"], want["dy"]])) <= 1e-8
    assert r.report.be_2x2 <= max(1e-10, 10 * w["be_2x2"])
    dev.close()


# ---- device-pointer values --------------------------------------
def test_device_pointer_values_match_host_path():
    import ctypes as C

    import torch

    from paper_2110_03636_b200 import _lib
    from paper_2110_03636_b200.solver import system_values
    s = acopf.generate(200, 7, 7)
    cfg = SolverConfig()
    host = Device(0)
    host.analyze(s)
    want = host.solve_full(s, cfg)
    dev = Device(0)
    dev.analyze(s, host.perm())
    ts = [torch.tensor(np.asarray(v), dtype=torch.float64, device="cuda:0") for v in system_values(s)]
    torch.cuda.synchronize()
    v = _lib.Values(*[C.cast(C.c_void_p(t.data_ptr()), _lib.F64P) for t in ts])
    _lib.check(_lib.lib().hykkt_upload_values_device(dev.h, C.byref(v)))
    rep = dev.solve_resident(cfg)
    assert rep.status == want.report.status and rep.cg_iterations == want.report.cg_iterations
    ptrs = [C.c_void_p() for _ in range(4)]
    _lib.check(_lib.lib().hykkt_solution_device(dev.h, *[C.byref(p) for p in ptrs]))
    got = dev.download()
    assert np.array_equal(got.stacked(), want.solution.stacked())
    # host arrays are rejected by the *_device entry point
    hv = [np.ascontiguousarray(x, np.float64) for x in system_values(s)]
    bad = _lib.Values(*[x.ctypes.data_as(_lib.F64P) for x in hv])
    assert _lib.lib().hykkt_upload_values_device(dev.h, C.byref(bad)) == -1
    host.close()
    dev.close()


# ---- handle re-use (stale flags after re-analysis) -------------------
def test_reanalysis_between_batched_solves(ref):
    from paper_2110_03636_b200 import _lib
    from paper_2110_03636_b200.solver import Batch, stack_values
    cfg = SolverConfig()
    a = acopf.batch(60, 3, seed=7)
    b = acopf.batch(120, 3, seed=9)
    dev = Device(0)
    bt = Batch(dev)
    for systems in (a, b, a):
        dev.analyze(systems[0])
        perm = dev.perm()
        with pytest.raises(_lib.HykktError):  # the previous batch belongs to the old pattern
            bt.solve_resident(cfg)
        bt.upload(stack_values(systems))
        reps = bt.solve_resident(cfg)
        out = bt.download()
        for k, s in enumerate(systems):
            want = ref.solve_full(s, cfg, perm)
            got = np.concatenate([out["dx"][k], out["ds"][k], out["dy"][k], out["dyd"][k]])
            assert rel(got, want.stacked()) <= 1e-8
            assert abs(reps[k].cg_iterations - want.report["cg_iterations"]) <= 1
    dev.close()


# ---- pipelined batch copies (hykkt_batch_upload_async / _download_async) ------
def test_async_batch_copies_match_synchronous_path():
    """Three drifted value sets through the pipelined protocol (upload of set
    k+1 issued before the solve of set k, asynchronous downloads) give the
    same reports and solutions, bit for bit, as upload / solve / download."""
    from paper_2110_03636_b200.solver import Batch, stack_values
    cfg = SolverConfig()
    base = acopf.batch(120, 5, seed=7)
    sets = [base] + [[acopf.drift(x, 0.01, 31 * k + i) for i, x in enumerate(base)] for k in (1, 2)]
    vals = [stack_values(v) for v in sets]
    dev = Device(0)
    dev.analyze(base[0])
    bt = Batch(dev)
    want = []
    for v in vals:
        bt.upload(v)
        reps = bt.solve_resident(cfg)
        want.append(([r.cg_iterations for r in reps], {k: a.copy() for k, a in bt.download().items()}))
    outs = [dict(dx=np.zeros((5, base[0].n_x)), ds=np.zeros((5, base[0].m_d)), dy=np.zeros((5, base[0].m_c)),
                 dyd=np.zeros((5, base[0].m_d))) for _ in vals]
    bt.upload_async(vals[0])
    its = []
    for k in range(len(vals)):
        if k + 1 < len(vals):
            bt.upload_async(vals[k + 1])
        reps = bt.solve_resident(cfg)
        its.append([r.cg_iterations for r in reps])
        bt.download_async(outs[k])
    bt.sync()
    for k in range(len(vals)):
        assert its[k] == want[k][0]
        for name in ("dx", "ds", "dy", "dyd"):
            assert np.array_equal(outs[k][name], want[k][1][name]), (k, name)
    dev.close()


# ---- device BE / RR (metrics.cpp:28-240 on the device) ----------------------------
@pytest.mark.parametrize("nb,gamma", [(120, 1e4), (500, 1e8)])
def test_device_metrics_match_host_and_reference(ref, nb, gamma, monkeypatch):
    s = acopf.generate(nb, 7, 7)
    cfg = SolverConfig(gamma=gamma)
    perm = ref.hgamma_amd(s, cfg)
    want = ref.solve_full(s, cfg, perm).report
    dev = Device(0)
    dev.analyze(s, perm)
    d = dev.solve_full(s, cfg).report
    monkeypatch.setenv("HYKKT_METRICS_HOST", "1")
    h = dev.solve_full(s, cfg).report
    for name in ("be_4x4", "rr_4x4", "be_2x2", "rr_2x2", "be_2x2_scaled", "rr_2x2_scaled"):
        dv, hv, rv = getattr(d, name), getattr(h, name), want[name]
        assert np.isfinite(dv), name
        # rounding-level quantities: agree in magnitude, not digits
        assert dv <= 10 * max(hv, 1e-17) and hv <= 10 * max(dv, 1e-17), (name, dv, hv)
        assert dv <= 10 * max(rv, 1e-16), (name, dv, rv)
    assert d.be_4x4 <= 1e-10
    dev.close()


def test_device_metrics_reduced_handle(ref):
    s = ref.generate(60, 15, 12, seed=31)[0]
    red = ref.reduce(s)
    cfg = SolverConfig()
    perm = ref.hgamma_amd(s, cfg)
    want = ref.solve_reduced(red, cfg, perm)["report"]
    dev = Device(0)
    dev.analyze_reduced(red, perm)
    r = dev.solve_reduced(red, cfg)
    assert r.report.be_2x2 <= 10 * max(want["be_2x2"], 1e-16)
    assert np.isnan(r.report.be_4x4)
    dev.close()
