"""GPU parity: the sm_100a path (through the C ABI) against the compiled
reference (oracle/_ref) on identical inputs and the identical ordering.

Tolerances (BASELINE.json north_star): solution relative error <= 1e-8,
backward error be_4x4 <= 1e-10, CG iterations within +-1, identical status,
delta1 and delta2.  Factor-level checks mirror tests/test_sparse_core.cpp.
"""
import numpy as np
import pytest

from paper_2110_03636_b200 import (CholeskyFactor, Device, NotSpdFailure, SolverConfig,
                                   SolveStatus, acopf, solve_sequence)
from paper_2110_03636_b200.kkt import CscMatrix

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ---- Cholesky-level known answers (test_sparse_core.cpp:248-272) -----------
def test_chol_diag_known_answer():
    a = CscMatrix.from_triplets(2, 2, [0, 1], [0, 1], [4.0, 9.0])
    f = CholeskyFactor(a)
    assert f.factorize(a.values, 0.0) is None
    L = f.factor()
    assert sorted(L["l_values"].tolist()) == [2.0, 3.0]
    x = f.solve([8.0, 27.0])
    np.testing.assert_allclose(x, [2.0, 3.0], rtol=0, atol=1e-15)


def test_chol_not_spd_known_answer():
    a = CscMatrix.from_triplets(2, 2, [0, 1, 1], [0, 0, 1], [1.0, 2.0, 1.0])
    f = CholeskyFactor(a, perm=[0, 1])
    r = f.factorize(a.values, 0.0)
    assert isinstance(r, NotSpdFailure)
    assert r.column == 1
    assert r.pivot == pytest.approx(-3.0)


def _random_spd_lower(n, per_col, rng):
    rows, cols, vals = [], [], []
    absr = np.zeros(n)
    for j in range(n - 1):
        for i in set(rng.integers(j + 1, n, size=per_col).tolist()):
            v = rng.uniform(-1, 1)
            rows.append(i); cols.append(j); vals.append(v)
            absr[i] += abs(v); absr[j] += abs(v)
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(absr[i] + 0.5 + rng.uniform(0, 1))
    return CscMatrix.from_triplets(n, n, rows, cols, vals)


@pytest.mark.parametrize("n,seed", [(30, 1), (200, 2), (1000, 3)])
def test_chol_matches_reference(ref, n, seed):
    rng = np.random.default_rng(seed)
    a = _random_spd_lower(n, 3, rng)
    want = ref.numeric_cholesky(a, None, 0.0)
    f = CholeskyFactor(a, perm=want["perm"])
    assert f.factorize(a.values, 0.0) is None
    got = f.factor()
    assert np.array_equal(got["l_colptr"], want["l_colptr"])
    assert np.array_equal(got["l_rowidx"], want["l_rowidx"])
    assert np.array_equal(got["parent"], want["parent"])
    assert rel(got["l_values"], want["l_values"]) <= 1e-13
    b = rng.uniform(-1, 1, n)
    assert rel(f.solve(b), ref.factor_solve(want, b)) <= 1e-12
    ref.free_chol(want)


# ---- KKT path ---------------------------------------------------------------
def _compare(sys_, cfg, perm, ref, sol_tol=1e-8):
    want = ref.solve_full(sys_, cfg, perm)
    dev = Device(0)
    dev.analyze(sys_, perm)
    got = dev.solve_full(sys_, cfg)
    assert got.report.status == SolveStatus(want.report["status"])
    assert got.report.delta1_final == want.report["delta1_final"]
    assert got.report.delta2_used == want.report["delta2_used"]
    assert got.report.ruiz_iterations == want.report["ruiz_iterations"]
    assert abs(got.report.cg_iterations - want.report["cg_iterations"]) <= 1
    if got.solution is not None:
        assert rel(got.solution.stacked(), want.stacked()) <= sol_tol
        assert got.report.be_4x4 <= max(1e-10, 10 * want.report["be_4x4"])
    dev.close()
    return got, want


@pytest.mark.parametrize("nb", [60, 500, 2000])
def test_acopf_solve_full_matches_reference(ref, nb):
    s = acopf.generate(nb, 7, 7)
    cfg = SolverConfig()
    perm = ref.hgamma_amd(s, cfg)
    _compare(s, cfg, perm, ref)


@pytest.mark.parametrize("nx,mc,md,seed", [(240, 60, 50, 23), (60, 15, 12, 31), (40, 10, 8, 37)])
def test_reference_generator_instances(ref, nx, mc, md, seed):
    s = ref.generate(nx, mc, md, seed=seed)[0]
    cfg = SolverConfig()
    perm = ref.hgamma_amd(s, cfg)
    _compare(s, cfg, perm, ref)


def test_own_ordering_solves(ref):
    s = acopf.generate(500, 7, 7)
    dev = Device(0)
    dev.analyze(s)  # own minimum-degree ordering
    got = dev.solve_full(s, SolverConfig())
    want = ref.solve_full(s, SolverConfig())
    assert rel(got.solution.stacked(), want.stacked()) <= 1e-8
    assert abs(got.report.cg_iterations - want.report["cg_iterations"]) <= 1


def test_resident_batch_matches_reference(ref):
    from paper_2110_03636_b200.solver import Batch, stack_values
    systems = acopf.batch(120, 4, seed=7)
    cfg = SolverConfig()
    perm = ref.hgamma_amd(systems[0], cfg)
    dev = Device(0)
    dev.analyze(systems[0], perm)
    b = Batch(dev)
    b.upload(stack_values(systems))
    reps = b.solve_resident(cfg)
    out = b.download()
    for k, s in enumerate(systems):
        want = ref.solve_full(s, cfg, perm)
        got = np.concatenate([out["dx"][k], out["ds"][k], out["dy"][k], out["dyd"][k]])
        assert rel(got, want.stacked()) <= 1e-8
        assert abs(reps[k].cg_iterations - want.report["cg_iterations"]) <= 1
