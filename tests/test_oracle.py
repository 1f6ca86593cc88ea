"""CPU: the checker itself.  The C restatement (oracle/hykkt_oracle.c) must
be bit-identical to the compiled reference (oracle/_ref) and to the golden
fixtures; the reference's own known-answer tests are restated here."""
import numpy as np
import pytest

from golden_util import NAMES, load, stacked
from oracle import restatement as rs
from paper_2110_03636_b200.kkt import CscMatrix


@pytest.mark.parametrize("name", NAMES)
def test_restatement_reproduces_golden_bitwise(name):
    s, cfg, perm, want = load(name)
    rep, dx, ds, dy, dyd, _ = rs.solve_full(s, cfg, perm)
    assert rep["status"] == want["report"]["status"]
    assert rep["cg_iterations"] == want["report"]["cg_iterations"]
    assert rep["ruiz_iterations"] == want["report"]["ruiz_iterations"]
    assert rep["factorization_attempts"] == want["report"]["factorization_attempts"]
    assert rep["delta1_final"] == want["report"]["delta1_final"]
    assert rep["delta2_used"] == want["report"]["delta2_used"]
    if rep["status"] <= 1:
        assert np.array_equal(np.concatenate([dx, ds, dy, dyd]), stacked(want))


@pytest.mark.parametrize("name", NAMES)
def test_reference_reproduces_golden_bitwise(ref, name):
    s, cfg, perm, want = load(name)
    got = ref.solve_full(s, cfg, perm)
    assert got.report["status"] == want["report"]["status"]
    if got.report["status"] <= 1:
        assert np.array_equal(got.stacked(), stacked(want))
    assert np.array_equal(ref.hgamma_amd(s, cfg), perm)


def test_restatement_matches_reference_on_fresh_instances(ref):
    from paper_2110_03636_b200 import SolverConfig, acopf
    for s in [acopf.generate(80, 3, 5), ref.generate(50, 12, 9, seed=41)[0]]:
        cfg = SolverConfig()
        perm = ref.hgamma_amd(s, cfg)
        w = ref.solve_full(s, cfg, perm)
        rep, dx, ds, dy, dyd, _ = rs.solve_full(s, cfg, perm)
        assert np.array_equal(np.concatenate([dx, ds, dy, dyd]), w.stacked())


# ---- reference known answers (tests/test_sparse_core.cpp:248-272) -----------
def test_kat_diag_4_9():
    a = CscMatrix.from_triplets(2, 2, [0, 1], [0, 1], [4.0, 9.0])
    r = rs.cholesky(a, [0, 1], 0.0, b=[8.0, 27.0])
    assert r["failed_column"] == -1
    assert r["l_values"].tolist() == [2.0, 3.0]
    assert r["x"].tolist() == [2.0, 3.0]


def test_kat_not_spd_fails_at_column_1():
    a = CscMatrix.from_triplets(2, 2, [0, 1, 1], [0, 0, 1], [1.0, 2.0, 1.0])
    r = rs.cholesky(a, [0, 1], 0.0)
    assert r["failed_column"] == 1
    assert r["failed_pivot"] == -3.0


def test_kat_chol_reference_agreement(ref):
    rng = np.random.default_rng(4)
    n = 60
    rows, cols, vals = [], [], []
    for j in range(n):
        rows.append(j); cols.append(j); vals.append(8.0 + rng.uniform())
        for i in set(rng.integers(j + 1, n, size=3).tolist()) if j + 1 < n else []:
            rows.append(i); cols.append(j); vals.append(rng.uniform(-1, 1))
    a = CscMatrix.from_triplets(n, n, rows, cols, vals)
    want = ref.numeric_cholesky(a, None, 0.0)
    got = rs.cholesky(a, want["perm"], 0.0)
    assert np.array_equal(got["l_values"], want["l_values"])
    ref.free_chol(want)
