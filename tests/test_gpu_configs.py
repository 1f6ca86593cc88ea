"""GPU parity at every BASELINE.json config's stated size (SURVEY.md §8
config table), against the compiled reference (oracle/_ref) on identical
inputs and the identical elimination ordering:

  C1  nb = 500      gamma = 1e4                       (test_gpu_parity.py)
  C2  nb = 2000     10-step drifted IPM sequence, symbolic reused, delta_min
                    carried (solve_sequence, solver.cpp:352-412)
  C3  nb = 10000    gamma sweep 1e2 ... 1e8, CG counts within +-1 per gamma
  C4  nb = 70000    solution and backward error
  C5  256 x nb 2000 the bench's batch, two consecutive calls (the second on
                    drifted values, so the history-LPT system order runs)

Gates (north_star): solution relative error <= 1e-8 (stacked dx, ds, dy,
dyd as acceptance.cpp:135-139), be_4x4 <= 1e-10 (and <= 10x the
reference's), CG iterations within +-1, identical status / delta1 / delta2 /
attempts.  Achieved errors are printed (pytest -s) and collected by
tools/parity_report.py into profiles/.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2110_03636_b200 import Device, SolverConfig, SolveStatus, acopf, solve_sequence
from paper_2110_03636_b200.solver import Batch, stack_values

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SOL_TOL = 1e-8
BE_TOL = 1e-10


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def check_report(got, want):
    assert int(got.status) == want["status"]
    assert got.delta1_final == want["delta1_final"]
    assert got.delta2_used == want["delta2_used"]
    assert got.factorization_attempts == want["factorization_attempts"]
    assert got.ruiz_iterations == want["ruiz_iterations"]
    if want["status"] != SolveStatus.kFailedDeltaMaxExceeded:
        assert abs(got.cg_iterations - want["cg_iterations"]) <= 1


@pytest.fixture(scope="module")
def c3():
    return acopf.generate(10000, 7, 7)


@pytest.fixture(scope="module")
def c3_perm(ref, c3):
    return ref.hgamma_amd(c3, SolverConfig())


@pytest.mark.parametrize("gamma", [1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8])
def test_c3_gamma_sweep(ref, c3, c3_perm, gamma):
    """configs[2]: ACTIVSg10k-shaped (n_x = 76k, N = 200k), gamma sweep;
    proj/tests/test_cli.cpp:204-240 is the reference's own sweep."""
    cfg = SolverConfig(gamma=gamma)
    want = ref.solve_full(c3, cfg, c3_perm)
    dev = Device(0)
    dev.analyze(c3, c3_perm)
    got = dev.solve_full(c3, cfg)
    check_report(got.report, want.report)
    err = rel(got.solution.stacked(), want.stacked())
    print(f"C3 gamma={gamma:g}: cg {got.report.cg_iterations} (ref {want.report['cg_iterations']}) "
          f"sol rel err {err:.2e} be_4x4 {got.report.be_4x4:.2e} (ref {want.report['be_4x4']:.2e})")
    assert err <= SOL_TOL
    assert got.report.be_4x4 <= max(BE_TOL, 10 * want.report["be_4x4"])
    dev.close()


def test_c4_matches_reference(ref):
    """configs[3]: ACTIVSg70k-shaped (n_x = 532k, N = 1.4M), the roofline
    config; the device's own ordering is handed to the reference (its AMD
    takes ~70 s here)."""
    s = acopf.generate(70000, 7, 7)
    cfg = SolverConfig()
    dev = Device(0)
    dev.analyze(s)
    perm = dev.perm()
    got = dev.solve_full(s, cfg)
    want = ref.solve_full(s, cfg, perm)
    check_report(got.report, want.report)
    err = rel(got.solution.stacked(), want.stacked())
    print(f"C4: cg {got.report.cg_iterations} (ref {want.report['cg_iterations']}) sol rel err {err:.2e} "
          f"be_4x4 {got.report.be_4x4:.2e} (ref {want.report['be_4x4']:.2e})")
    assert err <= SOL_TOL
    assert got.report.be_4x4 <= BE_TOL
    dev.close()


def test_c2_sequence_matches_reference(ref):
    """configs[1]: a 10-step drifted ACTIVSg2000-shaped IPM sequence through
    solve_sequence (one symbolic analysis, delta_min carried) vs the
    reference's solve_sequence (which orders with its own AMD)."""
    seq = acopf.sequence(2000, 10, seed=7)
    cfg = SolverConfig()
    want = ref.solve_sequence(seq, cfg)
    perm = ref.hgamma_amd(seq[0], cfg)
    got = solve_sequence(seq, cfg, perm=perm)
    assert got.pattern_uniform == want["stats"]["pattern_uniform"]
    assert got.stats.symbolic_analyses == want["stats"]["symbolic_analyses"] == 1
    assert got.stats.numeric_factorizations == want["stats"]["numeric_factorizations"]
    assert got.stats.factorization_attempts == want["stats"]["factorization_attempts"]
    for k in range(len(seq)):
        check_report(got.reports[k], want["reports"][k])
        assert got.reports[k].symbolic_reused == bool(want["reports"][k]["symbolic_reused"])
        err = rel(got.solutions[k].stacked(), want["solutions"][k])
        assert err <= SOL_TOL, (k, err)
        assert got.reports[k].be_4x4 <= BE_TOL


def test_sequence_with_regularization_carries_delta_min(ref):
    """A kIndefinite sequence (the ladder climbs on every matrix): the
    carried delta_min_current makes later matrices start at the carried
    rung, exactly as the reference's solve_sequence."""
    seq = ref.generate(60, 15, 12, klass=1, length=4, seed=44)
    cfg = SolverConfig()
    want = ref.solve_sequence(seq, cfg)
    perm = ref.hgamma_amd(seq[0], cfg)
    got = solve_sequence(seq, cfg, perm=perm)
    assert got.stats.factorization_attempts == want["stats"]["factorization_attempts"]
    for k in range(len(seq)):
        check_report(got.reports[k], want["reports"][k])


def _ref_solutions(ref, systems, cfg, perm):
    with ThreadPoolExecutor(max_workers=16) as ex:
        return list(ex.map(lambda s: ref.solve_full(s, cfg, perm), systems))


def test_c5_bench_batch_two_calls(ref):
    """configs[4]: the bench's exact workload — 256 ACTIVSg2000-shaped
    systems (value seeds 7 + b) — solved twice through hykkt_batch_*; the
    second call runs on drifted values (drift 0.01) in the history-LPT order
    taken from the first call's CG counts.  Every system is checked."""
    B = 256
    cfg = SolverConfig()
    systems = acopf.batch(2000, B, seed=7)
    dev = Device(0)
    dev.analyze(systems[0])
    perm = dev.perm()
    bt = Batch(dev)
    drifted = [acopf.drift(s, 0.01, 1000 + b) for b, s in enumerate(systems)]
    worst = 0.0
    for call, batch in enumerate((systems, drifted)):
        bt.upload(stack_values(batch))
        reps = bt.solve_resident(cfg)
        out = bt.download()
        wants = _ref_solutions(ref, batch, cfg, perm)
        for k, want in enumerate(wants):
            check_report(reps[k], want.report)
            got = np.concatenate([out["dx"][k], out["ds"][k], out["dy"][k], out["dyd"][k]])
            err = rel(got, want.stacked())
            worst = max(worst, err)
            assert err <= SOL_TOL, (call, k, err)
    print(f"C5: 2 x {B} systems, worst sol rel err {worst:.2e}")
    dev.close()
