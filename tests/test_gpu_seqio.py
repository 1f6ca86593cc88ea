"""GPU runs of the sequence IO surface (seqio.cmd_solve / cmd_sweep_gamma)
on the manifest the reference wrote (tests/golden/seq_ref/), checked
against the reference's own solve.csv / sweep.csv / run_manifest.json for
the same sequence (proj/core/src/driver.cpp:182-279).  The reference's AMD
permutation (perm.npy) is handed over, so nnz_fac and ratio are exact.
Gates as everywhere: identical status / delta1 / delta2 / attempts, CG
iterations within +-1, be_4x4 <= max(1e-10, 10x the reference's)."""
import csv
from pathlib import Path

import numpy as np
import pytest

from paper_2110_03636_b200 import SolverConfig, seqio

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden" / "seq_ref"


def rows(p):
    lines = Path(p).read_text().splitlines()
    return lines[0], list(csv.DictReader(lines[1:]))


def close_be(got, want):
    return float(got) <= max(1e-10, 10 * float(want))


def test_cmd_solve_matches_reference(tmp_path):
    perm = np.load(G / "perm.npy")
    rc = seqio.cmd_solve(G / "seq" / "manifest.json", SolverConfig(), tmp_path, perm=perm)
    assert rc == seqio.EXIT_OK
    schema, got = rows(tmp_path / "solve.csv")
    ref_schema, want = rows(G / "solve" / "solve.csv")
    assert schema == ref_schema and len(got) == len(want) == 3
    for g, w in zip(got, want):
        for k in ("k", "delta1", "delta2", "nnz_fac", "ratio", "status"):
            assert g[k] == w[k], k
        assert abs(int(g["cg_iterations"]) - int(w["cg_iterations"])) <= 1
        assert close_be(g["be_4x4"], w["be_4x4"]) and close_be(g["be_2x2"], w["be_2x2"])
    m = seqio.RunManifest.from_json_string((tmp_path / "run_manifest.json").read_text())
    r = seqio.RunManifest.from_json_string((G / "solve" / "run_manifest.json").read_text())
    assert m.kind == "solve" and m.runs[0].stats == r.runs[0].stats
    for a, b in zip(m.runs[0].reports, r.runs[0].reports):
        assert a.factorization_attempts == b.factorization_attempts
        assert a.ruiz_iterations == b.ruiz_iterations
        assert a.symbolic_reused == b.symbolic_reused


def test_cmd_sweep_gamma_matches_reference(tmp_path):
    perm = np.load(G / "perm.npy")
    rc = seqio.cmd_sweep_gamma(G / "seq" / "manifest.json", [1e2, 1e4, 1e6], SolverConfig(), tmp_path, perm=perm)
    assert rc == seqio.EXIT_OK
    schema, got = rows(tmp_path / "sweep.csv")
    ref_schema, want = rows(G / "sweep" / "sweep.csv")
    assert schema == ref_schema and len(got) == len(want) == 9
    for g, w in zip(got, want):
        assert (g["gamma"], g["k"], g["delta1"]) == (w["gamma"], w["k"], w["delta1"])
        assert abs(int(g["cg_iterations"]) - int(w["cg_iterations"])) <= 1
        assert close_be(g["be_4x4"], w["be_4x4"])


def test_cli_entry_point_writes_reports(tmp_path):
    rc = seqio.main(["solve", str(G / "seq" / "manifest.json"), str(tmp_path)])
    assert rc == seqio.EXIT_OK
    assert (tmp_path / "solve.csv").exists() and (tmp_path / "run_manifest.json").exists()
