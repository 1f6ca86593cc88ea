"""The sequence IO surface (paper_2110_03636_b200/seqio.py) against files the
reference itself wrote (tests/golden/seq_ref/, made by
tests/golden/make_seq_golden.sh from proj/core/src/manifest.cpp,
matrix_market.cpp and driver.cpp): loading, byte-identical re-writing of the
manifest / Matrix Market / vector files, the run manifest and both CSV
reports, and the reference's error conventions.  CPU only."""
from pathlib import Path

import numpy as np
import pytest

from paper_2110_03636_b200 import seqio

G = Path(__file__).resolve().parent / "golden" / "seq_ref"


def test_load_reference_sequence():
    systems, uniform = seqio.load_sequence(G / "seq" / "manifest.json")
    assert len(systems) == 3 and uniform
    s = systems[0]
    assert (s.n_x, s.m_c, s.m_d) == (60, 15, 12)
    assert s.h.nnz == 186 and np.all(s.h.rowidx >= s.h.col_of_entries())
    assert s.d_x.shape == (60,) and s.r_yd.shape == (12,)
    # drifted values, one pattern
    assert not np.array_equal(systems[0].h.values, systems[1].h.values)


def test_save_sequence_is_byte_identical_to_reference(tmp_path):
    systems, _ = seqio.load_sequence(G / "seq" / "manifest.json")
    seqio.save_sequence(tmp_path, systems)
    ref_files = sorted(p.name for p in (G / "seq").iterdir())
    assert sorted(p.name for p in tmp_path.iterdir()) == ref_files
    for name in ref_files:
        assert (tmp_path / name).read_bytes() == (G / "seq" / name).read_bytes(), name


@pytest.mark.parametrize("kind", ["solve", "sweep"])
def test_run_manifest_and_csv_round_trip_reference_bytes(kind):
    text = (G / kind / "run_manifest.json").read_text()
    m = seqio.RunManifest.from_json_string(text)
    assert m.kind == kind
    assert m.to_json_string() + "\n" == text
    assert seqio.csv_text(m) == (G / kind / f"{kind}.csv").read_text()


def test_matrix_market_round_trip_and_duplicates(tmp_path):
    p = tmp_path / "a.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n% comment\n3 2 4\n1 1 1.5\n3 2 -2\n"
                 "1 1 0.25\n2 1 1e-3\n")
    a, sym = seqio.read_matrix_market(p)
    assert not sym and (a.nrows, a.ncols, a.nnz) == (3, 2, 3)
    assert np.allclose(a.to_dense(), [[1.75, 0], [1e-3, 0], [0, -2]])
    seqio.write_matrix_market(tmp_path / "b.mtx", a, False)
    b, _ = seqio.read_matrix_market(tmp_path / "b.mtx")
    assert np.array_equal(b.values, a.values) and np.array_equal(b.rowidx, a.rowidx)


@pytest.mark.parametrize("body,msg", [
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n", "upper-triangle"),
    ("MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n", "banner"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", "declared"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", "out of range"),
])
def test_matrix_market_errors(tmp_path, body, msg):
    p = tmp_path / "bad.mtx"
    p.write_text(body)
    with pytest.raises(seqio.MatrixMarketError, match=msg):
        seqio.read_matrix_market(p)


def test_manifest_errors_are_usage_exit_codes(tmp_path):
    bad = tmp_path / "manifest.json"
    bad.write_text('{"version": 1, "systems": [{"n_x": 61, "m_c": 15, "m_d": 12, "H": "%s", "J": "%s", '
                   '"J_d": "%s", "vectors": "%s"}]}' % tuple(str(G / "seq" / f) for f in
                                                            ("sys0_H.mtx", "sys0_J.mtx", "sys0_Jd.mtx",
                                                             "sys0_vectors.json")))
    with pytest.raises(seqio.ManifestError, match="dimensions"):
        seqio.load_sequence(bad)
    assert seqio.cmd_solve(bad, seqio.SolverConfig(), tmp_path / "out") == seqio.EXIT_USAGE
    empty = tmp_path / "empty.json"
    empty.write_text('{"version": 1, "systems": []}')
    assert seqio.cmd_solve(empty, seqio.SolverConfig(), tmp_path / "out") == seqio.EXIT_USAGE
