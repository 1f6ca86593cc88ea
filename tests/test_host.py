"""CPU: host-side analysis and the ACOPF generator (no GPU needed)."""
import numpy as np
import pytest

from paper_2110_03636_b200 import acopf
from paper_2110_03636_b200.solver import host_analyze


@pytest.mark.parametrize("nb", [60, 500, 2000])
def test_generator_sizes_follow_appendix_b(nb):
    s = acopf.generate(nb, 7, 7)
    nbr = round(1.3 * nb)
    ng = nb // 5
    assert s.n_x == 2 * nb + 4 * nbr + 2 * ng
    assert s.m_c == 2 * nb + 4 * nbr
    assert s.m_d == 2 * nbr
    assert s.h.nnz == nb + 6 * nbr + s.n_x
    assert s.j.nnz == 24 * nbr + 2 * ng
    assert s.j_d.nnz == 4 * nbr
    assert (s.h.rowidx >= s.h.col_of_entries()).all()  # lower storage


def test_generator_is_deterministic_and_pattern_shared():
    a, b = acopf.generate(300, 7, 7), acopf.generate(300, 7, 7)
    assert np.array_equal(a.h.values, b.h.values) and np.array_equal(a.r_y, b.r_y)
    c = acopf.generate(300, 7, 8)
    assert a.same_pattern_as(c) and not np.array_equal(a.h.values, c.h.values)
    seq = acopf.sequence(100, 3)
    assert all(x.same_pattern_as(seq[0]) for x in seq)


@pytest.mark.parametrize("nb", [60, 500])
def test_symbolic_counts_match_reference(ref, nb):
    s = acopf.generate(nb, 7, 7)
    perm = ref.hgamma_amd(s)
    st, used = host_analyze(s, perm)
    want = ref.pattern_stats(s, perm=perm)
    assert np.array_equal(used, perm)
    assert st["nnz_h_tilde"] == want["nnz_h_tilde"]
    assert st["nnz_h_gamma"] == want["nnz_h_gamma"]
    assert st["nnz_l"] == want["nnz_l"]
    assert st["etree_height"] == want["etree_height"]


def test_own_ordering_is_a_permutation_with_reasonable_fill(ref):
    s = acopf.generate(500, 7, 7)
    st, perm = host_analyze(s)
    assert sorted(perm.tolist()) == list(range(s.n_x))
    amd = ref.pattern_stats(s)
    assert st["nnz_l"] <= 1.25 * amd["nnz_l"]  # minimum degree vs the reference AMD


def test_reference_generator_patterns_analyse(ref):
    for seed in (23, 31):
        s = ref.generate(240, 60, 50, seed=seed)[0]
        perm = ref.hgamma_amd(s)
        st, _ = host_analyze(s, perm)
        assert st["nnz_l"] == ref.pattern_stats(s, perm=perm)["nnz_l"]


@pytest.mark.parametrize("nb,nchunk", [(60, 4), (120, 4), (500, 8), (2000, 8), (500, 16)])
def test_sys_stream_program_emulates_supernodal_solve(nb, nchunk):
    """The system-per-CTA stream program (sysplan.cpp): every substep reads
    only its resident ring window and the emulated solve equals a plain
    supernodal forward + backward solve."""
    from paper_2110_03636_b200.solver import sysplan_check
    s = acopf.generate(nb, 7, 7)
    st = sysplan_check(s, nchunk=nchunk)
    assert st["max_rel_err"] < 1e-12
    assert st["value_len"] % 1024 == 0 and st["index_len"] % 1024 == 0
    assert st["max_segs_per_step"] <= 1024


def test_sys_stream_program_wide_supernodes(ref):
    """Reference-generator patterns fill in (wide supernodes -> warp tasks
    and multi-substep segment regions)."""
    from paper_2110_03636_b200.solver import sysplan_check
    for seed in (23, 31):
        s = ref.generate(240, 60, 50, seed=seed)[0]
        st = sysplan_check(s, perm=ref.hgamma_amd(s), nchunk=16)
        assert st["max_rel_err"] < 1e-12
