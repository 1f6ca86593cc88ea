"""CPU: the C-ABI library loads, exports every symbol include/hykkt.h
declares, and rejects malformed input with status codes (no compute)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2110_03636_b200 import _lib
from paper_2110_03636_b200.kkt import BlockKkt4x4, CscMatrix
from paper_2110_03636_b200.solver import host_analyze

HEADER = Path(__file__).resolve().parents[1] / "include" / "hykkt.h"


def declared():
    src = HEADER.read_text()
    return sorted(set(re.findall(r"\b(hykkt_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    L = _lib.lib()
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(_lib.EXPORTS) <= set(names)


def test_config_defaults_mirror_reference():
    cfg = _lib.Config()
    _lib.lib().hykkt_config_default(C.byref(cfg))
    assert (cfg.gamma, cfg.delta_min, cfg.delta_max, cfg.delta2, cfg.cg_tol) == (1e4, 1e-9, 1e-6, 1e-9, 1e-12)
    assert (cfg.cg_max_iter, cfg.small_quadratic_threshold, cfg.pivot_floor) == (500, 1e-12, 1e-13)
    assert (cfg.ruiz_tol, cfg.ruiz_max_iters) == (0.01, 20)


def _tiny(h_rows=(0, 1, 1), h_cols=(0, 0, 1)):
    h = CscMatrix.from_triplets(2, 2, list(h_rows), list(h_cols), [4.0] * len(h_rows))
    j = CscMatrix.from_triplets(1, 2, [0, 0], [0, 1], [1.0, 1.0])
    jd = CscMatrix.empty(0, 2)
    z = np.zeros
    return BlockKkt4x4(h, j, jd, z(2), z(0), z(2), z(0), z(1), z(0))


def test_host_analyze_accepts_valid_input():
    st, perm = host_analyze(_tiny())
    assert st["n"] == 2 and sorted(perm.tolist()) == [0, 1]


def test_upper_triangle_input_is_rejected():
    s = _tiny()
    s.h = CscMatrix(2, 2, np.array([0, 2, 3]), np.array([0, 1, 1]), np.ones(3))
    s.h.rowidx = np.array([0, 1, 0])  # column 1 has row 0 < 1: not lower
    s.h.colptr = np.array([0, 1, 3])
    s.h.rowidx = np.array([0, 0, 1])
    with pytest.raises(_lib.InvalidMatrixError):
        host_analyze(s)


def test_unsorted_rows_are_rejected():
    s = _tiny()
    s.h = CscMatrix(2, 2, np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3))
    with pytest.raises(_lib.InvalidMatrixError):
        host_analyze(s)


def test_bad_permutation_is_rejected():
    with pytest.raises(_lib.InvalidMatrixError):
        host_analyze(_tiny(), perm=[0, 0])


def test_dimension_mismatch_is_rejected():
    s = _tiny()
    s.j = CscMatrix.from_triplets(1, 3, [0], [2], [1.0])
    with pytest.raises(_lib.InvalidMatrixError):
        host_analyze(s)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2110_03636_b200 import Device
    with pytest.raises(_lib.HykktError):
        Device(0)
