"""Host-side value types mirroring the reference's (plain numpy arrays).

CscMatrix      <- hkkt::CscMatrix   (proj/core/include/hkkt/csc_matrix.hpp:41-94)
BlockKkt4x4    <- hkkt::BlockKkt4x4 (proj/core/include/hkkt/kkt_system.hpp:31-50)
FullSolution   <- hkkt::FullSolution (kkt_system.hpp:66-71)
Reduced2x2     <- hkkt::Reduced2x2 (kkt_system.hpp:56-64)
HGammaSystem   <- hkkt::HGammaSystem (solver.hpp:69-73)

Indices are int64 like the reference (csc_matrix.hpp:25); the device path
narrows them to int32 at the C-ABI boundary.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np


@dataclass
class CscMatrix:
    nrows: int
    ncols: int
    colptr: np.ndarray
    rowidx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowidx.shape[0])

    @staticmethod
    def empty(nrows: int, ncols: int) -> "CscMatrix":
        return CscMatrix(nrows, ncols, np.zeros(ncols + 1, np.int64), np.zeros(0, np.int64),
                         np.zeros(0, np.float64))

    @staticmethod
    def from_triplets(nrows, ncols, rows, cols, vals) -> "CscMatrix":
        """Sorted CSC, duplicates summed (CscMatrix::from_triplets,
        csc_matrix.cpp:81-132)."""
        rows = np.asarray(rows, np.int64)
        cols = np.asarray(cols, np.int64)
        vals = np.asarray(vals, np.float64)
        if rows.size and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0 or cols.max() >= ncols):
            raise ValueError("triplet outside matrix")
        order = np.lexsort((rows, cols))  # stable: by col, then row
        r, c, v = rows[order], cols[order], vals[order]
        if r.size:
            key_change = np.ones(r.size, bool)
            key_change[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            starts = np.flatnonzero(key_change)
            summed = np.add.reduceat(v, starts)
            r, c, v = r[starts], c[starts], summed
        colptr = np.zeros(ncols + 1, np.int64)
        np.add.at(colptr, c + 1, 1)
        colptr = np.cumsum(colptr)
        return CscMatrix(nrows, ncols, colptr, r.astype(np.int64), v.astype(np.float64))

    def with_values(self, values) -> "CscMatrix":
        return replace(self, values=np.ascontiguousarray(values, np.float64))

    def same_pattern_as(self, o: "CscMatrix") -> bool:
        return (self.nrows == o.nrows and self.ncols == o.ncols and
                np.array_equal(self.colptr, o.colptr) and np.array_equal(self.rowidx, o.rowidx))

    def col_of_entries(self) -> np.ndarray:
        return np.repeat(np.arange(self.ncols, dtype=np.int64), np.diff(self.colptr))

    def to_dense(self, symmetric_lower: bool = False) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        cols = self.col_of_entries()
        np.add.at(d, (self.rowidx, cols), self.values)
        if symmetric_lower:
            off = self.rowidx != cols
            np.add.at(d, (cols[off], self.rowidx[off]), self.values[off])
        return d


@dataclass
class BlockKkt4x4:
    h: CscMatrix      # n_x x n_x, lower triangle
    j: CscMatrix      # m_c x n_x
    j_d: CscMatrix    # m_d x n_x
    d_x: np.ndarray
    d_s: np.ndarray
    r_tilde_x: np.ndarray
    r_s: np.ndarray
    r_y: np.ndarray
    r_yd: np.ndarray

    @property
    def n_x(self) -> int:
        return self.h.ncols

    @property
    def m_c(self) -> int:
        return self.j.nrows

    @property
    def m_d(self) -> int:
        return self.j_d.nrows

    @property
    def total_size(self) -> int:
        return self.n_x + 2 * self.m_d + self.m_c

    def stacked_rhs(self) -> np.ndarray:
        return np.concatenate([self.r_tilde_x, self.r_s, self.r_y, self.r_yd])

    def same_pattern_as(self, o: "BlockKkt4x4") -> bool:
        return (self.h.same_pattern_as(o.h) and self.j.same_pattern_as(o.j)
                and self.j_d.same_pattern_as(o.j_d))


@dataclass
class FullSolution:
    dx: np.ndarray
    ds: np.ndarray
    dy: np.ndarray
    dyd: np.ndarray

    def stacked(self) -> np.ndarray:
        return np.concatenate([self.dx, self.ds, self.dy, self.dyd])


@dataclass
class Reduced2x2:
    """[[H_tilde, J^T], [J, 0]] with right-hand side (r_x, r_y); H_tilde
    lower triangle with its full diagonal."""
    h_tilde: CscMatrix
    j: CscMatrix
    r_x: np.ndarray
    r_y: np.ndarray

    @property
    def n_x(self) -> int:
        return self.h_tilde.ncols

    @property
    def m_c(self) -> int:
        return self.j.nrows

    def same_pattern_as(self, o: "Reduced2x2") -> bool:
        return self.h_tilde.same_pattern_as(o.h_tilde) and self.j.same_pattern_as(o.j)


@dataclass
class HGammaSystem:
    h_gamma: CscMatrix  # lower triangle
    r_hat_x: np.ndarray
    gamma_used: float = 0.0
