"""Host-side containers for the data that crosses the direction-solver boundary.

These mirror the reference's problem and operator types field for field so
that an object built here and one built by ``qpipm`` are interchangeable at
the boundary (the GPU solver reads them by attribute, never by type):

* ``SparseMatrix``  -- qpipm/model.py:17-95 (CSR, strictly increasing columns
  per row; the reference's per-row Python check is replaced by a vectorised one)
* ``DiagonalHessian`` / ``SparseHessian`` / ``DenseHessian`` /
  ``QuasiNewtonHessian`` -- model.py:98-162
* ``Bounds`` / ``QpProblem`` -- model.py:189-258
* ``BoundIndexMap`` -- kkt.py:19-41
* ``IterateState`` -- kkt.py:44-69
* ``KktOperator`` + ``build_operator`` -- kkt.py:146-208.  Only the diagonal
  data (``q_diag_extra``, ``d_diag``) is produced; the reference's per-iteration
  ``row_submatrix`` copies (kkt.py:206-207) are not made -- the device keeps one
  resident copy of B per problem.

Nothing here computes on the hot path; the arithmetic is in ``csrc/``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np


class DimensionError(ValueError):
    """Operand shapes are inconsistent (qpipm/model.py:13-14)."""


@dataclass(frozen=True, eq=False)
class SparseMatrix:
    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        ro = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(self.col_indices, dtype=np.int64)
        vals = np.ascontiguousarray(self.values, dtype=np.float64)
        object.__setattr__(self, "row_offsets", ro)
        object.__setattr__(self, "col_indices", ci)
        object.__setattr__(self, "values", vals)
        if ro.shape != (self.n_rows + 1,):
            raise DimensionError("row_offsets must have length n_rows + 1")
        if ro[0] != 0 or ro[-1] != len(vals):
            raise ValueError("row_offsets must start at 0 and end at nnz")
        if np.any(np.diff(ro) < 0):
            raise ValueError("row_offsets must be nondecreasing")
        if len(ci) != len(vals):
            raise DimensionError("col_indices and values must have equal length")
        if len(ci) and (ci.min() < 0 or ci.max() >= self.n_cols):
            raise ValueError("column index out of range")
        if len(ci) > 1:
            # strictly increasing inside each row: every adjacent pair that is
            # not separated by a row boundary must increase
            inc = np.diff(ci) > 0
            boundary = np.zeros(len(ci) - 1, dtype=bool)
            starts = ro[1:-1]
            starts = starts[(starts > 0) & (starts < len(ci))]
            boundary[starts - 1] = True
            bad = np.nonzero(~inc & ~boundary)[0]
            if len(bad):
                row = int(np.searchsorted(ro, bad[0], side="right") - 1)
                raise ValueError(f"column indices not strictly increasing in row {row}")

    @classmethod
    def from_dense(cls, a) -> "SparseMatrix":
        a = np.asarray(a, dtype=np.float64)
        rows, cols = np.nonzero(a)
        ro = np.zeros(a.shape[0] + 1, dtype=np.int64)
        np.add.at(ro, rows + 1, 1)
        return cls(a.shape[0], a.shape[1], np.cumsum(ro), cols, a[rows, cols])

    @classmethod
    def empty(cls, n_rows: int, n_cols: int) -> "SparseMatrix":
        return cls(n_rows, n_cols, np.zeros(n_rows + 1, dtype=np.int64),
                   np.zeros(0, dtype=np.int64), np.zeros(0))

    @property
    def nnz(self) -> int:
        return len(self.values)

    def row_submatrix_arrays(self, rows):
        """(row_offsets, col_indices, values) of the given rows, in order."""
        rows = np.asarray(rows, dtype=np.int64)
        lens = self.row_offsets[rows + 1] - self.row_offsets[rows]
        ro = np.zeros(len(rows) + 1, dtype=np.int64)
        np.cumsum(lens, out=ro[1:])
        if ro[-1] == 0:
            return ro, np.zeros(0, np.int64), np.zeros(0)
        # gather index: for output slot k in row i -> row_offsets[rows[i]] + (k - ro[i])
        starts = np.repeat(self.row_offsets[rows] - ro[:-1], lens)
        idx = starts + np.arange(ro[-1], dtype=np.int64)
        return ro, self.col_indices[idx], self.values[idx]


@dataclass(frozen=True, eq=False)
class DiagonalHessian:
    d: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "d", np.ascontiguousarray(self.d, dtype=np.float64))

    @property
    def n(self):
        return len(self.d)


@dataclass(frozen=True, eq=False)
class SparseHessian:
    """Symmetric sparse Hessian; full (not triangular) CSR storage."""
    m: SparseMatrix

    @property
    def n(self):
        return self.m.n_rows


@dataclass(frozen=True, eq=False)
class DenseHessian:
    m: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "m", np.ascontiguousarray(self.m, dtype=np.float64))

    @property
    def n(self):
        return self.m.shape[0]


@dataclass(frozen=True, eq=False)
class QuasiNewtonHessian:
    """H = diag(h0) + U diag(w) U^T (model.py:144-162)."""
    h0_diag: np.ndarray
    u: np.ndarray
    w: np.ndarray

    def __post_init__(self):
        h0 = np.ascontiguousarray(self.h0_diag, dtype=np.float64)
        u = np.ascontiguousarray(self.u, dtype=np.float64)
        w = np.ascontiguousarray(self.w, dtype=np.float64)
        if u.ndim != 2 or u.shape[0] != len(h0) or u.shape[1] != len(w):
            raise DimensionError("update matrix must be n x k with k weights")
        object.__setattr__(self, "h0_diag", h0)
        object.__setattr__(self, "u", u)
        object.__setattr__(self, "w", w)

    @property
    def n(self):
        return len(self.h0_diag)


Hessian = Union[DiagonalHessian, SparseHessian, DenseHessian, QuasiNewtonHessian]


@dataclass(frozen=True, eq=False)
class Bounds:
    lower: np.ndarray
    upper: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lower, dtype=np.float64)
        hi = np.asarray(self.upper, dtype=np.float64)
        if lo.shape != hi.shape:
            raise DimensionError("lower and upper must have equal length")
        object.__setattr__(self, "lower", lo)
        object.__setattr__(self, "upper", hi)

    def __len__(self):
        return len(self.lower)

    @classmethod
    def free(cls, n: int) -> "Bounds":
        return cls(np.full(n, -np.inf), np.full(n, np.inf))


@dataclass(frozen=True, eq=False)
class QpProblem:
    """min 1/2 x'Hx + p'x  s.t.  l <= Ax <= u, Cx = b, lx <= x <= ux."""
    n: int
    hessian: Hessian
    p: np.ndarray
    a: SparseMatrix
    lin_bounds: Bounds
    c: SparseMatrix
    b: np.ndarray
    var_bounds: Bounds

    def __post_init__(self):
        object.__setattr__(self, "p", np.asarray(self.p, dtype=np.float64))
        object.__setattr__(self, "b", np.asarray(self.b, dtype=np.float64))

    @property
    def m_lin(self) -> int:
        return self.a.n_rows

    @property
    def m_eq(self) -> int:
        return self.c.n_rows


@dataclass(frozen=True, eq=False)
class BoundIndexMap:
    lin_lower: np.ndarray
    lin_upper: np.ndarray
    var_lower: np.ndarray
    var_upper: np.ndarray

    @classmethod
    def from_problem(cls, problem) -> "BoundIndexMap":
        return cls(
            lin_lower=np.where(np.isfinite(problem.lin_bounds.lower))[0],
            lin_upper=np.where(np.isfinite(problem.lin_bounds.upper))[0],
            var_lower=np.where(np.isfinite(problem.var_bounds.lower))[0],
            var_upper=np.where(np.isfinite(problem.var_bounds.upper))[0],
        )

    @property
    def m_lin_lower(self):
        return len(self.lin_lower)

    @property
    def m_lin_upper(self):
        return len(self.lin_upper)


@dataclass(eq=False)
class IterateState:
    x: np.ndarray
    s_lA: np.ndarray
    s_uA: np.ndarray
    s_lx: np.ndarray
    s_ux: np.ndarray
    lam_e: np.ndarray
    lam_lA: np.ndarray
    lam_uA: np.ndarray
    lam_lx: np.ndarray
    lam_ux: np.ndarray
    mu: float


@dataclass(frozen=True, eq=False)
class KktOperator:
    """Diagonal data of [[Q + 2B'D^{-1}B, B'], [B, D]] for one IPM iteration.

    Q = H + diag(q_diag_extra); B = (C; A_l; -A_u); D = diag(d_diag).
    """
    problem: QpProblem
    bmap: BoundIndexMap
    q_diag_extra: np.ndarray
    d_diag: np.ndarray

    @property
    def n(self) -> int:
        return self.problem.n

    @property
    def m(self) -> int:
        return len(self.d_diag)

    @property
    def dim(self) -> int:
        return self.n + self.m

    def split(self, v):
        return v[:self.n], v[self.n:]


def build_operator(problem, state, bmap=None) -> KktOperator:
    """Diagonal data for one IPM iteration (kkt.py:190-202)."""
    if bmap is None:
        bmap = BoundIndexMap.from_problem(problem)
    q_extra = np.zeros(problem.n)
    np.add.at(q_extra, bmap.var_lower, state.lam_lx / state.s_lx)
    np.add.at(q_extra, bmap.var_upper, state.lam_ux / state.s_ux)
    d_diag = np.concatenate([
        np.full(problem.m_eq, state.mu),
        state.s_lA / state.lam_lA,
        state.s_uA / state.lam_uA,
    ])
    return KktOperator(problem=problem, bmap=bmap, q_diag_extra=q_extra, d_diag=d_diag)
