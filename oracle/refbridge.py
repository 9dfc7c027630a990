"""Package objects -> reference (`qpipm`) objects.  TEST INFRASTRUCTURE ONLY.

The seeded generators (paper_2308_00637_b200/workloads.py) build the package's
mirror types; the reference wants its own classes.  Field-for-field
conversion, no arithmetic.  Used by tests/ and bench.py's reference legs.
"""

from __future__ import annotations

import numpy as np

from . import build_ref

STATE_KEYS = ("x", "s_lA", "s_uA", "s_lx", "s_ux", "lam_e", "lam_lA", "lam_uA", "lam_lx", "lam_ux")


def ref_sparse(model, m):
    # the arrays were validated by the package's vectorised constructor; the
    # reference constructor's per-row Python loop (model.py:48-51) would take
    # minutes on 2e8 nonzeros, so the frozen dataclass is filled directly
    obj = object.__new__(model.SparseMatrix)
    object.__setattr__(obj, "n_rows", int(m.n_rows))
    object.__setattr__(obj, "n_cols", int(m.n_cols))
    object.__setattr__(obj, "row_offsets", np.asarray(m.row_offsets, dtype=np.int64))
    object.__setattr__(obj, "col_indices", np.asarray(m.col_indices, dtype=np.int64))
    object.__setattr__(obj, "values", np.asarray(m.values, dtype=np.float64))
    return obj


def ref_problem(p):
    qp = build_ref.import_qpipm()
    model = qp.model
    h = p.hessian
    kind = type(h).__name__
    if kind == "DiagonalHessian":
        rh = model.DiagonalHessian(h.d)
    elif kind == "SparseHessian":
        rh = model.SparseHessian(ref_sparse(model, h.m))
    elif kind == "DenseHessian":
        rh = model.DenseHessian(h.m)
    elif kind == "QuasiNewtonHessian":
        rh = model.QuasiNewtonHessian(h.h0_diag, h.u, h.w)
    else:
        raise TypeError(kind)
    return model.QpProblem(
        n=p.n, hessian=rh, p=p.p, a=ref_sparse(model, p.a),
        lin_bounds=model.Bounds(p.lin_bounds.lower, p.lin_bounds.upper),
        c=ref_sparse(model, p.c), b=p.b,
        var_bounds=model.Bounds(p.var_bounds.lower, p.var_bounds.upper))


def ref_state(s):
    qp = build_ref.import_qpipm()
    return qp.kkt.IterateState(**{k: np.array(getattr(s, k), dtype=np.float64) for k in STATE_KEYS}, mu=s.mu)


def ref_operator(problem, state):
    """The reference's KktOperator of a package (problem, state)."""
    qp = build_ref.import_qpipm()
    return qp.kkt.build_operator(ref_problem(problem), ref_state(state))
