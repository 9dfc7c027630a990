"""Rebuild golden-fixture instances (tests/golden/*.npz) as package objects."""

from pathlib import Path

import numpy as np

from paper_2308_00637_b200.problem import (Bounds, DenseHessian, DiagonalHessian, IterateState,
                                           QpProblem, QuasiNewtonHessian, SparseHessian, SparseMatrix,
                                           build_operator)

GOLDEN = Path(__file__).resolve().parent / "golden"
STATE_KEYS = ("x", "s_lA", "s_uA", "s_lx", "s_ux", "lam_e", "lam_lA", "lam_uA", "lam_lx", "lam_ux")


def load(name):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def problem_from(z, pre):
    n = int(z[pre + "n"])
    mats = {}
    for name in ("a", "c"):
        r, c = z[pre + name + "_shape"]
        mats[name] = SparseMatrix(int(r), int(c), z[pre + name + "_ro"], z[pre + name + "_ci"], z[pre + name + "_v"])
    kind = str(z[pre + "hkind"])
    if kind == "DiagonalHessian":
        h = DiagonalHessian(z[pre + "h_d"])
    elif kind == "SparseHessian":
        h = SparseHessian(SparseMatrix(n, n, z[pre + "h_ro"], z[pre + "h_ci"], z[pre + "h_v"]))
    elif kind == "DenseHessian":
        h = DenseHessian(z[pre + "h_m"])
    else:
        h = QuasiNewtonHessian(z[pre + "h_h0"], z[pre + "h_u"], z[pre + "h_w"])
    return QpProblem(n=n, hessian=h, p=z[pre + "p"], a=mats["a"],
                     lin_bounds=Bounds(z[pre + "lin_lo"], z[pre + "lin_hi"]), c=mats["c"], b=z[pre + "b"],
                     var_bounds=Bounds(z[pre + "var_lo"], z[pre + "var_hi"]))


def state_from(z, pre):
    return IterateState(**{k: np.array(z[pre + "st_" + k]) for k in STATE_KEYS}, mu=float(z[pre + "st_mu"]))


def instance(z, i):
    pre = f"i{i}_"
    problem = problem_from(z, pre)
    state = state_from(z, pre)
    return problem, state, build_operator(problem, state), pre
