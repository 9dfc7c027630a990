"""CPU oracle for the SVM dual frontend -- TEST INFRASTRUCTURE ONLY.

The checker for ``paper_2308_00637_b200/svm.py`` (only ``tests/`` may import
it).  Restates, with the reference's numpy operations in the reference's
order (so results are bit-identical to ``qpipm.svm`` on the same inputs --
pinned by ``tests/test_oracle_golden.py::test_svm_*`` against
``tests/golden/svm.npz`` made by ``oracle/make_golden_svm.py``):

  gram_matrix        qpipm/svm.py:166-176  (_gram_matrix)
  dual_hessian       qpipm/svm.py:185      (np.outer(y, y) * gram)
  decision_values    qpipm/svm.py:194-196  (_decision_values)
  bias               qpipm/svm.py:198-205  (extract_model's bias rule)
  dual_problem       qpipm/svm.py:179-195  (build_svm_dual), as this package's
                     QpProblem so the oracle IPM (qp_oracle.solve) can run it
"""

from __future__ import annotations

import numpy as np


def gram_matrix(x: np.ndarray, sigma: float) -> np.ndarray:
    """svm.py:166-176: dense RBF Gram matrix, exactly symmetric."""
    sq = (x * x).sum(axis=1)
    g = x @ x.T
    g = 0.5 * (g + g.T)
    d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * g, 0.0)
    d2 = 0.5 * (d2 + d2.T)
    return np.exp(-d2 / (2.0 * sigma))


def dual_hessian(x: np.ndarray, y: np.ndarray, sigma: float) -> np.ndarray:
    """svm.py:185: H = outer(y, y) * K."""
    return np.outer(y, y) * gram_matrix(x, sigma)


def decision_values(x: np.ndarray, y: np.ndarray, sigma: float, alpha: np.ndarray) -> np.ndarray:
    """svm.py:194-196: g = K (alpha o y), without the bias."""
    return gram_matrix(x, sigma) @ (alpha * y)


def bias(x: np.ndarray, y: np.ndarray, sigma: float, c: float, alpha: np.ndarray) -> float:
    """svm.py:198-205: mean over free SVs, else the KKT interval midpoint."""
    tau = 1e-5 * c
    g = decision_values(x, y, sigma, alpha)
    free = np.where((alpha > tau) & (alpha < c - tau))[0]
    if len(free):
        return float(np.mean(y[free] - g[free]))
    upper_set = ((alpha <= tau) & (y > 0)) | ((alpha >= c - tau) & (y < 0))
    lower_set = ((alpha <= tau) & (y < 0)) | ((alpha >= c - tau) & (y > 0))
    cand = y - g
    hi = cand[upper_set].min() if np.any(upper_set) else cand.max()
    lo = cand[lower_set].max() if np.any(lower_set) else cand.min()
    return 0.5 * (lo + hi)


def dual_problem(x: np.ndarray, y: np.ndarray, sigma: float, c: float):
    """svm.py:179-195 as a host QpProblem with a DenseHessian."""
    from paper_2308_00637_b200.problem import Bounds, DenseHessian, QpProblem, SparseMatrix
    n = len(y)
    return QpProblem(
        n=n, hessian=DenseHessian(dual_hessian(x, y, sigma)), p=-np.ones(n),
        a=SparseMatrix.empty(0, n), lin_bounds=Bounds.free(0),
        c=SparseMatrix(1, n, np.array([0, n]), np.arange(n), y),
        b=np.zeros(1), var_bounds=Bounds(np.zeros(n), np.full(n, c)))


# the seeded generator lives with the other BASELINE-shaped generators
from paper_2308_00637_b200.workloads import svm_dual_data as synthetic_dataset  # noqa: E402,F401
