"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public benchmark or dataset is involved: every config is synthetic, and the
draw order below is fixed so that the GPU path and the CPU oracle see the
same arrays.  ``scale`` shrinks a config for parity
tests (the oracle must finish in seconds); ``scale=1`` is the BASELINE size.

Each generator returns ``(problem, state, meta)``: a QpProblem, an interior
IterateState that produces the operator the PCG sweep runs on, and a dict with
the seeds and sizes (recorded in the bench line).
"""

from __future__ import annotations

import numpy as np

from .problem import (Bounds, BoundIndexMap, DenseHessian, DiagonalHessian, IterateState,
                      QpProblem, SparseHessian, SparseMatrix)


def _state_from_initial(problem, lin_lower_slack=None):
    """The IPM starting point of qpipm/ipm.py:73-104 (unit multipliers)."""
    bmap = BoundIndexMap.from_problem(problem)
    lo, hi = problem.var_bounds.lower, problem.var_bounds.upper
    x = np.zeros(problem.n)
    flo, fhi = np.isfinite(lo), np.isfinite(hi)
    x[flo & fhi] = 0.5 * (lo[flo & fhi] + hi[flo & fhi])
    x[flo & ~fhi] = lo[flo & ~fhi] + 1.0
    x[~flo & fhi] = hi[~flo & fhi] - 1.0
    a = problem.a
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_offsets))
    ax = np.bincount(rows, weights=a.values * x[a.col_indices], minlength=a.n_rows) if a.nnz else np.zeros(a.n_rows)

    def slack(gap):
        return np.maximum(1.0, np.abs(gap))

    ll, lu = problem.lin_bounds.lower, problem.lin_bounds.upper
    return IterateState(
        x=x,
        s_lA=slack(ax[bmap.lin_lower] - ll[bmap.lin_lower]) if lin_lower_slack is None else lin_lower_slack,
        s_uA=slack(lu[bmap.lin_upper] - ax[bmap.lin_upper]),
        s_lx=slack(x[bmap.var_lower] - lo[bmap.var_lower]),
        s_ux=slack(hi[bmap.var_upper] - x[bmap.var_upper]),
        lam_e=np.zeros(problem.m_eq),
        lam_lA=np.ones(len(bmap.lin_lower)), lam_uA=np.ones(len(bmap.lin_upper)),
        lam_lx=np.ones(len(bmap.var_lower)), lam_ux=np.ones(len(bmap.var_upper)),
        mu=1.0)


def dense_qp(seed: int = 0, n: int = 200, m: int = 400):
    """Config 1: dense random convex QP, H = Q'Q + 1e-2 I, Ax >= A x0 - s0."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, n))
    c = rng.standard_normal(n)
    a = rng.standard_normal((m, n)) / np.sqrt(n)
    x0 = rng.standard_normal(n)
    s0 = rng.uniform(0.1, 1.0, m)
    problem = QpProblem(
        n=n, hessian=DenseHessian(q.T @ q + 1e-2 * np.eye(n)), p=c,
        a=SparseMatrix.from_dense(a), lin_bounds=Bounds(a @ x0 - s0, np.full(m, np.inf)),
        c=SparseMatrix.empty(0, n), b=np.zeros(0), var_bounds=Bounds.free(n))
    return problem, _state_from_initial(problem), dict(config="cfg1", seed=seed, n=n, m=m)


def svm_primal(seed: int = 2, d: int = 500, n_samples: int = 50_000, c_reg: float = 1.0):
    """Config 2: soft-margin linear SVM primal; A = [diag(y)X, y, I], 502 nnz/row."""
    rng = np.random.default_rng(seed)
    y_true = np.repeat([1.0, -1.0], [n_samples - n_samples // 2, n_samples // 2])
    rng.shuffle(y_true)
    x = rng.standard_normal((n_samples, d)) + y_true[:, None] * (0.5 / np.sqrt(d))
    flip = rng.random(n_samples) < 0.1
    y = np.where(flip, -y_true, y_true)
    n = d + 1 + n_samples
    per_row = d + 2
    cols = np.empty((n_samples, per_row), dtype=np.int64)
    cols[:, :d] = np.arange(d)
    cols[:, d] = d
    cols[:, d + 1] = d + 1 + np.arange(n_samples)
    vals = np.empty((n_samples, per_row))
    vals[:, :d] = y[:, None] * x
    vals[:, d] = y
    vals[:, d + 1] = 1.0
    a = SparseMatrix(n_samples, n, np.arange(n_samples + 1, dtype=np.int64) * per_row,
                     cols.ravel(), vals.ravel())
    hd = np.concatenate([np.ones(d), [0.0], np.zeros(n_samples)])
    p = np.concatenate([np.zeros(d + 1), np.full(n_samples, c_reg)])
    lx = np.concatenate([np.full(d + 1, -np.inf), np.zeros(n_samples)])
    problem = QpProblem(
        n=n, hessian=DiagonalHessian(hd), p=p, a=a,
        lin_bounds=Bounds(np.ones(n_samples), np.full(n_samples, np.inf)),
        c=SparseMatrix.empty(0, n), b=np.zeros(0),
        var_bounds=Bounds(lx, np.full(n, np.inf)))
    return problem, _state_from_initial(problem), dict(config="cfg2", seed=seed, d=d, n_samples=n_samples)


def rt_like(seed: int = 3, n_vox: int = 200_000, n_beam: int = 20_000, density: float = 0.005,
            target_frac: float = 0.2, dose_target: float = 60.0, dose_max: float = 20.0):
    """Configs 3/4: radiation-therapy-like QP.

    Each beamlet column j has a contiguous voxel band [s_j, s_j + L), L =
    density * n_vox, with values exp(-r/5) * U(0.5, 1) where r = 0..L-1 is the
    voxel offset within the band (unit: one voxel; most values are therefore
    tiny, as SURVEY.md 7.3-9 notes).  The first target_frac of the voxels are
    targets: H = sym(D_t' D_t), p = -dose_target * D_t' 1.  The rest are
    organs at risk: D_oar x <= dose_max, plus x >= 0.
    """
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    band = max(1, int(round(density * n_vox)))
    starts = rng.integers(0, n_vox - band + 1, size=n_beam)
    r = np.arange(band, dtype=np.float64)
    vals = np.exp(-r / 5.0)[None, :] * rng.uniform(0.5, 1.0, size=(n_beam, band))
    # column j holds the rows starts[j] .. starts[j] + band - 1 (no duplicates):
    # that IS a CSC matrix; its CSR conversion is one counting pass and leaves
    # the column indices of every row sorted (same arrays as building it from
    # COO triplets, without their sort)
    rows = starts[:, None] + np.arange(band)[None, :]
    dmat = sp.csc_matrix((vals.ravel(), rows.ravel(), np.arange(n_beam + 1, dtype=np.int64) * band),
                         shape=(n_vox, n_beam)).tocsr()
    n_t = int(round(target_frac * n_vox))
    d_t = dmat[:n_t]
    d_oar = dmat[n_t:].tocsr()
    d_oar.sort_indices()
    hm = (d_t.T @ d_t).tocsr()
    hm = ((hm + hm.T) * 0.5).tocsr()
    hm.sum_duplicates()
    hm.sort_indices()
    p = -dose_target * np.asarray(d_t.T @ np.ones(n_t)).ravel()
    m = d_oar.shape[0]
    problem = QpProblem(
        n=n_beam, hessian=SparseHessian(SparseMatrix(n_beam, n_beam, hm.indptr, hm.indices, hm.data)),
        p=p, a=SparseMatrix(m, n_beam, d_oar.indptr, d_oar.indices, d_oar.data),
        lin_bounds=Bounds(np.full(m, -np.inf), np.full(m, dose_max)),
        c=SparseMatrix.empty(0, n_beam), b=np.zeros(0),
        var_bounds=Bounds(np.zeros(n_beam), np.full(n_beam, np.inf)))
    meta = dict(config="cfg3" if n_vox <= 200_000 else "cfg4", seed=seed, n_vox=n_vox,
                n_beam=n_beam, band=band, nnz_A=int(d_oar.nnz), nnz_H=int(hm.nnz))
    return problem, _state_from_initial(problem), meta


def random_sweep(seed: int = 5, m: int = 4_000_000, n: int = 1_000_000, per_row: int = 16,
                 log10_w_spread: float = 6.0):
    """Config 5: random CSR A (m x n, per_row distinct columns per row, N(0,1)),
    H = diag(U(1e-2, 1)), W with log10 w ~ U(-spread, spread) via s_lA = w,
    lambda_lA = 1 (so build_operator yields d_diag = w, kkt.py:200), Ax >= 0.

    Draw order: column indices (rows with a repeated column are redrawn until
    none remain), values, h, log10 w, rhs.
    """
    if per_row > n:
        raise ValueError(f"cannot draw {per_row} distinct columns out of {n}")
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, n, size=(m, per_row), dtype=np.int64)
    cols.sort(axis=1)
    while True:
        dup = np.nonzero(np.any(cols[:, 1:] == cols[:, :-1], axis=1))[0]
        if len(dup) == 0:
            break
        redraw = rng.integers(0, n, size=(len(dup), per_row), dtype=np.int64)
        redraw.sort(axis=1)
        cols[dup] = redraw
    vals = rng.standard_normal(m * per_row)
    h = rng.uniform(1e-2, 1.0, n)
    w = 10.0 ** rng.uniform(-log10_w_spread, log10_w_spread, m)
    rhs = rng.standard_normal(n + m)
    a = SparseMatrix(m, n, np.arange(m + 1, dtype=np.int64) * per_row, cols.ravel(), vals)
    problem = QpProblem(
        n=n, hessian=DiagonalHessian(h), p=np.zeros(n), a=a,
        lin_bounds=Bounds(np.zeros(m), np.full(m, np.inf)),
        c=SparseMatrix.empty(0, n), b=np.zeros(0), var_bounds=Bounds.free(n))
    state = IterateState(
        x=np.zeros(n), s_lA=w, s_uA=np.zeros(0), s_lx=np.zeros(0), s_ux=np.zeros(0),
        lam_e=np.zeros(0), lam_lA=np.ones(m), lam_uA=np.zeros(0), lam_lx=np.zeros(0),
        lam_ux=np.zeros(0), mu=1.0)
    meta = dict(config="cfg5", seed=seed, m=m, n=n, per_row=per_row, nnz=m * per_row,
                rhs=rhs)
    return problem, state, meta


CONFIGS = {
    "cfg1": dense_qp,
    "cfg2": svm_primal,
    "cfg3": rt_like,
    "cfg4": lambda seed=4, **kw: rt_like(seed=seed, n_vox=2_000_000, n_beam=100_000,
                                          density=0.001, **kw),
    "cfg5": random_sweep,
}


def svm_dual_data(seed: int = 6, n: int = 20_000, d: int = 100, sep: float = 1.0, noise: float = 0.1):
    """Samples for the kernel-SVM dual (qpipm/svm.py:179-195): two Gaussian
    classes with means +-(sep/2)/sqrt(d) * 1, identity covariance, balanced
    +-1 labels with a fraction `noise` flipped -- the class model of
    BASELINE.json configs[1], at the dual frontend's dense-kernel cap
    (MAX_PRECOMPUTED_SAMPLES = 20,000, svm.py:11) by default.
    Returns (X dense n x d, y)."""
    rng = np.random.default_rng(seed)
    y = np.where(rng.permutation(n) < n // 2, 1.0, -1.0)
    x = rng.standard_normal((n, d)) + y[:, None] * (0.5 * sep / np.sqrt(d))
    flip = rng.permutation(n)[: int(noise * n)]
    y = y.copy()
    y[flip] = -y[flip]
    return x, y
