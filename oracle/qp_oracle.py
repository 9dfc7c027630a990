"""CPU oracle for the Jacobi-PCG hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference leg
may import it.  It restates, in numpy + scipy (the same third-party kernels
the reference calls: ``scipy.sparse`` csr/csc matvec, numpy dot/norm), the
reference algorithm of ``qpipm`` (``/root/reference/pkg/src/qpipm``), with
the operation order of each reference line kept so that its results are
bit-identical to the reference on the same inputs.  That claim is pinned by
``tests/test_oracle_golden.py`` against fixtures produced by running the
real reference (``oracle/make_golden.py``).

Third-party arithmetic the reference depends on (absent from /root/reference,
pins are floors only -- pkg/pyproject.toml:10-13 ``numpy>=1.24``,
``scipy>=1.10``): numpy 2.3.5 / scipy 1.18.1 in this image.

Restated functions (reference file:line):
  hessian_apply / hessian_diagonal    model.py:165-186
  b_blocks / apply_b / apply_bt        kkt.py:177-184 (+ build_operator's
                                       row_submatrix copies, kkt.py:206-207)
  apply_doubly_augmented              kkt.py:211-221
  jacobi_diagonal                     kkt.py:224-239
  pcg                                 linalg.py:66-133
  pcg_direction                       ipm.py:179-182
  IPM loop (initialize, residuals, rhs, recover, ratio test, step,
  infeasibilities, barrier update, solve)
                                      ipm.py:73-240, kkt.py:113-143, 242-284
The IPM loop is here only so IPM-level parity of the GPU direction solver can
be checked on the GPU box, where the reference package is not installed.
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import scipy.sparse as sp


# ----------------------------------------------------------------------------
# model.py:165-186
def hessian_apply(h, v):
    kind = type(h).__name__
    if kind == "DiagonalHessian":
        return h.d * v
    if kind == "SparseHessian":
        return _csr(h.m) @ v
    if kind == "DenseHessian":
        return h.m @ v
    return h.h0_diag * v + h.u @ (h.w * (h.u.T @ v))


def hessian_diagonal(h):
    kind = type(h).__name__
    if kind == "DiagonalHessian":
        return h.d.copy()
    if kind == "SparseHessian":
        return np.asarray(_csr(h.m).diagonal())
    if kind == "DenseHessian":
        return np.diag(h.m).copy()
    return h.h0_diag + (h.w * h.u ** 2).sum(axis=1)


_CSR_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _csr(m) -> sp.csr_matrix:
    """scipy view of a SparseMatrix (model.py:76-79)."""
    got = getattr(m, "csr", None)
    if isinstance(got, sp.csr_matrix):
        return got
    try:
        return _CSR_CACHE[m]
    except (KeyError, TypeError):
        pass
    out = sp.csr_matrix((m.values, m.col_indices, m.row_offsets), shape=(m.n_rows, m.n_cols))
    try:
        _CSR_CACHE[m] = out
    except TypeError:
        pass
    return out


_BLOCK_CACHE: dict = {}


def b_blocks(op):
    """(C, A_l, A_u) as scipy CSR (kkt.py:203-208; row_submatrix model.py:92-95)."""
    key = (id(op.problem), id(op.bmap))
    hit = _BLOCK_CACHE.get(key)
    if hit is not None and hit[0] is op.problem:
        return hit[1]
    a = _csr(op.problem.a)
    blocks = (_csr(op.problem.c),
              a[np.asarray(op.bmap.lin_lower, dtype=np.int64), :],
              a[np.asarray(op.bmap.lin_upper, dtype=np.int64), :])
    if len(_BLOCK_CACHE) > 64:
        _BLOCK_CACHE.clear()
    _BLOCK_CACHE[key] = (op.problem, blocks)
    return blocks


def _families(op):
    m_e = op.problem.m_eq
    m_l = len(op.bmap.lin_lower)
    return m_e, m_l


def apply_b(op, u):
    c, a_l, a_u = b_blocks(op)
    return np.concatenate([c @ u, a_l @ u, -(a_u @ u)])


def apply_bt(op, w):
    c, a_l, a_u = b_blocks(op)
    m_e, m_l = _families(op)
    return c.T @ w[:m_e] + a_l.T @ w[m_e:m_e + m_l] - a_u.T @ w[m_e + m_l:]


def apply_doubly_augmented(op, v):
    """[[Q + 2B'D^-1 B, B'], [B, D]] (u, w)  -- kkt.py:211-221."""
    v = np.asarray(v, dtype=np.float64)
    n = op.problem.n
    u, w = v[:n], v[n:]
    t = apply_b(op, u)
    top = (hessian_apply(op.problem.hessian, u) + op.q_diag_extra * u) \
        + apply_bt(op, 2.0 * t / op.d_diag + w)
    bottom = t + op.d_diag * w
    return np.concatenate([top, bottom])


def jacobi_diagonal(op):
    """diag(Q) + 2 sum_i B_ij^2 / D_ii ; D   -- kkt.py:224-239."""
    m_e, m_l = _families(op)
    inv_d = 1.0 / op.d_diag
    top = hessian_diagonal(op.problem.hessian) + op.q_diag_extra
    for mat, dinv in zip(b_blocks(op), (inv_d[:m_e], inv_d[m_e:m_e + m_l], inv_d[m_e + m_l:])):
        if mat.shape[0]:
            top += 2.0 * (mat.multiply(mat).T @ dinv)
    return np.concatenate([top, op.d_diag])


# ----------------------------------------------------------------------------
# linalg.py:13-47
class PcgBreakdownError(RuntimeError):
    def __init__(self, result):
        super().__init__("PCG breakdown: operator is not positive definite")
        self.result = result


@dataclass(frozen=True)
class PcgConfig:
    tol: float = 1e-7
    max_iters: int = 5000
    tol_is_relative: bool = True


@dataclass(frozen=True)
class PcgResult:
    solution: np.ndarray
    iterations: int
    final_residual_norm: float
    converged: bool


def pcg(apply_op: Callable, apply_prec: Callable, rhs, cfg, x0=None,
        callback: Optional[Callable] = None):
    """linalg.py:66-133, same control flow and the same floating-point ops."""
    rhs = np.asarray(rhs, dtype=np.float64)
    scale = np.linalg.norm(rhs) if cfg.tol_is_relative else 1.0
    threshold = cfg.tol * scale
    if x0 is None:
        x = np.zeros_like(rhs)
        r = rhs.copy()
    else:
        x = np.array(x0, dtype=np.float64)
        r = rhs - apply_op(x)
    rnorm = np.linalg.norm(r)
    best = (x.copy(), rnorm)
    if rnorm <= threshold:
        return PcgResult(x, 0, rnorm, True)
    z = apply_prec(r)
    p = z.copy()
    rz = float(r @ z)
    k = 0
    while k < cfg.max_iters:
        k += 1
        y = apply_op(p)
        pap = float(p @ y)
        if pap <= 0:
            raise PcgBreakdownError(PcgResult(best[0], k - 1, best[1], False))
        alpha = rz / pap
        x += alpha * p
        r -= alpha * y
        rnorm = np.linalg.norm(r)
        if callback is not None:
            callback(k, x.copy(), rnorm)
        if rnorm < best[1]:
            best = (x.copy(), rnorm)
        if rnorm > threshold:
            z = apply_prec(r)
            rz_next = float(r @ z)
            beta = rz_next / rz
            rz = rz_next
            p = z + beta * p
            continue
        # recurrence says converged: confirm on the explicit residual
        true_r = rhs - apply_op(x)
        true_norm = np.linalg.norm(true_r)
        if true_norm <= threshold:
            return PcgResult(x, k, true_norm, True)
        r, rnorm = true_r, true_norm
        if rnorm < best[1]:
            best = (x.copy(), rnorm)
        z = apply_prec(r)
        p = z.copy()
        rz = float(r @ z)
    true_norm = np.linalg.norm(rhs - apply_op(best[0]))
    return PcgResult(best[0], cfg.max_iters, true_norm, true_norm <= threshold)


def pcg_direction(op, rhs, cfg, callback=None):
    """The reference direction solver ipm._pcg_direction (ipm.py:179-182)."""
    inv_diag = 1.0 / jacobi_diagonal(op)
    return pcg(lambda v: apply_doubly_augmented(op, v), lambda v: inv_diag * v,
               rhs, cfg, callback=callback)


# ----------------------------------------------------------------------------
# IPM loop (ipm.py:73-240; kkt.py:113-143, 242-284).  Used only to check the
# GPU direction solver at IPM level where the reference is not installed.
@dataclass(frozen=True)
class IpmConfig:
    gamma: float = 0.99
    mu_init: float = 1.0
    mu_tol: float = 1e-6
    mu_shrink: float = 10.0
    max_iters: int = 200
    pcg: PcgConfig = PcgConfig()


def _bmap(problem):
    from paper_2308_00637_b200.problem import BoundIndexMap
    return BoundIndexMap.from_problem(problem)


def initialize(problem, cfg, bmap):
    from paper_2308_00637_b200.problem import IterateState
    lo, hi = problem.var_bounds.lower, problem.var_bounds.upper
    x = np.zeros(problem.n)
    flo, fhi = np.isfinite(lo), np.isfinite(hi)
    x[flo & fhi] = 0.5 * (lo[flo & fhi] + hi[flo & fhi])
    x[flo & ~fhi] = lo[flo & ~fhi] + 1.0
    x[~flo & fhi] = hi[~flo & fhi] - 1.0
    ax = _csr(problem.a) @ x

    def slack(gap):
        return np.maximum(1.0, np.abs(gap))

    ll, lu = problem.lin_bounds.lower, problem.lin_bounds.upper
    return IterateState(
        x=x,
        s_lA=slack(ax[bmap.lin_lower] - ll[bmap.lin_lower]),
        s_uA=slack(lu[bmap.lin_upper] - ax[bmap.lin_upper]),
        s_lx=slack(x[bmap.var_lower] - lo[bmap.var_lower]),
        s_ux=slack(hi[bmap.var_upper] - x[bmap.var_upper]),
        lam_e=np.zeros(problem.m_eq),
        lam_lA=np.ones(len(bmap.lin_lower)), lam_uA=np.ones(len(bmap.lin_upper)),
        lam_lx=np.ones(len(bmap.var_lower)), lam_ux=np.ones(len(bmap.var_upper)),
        mu=cfg.mu_init)


_RES_KEYS = ("r_H", "r_e", "r_lA", "r_uA", "r_lx", "r_ux", "r_c1", "r_c2", "r_c3", "r_c4")


def compute_residuals(problem, state, bmap):
    x, mu = state.x, state.mu
    a = _csr(problem.a)
    a_l = a[np.asarray(bmap.lin_lower, dtype=np.int64), :]
    a_u = a[np.asarray(bmap.lin_upper, dtype=np.int64), :]
    c = _csr(problem.c)
    r_H = hessian_apply(problem.hessian, x) + problem.p \
        - a_l.T @ state.lam_lA + a_u.T @ state.lam_uA - c.T @ state.lam_e
    r_H[bmap.var_lower] -= state.lam_lx
    r_H[bmap.var_upper] += state.lam_ux
    res = dict(
        r_H=r_H,
        r_e=c @ x - problem.b + mu * state.lam_e,
        r_lA=a_l @ x - state.s_lA - problem.lin_bounds.lower[bmap.lin_lower],
        r_uA=problem.lin_bounds.upper[bmap.lin_upper] - a_u @ x - state.s_uA,
        r_lx=x[bmap.var_lower] - state.s_lx - problem.var_bounds.lower[bmap.var_lower],
        r_ux=problem.var_bounds.upper[bmap.var_upper] - x[bmap.var_upper] - state.s_ux,
        r_c1=state.lam_lA * state.s_lA - mu,
        r_c2=state.lam_uA * state.s_uA - mu,
        r_c3=state.lam_lx * state.s_lx - mu,
        r_c4=state.lam_ux * state.s_ux - mu,
    )
    if not np.all(np.isfinite(np.concatenate([res[k] for k in _RES_KEYS]))):
        raise FloatingPointError("non-finite residual encountered")
    return res


def assemble_rhs(op, res, state):
    bmap = op.bmap
    r1 = -res["r_H"].copy()
    r1[bmap.var_lower] += -res["r_c3"] / state.s_lx - (state.lam_lx / state.s_lx) * res["r_lx"]
    r1[bmap.var_upper] += res["r_c4"] / state.s_ux + (state.lam_ux / state.s_ux) * res["r_ux"]
    r2 = np.concatenate([-res["r_e"], -res["r_lA"] - res["r_c1"] / state.lam_lA,
                         -res["r_uA"] - res["r_c2"] / state.lam_uA])
    rhs = np.concatenate([r1 + apply_bt(op, 2.0 * r2 / op.d_diag), r2])
    if not np.all(np.isfinite(rhs)):
        raise FloatingPointError("non-finite right-hand side")
    return rhs


def recover_directions(op, dx, d_lam_a, res, state):
    m_e, m_l = _families(op)
    d_lam_e, d_lam_lA, d_lam_uA = d_lam_a[:m_e], d_lam_a[m_e:m_e + m_l], d_lam_a[m_e + m_l:]
    ds_lA = -(res["r_c1"] + state.s_lA * d_lam_lA) / state.lam_lA
    ds_uA = -(res["r_c2"] + state.s_uA * d_lam_uA) / state.lam_uA
    ds_lx = dx[op.bmap.var_lower] + res["r_lx"]
    ds_ux = res["r_ux"] - dx[op.bmap.var_upper]
    d_lam_lx = -(res["r_c3"] + state.lam_lx * ds_lx) / state.s_lx
    d_lam_ux = -(res["r_c4"] + state.lam_ux * ds_ux) / state.s_ux
    d = dict(dx=dx, d_lam_e=d_lam_e, d_lam_lA=d_lam_lA, d_lam_uA=d_lam_uA,
             d_lam_lx=d_lam_lx, d_lam_ux=d_lam_ux, ds_lA=ds_lA, ds_uA=ds_uA,
             ds_lx=ds_lx, ds_ux=ds_ux)
    for block in d.values():
        if not np.all(np.isfinite(block)):
            raise FloatingPointError("non-finite direction component")
    return d


def _ratio(values, deltas):
    neg = deltas < 0
    if not np.any(neg):
        return np.inf
    return float(np.min(-values[neg] / deltas[neg]))


def step_lengths(state, d, gamma):
    slack = min(_ratio(state.s_lA, d["ds_lA"]), _ratio(state.s_uA, d["ds_uA"]),
                _ratio(state.s_lx, d["ds_lx"]), _ratio(state.s_ux, d["ds_ux"]))
    lam = min(_ratio(state.lam_lA, d["d_lam_lA"]), _ratio(state.lam_uA, d["d_lam_uA"]),
              _ratio(state.lam_lx, d["d_lam_lx"]), _ratio(state.lam_ux, d["d_lam_ux"]))
    return min(1.0, gamma * slack), min(1.0, gamma * lam)


def apply_step(state, d, ax, al):
    from paper_2308_00637_b200.problem import IterateState
    new = IterateState(
        x=state.x + ax * d["dx"], s_lA=state.s_lA + ax * d["ds_lA"],
        s_uA=state.s_uA + ax * d["ds_uA"], s_lx=state.s_lx + ax * d["ds_lx"],
        s_ux=state.s_ux + ax * d["ds_ux"], lam_e=state.lam_e + al * d["d_lam_e"],
        lam_lA=state.lam_lA + al * d["d_lam_lA"], lam_uA=state.lam_uA + al * d["d_lam_uA"],
        lam_lx=state.lam_lx + al * d["d_lam_lx"], lam_ux=state.lam_ux + al * d["d_lam_ux"],
        mu=state.mu)
    parts = [new.s_lA, new.s_uA, new.s_lx, new.s_ux, new.lam_lA, new.lam_uA, new.lam_lx, new.lam_ux]
    mins = [v.min() for v in parts if len(v)]
    if (min(mins) if mins else np.inf) <= 0.0:
        raise RuntimeError("step left the strict interior")
    return new


def infeasibilities(res):
    primal = float(np.linalg.norm(np.concatenate([res["r_lA"], res["r_uA"], res["r_lx"], res["r_ux"]])))
    dual = float(np.linalg.norm(res["r_H"]))
    compl = float(np.linalg.norm(np.concatenate([res["r_c1"], res["r_c2"], res["r_c3"], res["r_c4"]])))
    return primal, dual, compl


def objective(problem, x):
    return 0.5 * float(x @ hessian_apply(problem.hessian, x)) + float(problem.p @ x)


@dataclass
class IpmReport:
    x: np.ndarray
    status: str
    objective: float
    iterations: int
    trace: list
    wall_time: float


def solve(problem, cfg: IpmConfig = IpmConfig(), direction_solver=None, breakdown_types=()):
    """ipm.py:185-240.  ``direction_solver(op, rhs, pcg_cfg)`` defaults to the oracle PCG."""
    from paper_2308_00637_b200.problem import build_operator
    if direction_solver is None:
        direction_solver = pcg_direction
    catch = (PcgBreakdownError,) + tuple(breakdown_types)
    t0 = time.perf_counter()
    bmap = _bmap(problem)
    state = initialize(problem, cfg, bmap)
    res = compute_residuals(problem, state, bmap)
    trace = []
    status = "iteration_limit"
    for it in range(1, cfg.max_iters + 1):
        op = build_operator(problem, state, bmap)
        rhs = assemble_rhs(op, res, state)
        try:
            cg = direction_solver(op, rhs, cfg.pcg)
        except catch as exc:
            cg = exc.result
        sol = np.asarray(cg.solution)
        if not np.all(np.isfinite(sol)):
            status = "linear_solver_failure"
            break
        d = recover_directions(op, sol[:problem.n], sol[problem.n:], res, state)
        ax, al = step_lengths(state, d, cfg.gamma)
        state = apply_step(state, d, ax, al)
        res = compute_residuals(problem, state, bmap)
        primal, dual, compl = infeasibilities(res)
        trace.append(dict(iter=it, mu=state.mu, primal_inf=primal, dual_inf=dual,
                          compl_inf=compl, cg_iters=cg.iterations,
                          cg_resid=cg.final_residual_norm, alpha_x=ax, alpha_lam=al))
        full = float(np.linalg.norm(np.concatenate([res[k] for k in _RES_KEYS])))
        if full < state.mu:
            if state.mu < cfg.mu_tol:
                status = "converged"
                break
            state.mu = state.mu / cfg.mu_shrink
            res = compute_residuals(problem, state, bmap)
    return IpmReport(x=state.x.copy(), status=status, objective=objective(problem, state.x),
                     iterations=len(trace), trace=trace, wall_time=time.perf_counter() - t0)
