"""Interior-point solve with the whole IPM iteration on the device.

``solve(problem, cfg)`` mirrors ``qpipm.ipm.solve`` (ipm.py:185-240): same
configuration fields (``IpmConfig``: gamma, mu_init, mu_tol, mu_shrink,
max_iters, pcg), same report (x, status, trace of TraceRecord-like rows,
objective, iterations, wall_time) -- but the iterate, the residuals
(kkt.py:113-143), the right-hand side (kkt.py:242-257), the direction
recovery (kkt.py:260-284), the ratio test and the step (ipm.py:107-153) live
on the GPU (`qpk_ipm_solve`), around the same Jacobi-PCG direction solver.
Only the per-iteration scalars reach the host.
The reference IPM driven by ``gpu_direction`` remains the drop-in path; this
is the all-device path used for the "IPM wall time" measurement.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .direction import GpuKkt
from .pcg import PcgConfig
from .problem import BoundIndexMap


class SolveStatus(enum.Enum):
    CONVERGED = "converged"
    ITERATION_LIMIT = "iteration_limit"
    LINEAR_SOLVER_FAILURE = "linear_solver_failure"


@dataclass(frozen=True)
class IpmConfig:
    gamma: float = 0.99
    mu_init: float = 1.0
    mu_tol: float = 1e-6
    mu_shrink: float = 10.0
    max_iters: int = 200
    pcg: PcgConfig = field(default_factory=PcgConfig)


@dataclass(frozen=True)
class TraceRecord:
    iter: int
    mu: float
    primal_inf: float
    dual_inf: float
    compl_inf: float
    cg_iters: int
    cg_resid: float
    alpha_x: float
    alpha_lam: float


@dataclass(frozen=True)
class SolveReport:
    x: np.ndarray
    status: SolveStatus
    trace: list
    objective: float
    iterations: int
    wall_time: float
    cg_total: int


_STATUS = {0: SolveStatus.CONVERGED, 1: SolveStatus.ITERATION_LIMIT, 2: SolveStatus.LINEAR_SOLVER_FAILURE}


class DeviceIpm:
    """A problem resident on the device, ready for repeated IPM solves."""

    def __init__(self, problem, device: int = 0, scatter: int = _native.QPK_SCATTER_AUTO):
        self.problem = problem
        self.bmap = BoundIndexMap.from_problem(problem)
        self.kkt = GpuKkt(problem, self.bmap, device=device, scatter=scatter)
        lb, ub = problem.lin_bounds.lower, problem.lin_bounds.upper
        bnd = np.ascontiguousarray(np.concatenate([
            np.asarray(problem.b, dtype=np.float64),
            lb[self.bmap.lin_lower], ub[self.bmap.lin_upper]]), dtype=np.float64)
        vlo = np.ascontiguousarray(self.bmap.var_lower, dtype=np.int64)
        vhi = np.ascontiguousarray(self.bmap.var_upper, dtype=np.int64)
        lx = np.ascontiguousarray(problem.var_bounds.lower[vlo], dtype=np.float64)
        ux = np.ascontiguousarray(problem.var_bounds.upper[vhi], dtype=np.float64)
        p = np.ascontiguousarray(problem.p, dtype=np.float64)
        self._keep = (bnd, vlo, vhi, lx, ux, p)
        self.kkt.ctx.call("qpk_ipm_set_bounds", _native.ptr(p), _native.ptr(bnd), len(vlo), _native.ptr(vlo),
                          _native.ptr(lx), len(vhi), _native.ptr(vhi), _native.ptr(ux))

    def solve(self, cfg=None, verbose: bool = False) -> SolveReport:
        if cfg is None:
            cfg = IpmConfig()
        c = _native.IpmConfig(gamma=cfg.gamma, mu_init=cfg.mu_init, mu_tol=cfg.mu_tol, mu_shrink=cfg.mu_shrink,
                              max_iters=int(cfg.max_iters), pcg_tol=cfg.pcg.tol,
                              pcg_max_iters=int(cfg.pcg.max_iters),
                              pcg_tol_is_relative=int(bool(cfg.pcg.tol_is_relative)), verbose=int(verbose))
        x = np.empty(self.problem.n)
        trace = (_native.IpmTrace * max(1, int(cfg.max_iters)))()
        res = _native.IpmResult()
        self.kkt.ctx.call("qpk_ipm_solve", ctypes.byref(c), _native.ptr(x), ctypes.addressof(trace),
                          ctypes.byref(res))
        rows = [TraceRecord(t.iter, t.mu, t.primal_inf, t.dual_inf, t.compl_inf, t.cg_iters, t.cg_resid,
                            t.alpha_x, t.alpha_lam) for t in trace[:res.iterations]]
        return SolveReport(x=x, status=_STATUS[res.status], trace=rows, objective=res.objective,
                           iterations=res.iterations, wall_time=res.wall_ms * 1e-3, cg_total=int(res.cg_total))

    def close(self):
        self.kkt.close()


def solve(problem, cfg=None, verbose: bool = False, device: int = 0) -> SolveReport:
    """qpipm.ipm.solve with the IPM iteration on the GPU."""
    dev = DeviceIpm(problem, device=device)
    try:
        return dev.solve(cfg, verbose=verbose)
    finally:
        dev.close()
