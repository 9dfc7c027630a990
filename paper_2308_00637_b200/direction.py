"""Drop-in GPU direction solver for the reference IPM.

``gpu_direction(op, rhs, cfg)`` has the signature of the reference hook
``DirectionSolver = Callable[[KktOperator, np.ndarray, PcgConfig], PcgResult]``
(qpipm/ipm.py:176) and the semantics of ``_pcg_direction`` (ipm.py:179-182):
build the Jacobi diagonal, then run PCG from x0 = 0 on the doubly augmented
operator.  It is passed as ``solve(problem, cfg, direction_solver=gpu_direction)``
(ipm.py:185-187, called at ipm.py:206).

* ``op`` is read by attribute: ``op.problem`` (n, a, c, hessian, m_eq),
  ``op.bmap.lin_lower / lin_upper``, ``op.d_diag``, ``op.q_diag_extra``.  Both
  the reference's KktOperator and ``problem.KktOperator`` work.
* The problem data (B = (C; A_l; -A_u) and H) is uploaded once per problem
  object and cached; only the two diagonals cross per IPM iteration.
* Returns a ``PcgResult`` and raises ``PcgBreakdownError(result)`` on
  nonpositive curvature -- the caller's own types when ``qpipm`` is loaded
  (so the reference's ``except PcgBreakdownError`` at ipm.py:207 catches it),
  otherwise this package's mirrors in ``pcg.py``.
* There is no CPU fallback: without the CUDA library this raises.
"""

from __future__ import annotations

import os
import sys
import weakref

import numpy as np

from . import _native
from .pcg import result_types


class GpuKkt:
    """Device-resident doubly augmented operator of one QpProblem."""

    def __init__(self, problem, bmap, device: int = 0, scatter: int = _native.QPK_SCATTER_AUTO):
        import time
        t0 = time.perf_counter()
        timing = bool(os.environ.get("QPK_TIMING"))

        def lap(what):
            nonlocal t0
            if timing:
                t1 = time.perf_counter()
                print(f"[qpk setup] py {what:<12s} {(t1 - t0) * 1e3:8.1f} ms", file=sys.stderr, flush=True)
                t0 = t1
        self.ctx = _native.Context(device)
        lap("context")
        self._upload(problem, bmap, scatter, lap)

    def reload(self, problem, bmap, scatter: int = _native.QPK_SCATTER_AUTO):
        """Replace the problem held by this context (qpk_problem_begin again on
        the same qpk_ctx: buffers, stream and graph state are reused)."""
        self._upload(problem, bmap, scatter, lambda what: None)

    def _upload(self, problem, bmap, scatter, lap):
        self.n = int(problem.n)
        lin_lower = np.ascontiguousarray(bmap.lin_lower, dtype=np.int64)
        lin_upper = np.ascontiguousarray(bmap.lin_upper, dtype=np.int64)
        m_e = int(problem.c.n_rows)
        self.m = m_e + len(lin_lower) + len(lin_upper)
        self.dim = self.n + self.m
        c = self.ctx
        c.call("qpk_problem_begin", self.n, m_e, len(lin_lower), len(lin_upper))
        # B = (C; A_l; -A_u) in the reference's row order (kkt.py:177, 206-207)
        cm = problem.c
        if m_e:
            ro, ci, v = _csr_arrays(cm)
            c.call("qpk_problem_add_rows", int(cm.n_rows), _native.ptr(ro), _native.ptr(ci),
                   _native.ptr(v), None, 0, 1.0)
        am = problem.a
        if len(lin_lower) or len(lin_upper):
            ro, ci, v = _csr_arrays(am)
            for rows, sign in ((lin_lower, 1.0), (lin_upper, -1.0)):
                if len(rows):
                    c.call("qpk_problem_add_rows", int(am.n_rows), _native.ptr(ro), _native.ptr(ci),
                           _native.ptr(v), _native.ptr(rows), len(rows), sign)
        lap("add_rows")
        self._set_hessian(problem.hessian)
        lap("hessian")
        # AUTO lets the library pick per matrix (QPK_SCATTER in the environment overrides)
        c.call("qpk_problem_finalize", int(scatter))
        lap("finalize")
        self._hist = None

    def _set_hessian(self, h):
        kind = type(h).__name__
        c = self.ctx
        if kind == "DiagonalHessian":
            d = np.ascontiguousarray(h.d, dtype=np.float64)
            _dim(len(d), self.n, "Hessian")
            c.call("qpk_set_hessian_diag", _native.ptr(d))
        elif kind == "SparseHessian":
            ro, ci, v = _csr_arrays(h.m)
            _dim(h.m.n_rows, self.n, "Hessian")
            c.call("qpk_set_hessian_csr", _native.ptr(ro), _native.ptr(ci), _native.ptr(v))
        elif kind == "DenseHessian":
            mm = np.ascontiguousarray(h.m, dtype=np.float64)
            if mm.ndim != 2 or mm.shape != (self.n, self.n):
                from .problem import DimensionError
                raise DimensionError(f"dense Hessian has shape {mm.shape}, expected {(self.n, self.n)}")
            c.call("qpk_set_hessian_dense", _native.ptr(mm))
        elif kind == "DeviceDenseHessian":             # SVM dual: built on the device (svm.py)
            _dim(h.n, self.n, "Hessian")
            c.call("qpk_set_hessian_dense_dev", int(h.m_dev.data_ptr()))
        elif kind == "QuasiNewtonHessian":
            h0 = np.ascontiguousarray(h.h0_diag, dtype=np.float64)
            u = np.ascontiguousarray(h.u, dtype=np.float64)
            w = np.ascontiguousarray(h.w, dtype=np.float64)
            _dim(len(h0), self.n, "Hessian")
            c.call("qpk_set_hessian_lowrank", _native.ptr(h0), int(u.shape[1]), _native.ptr(u), _native.ptr(w))
        else:
            raise TypeError(f"unsupported Hessian type {kind}")

    # -- per IPM iteration -------------------------------------------------
    def set_diagonals(self, d_diag, q_extra):
        d = np.ascontiguousarray(d_diag, dtype=np.float64)
        q = np.ascontiguousarray(q_extra, dtype=np.float64)
        _dim(len(d), self.m, "d_diag")
        _dim(len(q), self.n, "q_diag_extra")
        self.ctx.call("qpk_set_diagonals", _native.ptr(d), _native.ptr(q))

    def jacobi(self) -> np.ndarray:
        out = np.empty(self.dim)
        self.ctx.call("qpk_jacobi", _native.ptr(out))
        return out

    def apply(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        _dim(len(v), self.dim, "vector")
        y = np.empty(self.dim)
        self.ctx.call("qpk_apply", _native.ptr(v), _native.ptr(y))
        return y

    def pcg(self, rhs, tol: float, max_iters: int, tol_is_relative: bool = True, history: bool = False):
        """Returns (x, info, hist-or-None)."""
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        _dim(len(rhs), self.dim, "rhs")
        x = np.empty(self.dim)
        info = _native.PcgInfo()
        hist = np.full(int(max_iters) + 1, np.nan) if history else None
        self.ctx.call("qpk_pcg", _native.ptr(rhs), float(tol), int(bool(tol_is_relative)), int(max_iters),
                      _native.ptr(x), _native.ctypes.byref(info), _native.ptr(hist) if history else None)
        if history:
            hist = hist[: info.iterations + 1]
        return x, info, hist

    def close(self):
        self.ctx.close()


class MultiGpuKkt(GpuKkt):
    """The same operator row-sharded over several GPUs, driven from THIS process
    (qpk_multi, include/qpk.h): the reference's single-process solve()
    (ipm.py:185-206) can use N GPUs through the unmodified hook.  Same methods
    and global-sized vectors as GpuKkt."""

    def __init__(self, problem, bmap, devices, scatter: int = _native.QPK_SCATTER_AUTO, emulate_ranks: int = 0):
        self.ctx = _native.MultiContext(devices, emulate_ranks=emulate_ranks)
        self.devices = list(devices)
        self.n = int(problem.n)
        lin_lower = np.ascontiguousarray(bmap.lin_lower, dtype=np.int64)
        lin_upper = np.ascontiguousarray(bmap.lin_upper, dtype=np.int64)
        m_e = int(problem.c.n_rows)
        self.m = m_e + len(lin_lower) + len(lin_upper)
        self.dim = self.n + self.m
        c = self.ctx
        keep = []                                    # the library reads these arrays at finalize
        c.call("qpk_multi_problem_begin", self.n, m_e, len(lin_lower), len(lin_upper))
        if m_e:
            ro, ci, v = _csr_arrays(problem.c)
            keep += [ro, ci, v]
            c.call("qpk_multi_problem_add_rows", int(problem.c.n_rows), _native.ptr(ro), _native.ptr(ci),
                   _native.ptr(v), None, 0, 1.0)
        if len(lin_lower) or len(lin_upper):
            ro, ci, v = _csr_arrays(problem.a)
            keep += [ro, ci, v]
            for rows, sign in ((lin_lower, 1.0), (lin_upper, -1.0)):
                if len(rows):
                    c.call("qpk_multi_problem_add_rows", int(problem.a.n_rows), _native.ptr(ro), _native.ptr(ci),
                           _native.ptr(v), _native.ptr(rows), len(rows), sign)
        keep += self._set_hessian_multi(problem.hessian)
        c.call("qpk_multi_problem_finalize", int(scatter))
        del keep
        self._hist = None

    def _set_hessian_multi(self, h):
        kind = type(h).__name__
        c = self.ctx
        if kind == "DiagonalHessian":
            d = np.ascontiguousarray(h.d, dtype=np.float64)
            _dim(len(d), self.n, "Hessian")
            c.call("qpk_multi_set_hessian_diag", _native.ptr(d))
            return [d]
        if kind == "SparseHessian":
            ro, ci, v = _csr_arrays(h.m)
            _dim(h.m.n_rows, self.n, "Hessian")
            c.call("qpk_multi_set_hessian_csr", _native.ptr(ro), _native.ptr(ci), _native.ptr(v))
            return [ro, ci, v]
        if kind == "DenseHessian":
            mm = np.ascontiguousarray(h.m, dtype=np.float64)
            if mm.ndim != 2 or mm.shape != (self.n, self.n):
                from .problem import DimensionError
                raise DimensionError(f"dense Hessian has shape {mm.shape}, expected {(self.n, self.n)}")
            c.call("qpk_multi_set_hessian_dense", _native.ptr(mm))
            return [mm]
        if kind == "QuasiNewtonHessian":
            h0 = np.ascontiguousarray(h.h0_diag, dtype=np.float64)
            u = np.ascontiguousarray(h.u, dtype=np.float64)
            w = np.ascontiguousarray(h.w, dtype=np.float64)
            _dim(len(h0), self.n, "Hessian")
            c.call("qpk_multi_set_hessian_lowrank", _native.ptr(h0), int(u.shape[1]), _native.ptr(u), _native.ptr(w))
            return [h0, u, w]
        raise TypeError(f"unsupported Hessian type {kind}")

    def set_diagonals(self, d_diag, q_extra):
        d = np.ascontiguousarray(d_diag, dtype=np.float64)
        q = np.ascontiguousarray(q_extra, dtype=np.float64)
        _dim(len(d), self.m, "d_diag")
        _dim(len(q), self.n, "q_diag_extra")
        self.ctx.call("qpk_multi_set_diagonals", _native.ptr(d), _native.ptr(q))

    def jacobi(self) -> np.ndarray:
        out = np.empty(self.dim)
        self.ctx.call("qpk_multi_jacobi", _native.ptr(out))
        return out

    def apply(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        _dim(len(v), self.dim, "vector")
        y = np.empty(self.dim)
        self.ctx.call("qpk_multi_apply", _native.ptr(v), _native.ptr(y))
        return y

    def pcg(self, rhs, tol: float, max_iters: int, tol_is_relative: bool = True, history: bool = False):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        _dim(len(rhs), self.dim, "rhs")
        x = np.empty(self.dim)
        info = _native.PcgInfo()
        hist = np.full(int(max_iters) + 1, np.nan) if history else None
        self.ctx.call("qpk_multi_pcg", _native.ptr(rhs), float(tol), int(bool(tol_is_relative)), int(max_iters),
                      _native.ptr(x), _native.ctypes.byref(info), _native.ptr(hist) if history else None)
        if history:
            hist = hist[: info.iterations + 1]
        return x, info, hist


def _dim(got, want, what):
    if got != want:
        from .problem import DimensionError
        raise DimensionError(f"{what} has length {got}, expected {want}")


def _csr_arrays(m):
    return (np.ascontiguousarray(m.row_offsets, dtype=np.int64),
            np.ascontiguousarray(m.col_indices, dtype=np.int64),
            np.ascontiguousarray(m.values, dtype=np.float64))


# one device copy per live problem object (the reference passes the same
# QpProblem to every IPM iteration; kkt.py:372-377)
_CACHE: "dict[int, tuple]" = {}


def _finalizer(key):
    entry = _CACHE.pop(key, None)
    if entry is not None:
        entry[1].close()


_DEVICES = None


def set_devices(devices):
    """GPUs the drop-in hook uses: None / one id = a single GPU (GpuKkt); a list
    of several ids = one process driving them all (MultiGpuKkt).  The hook's
    signature is the reference's, so the choice is made here (or through the
    environment: QPK_DEVICES=0,1,2,3)."""
    global _DEVICES
    _DEVICES = None if devices is None else [int(d) for d in np.atleast_1d(devices)]
    for key in list(_CACHE):
        _finalizer(key)


def _devices(default: int):
    if _DEVICES is not None:
        return _DEVICES
    env = os.environ.get("QPK_DEVICES")
    if env:
        return [int(t) for t in env.split(",") if t.strip() != ""]
    return [default]


def operator_for(op, device: int = 0) -> GpuKkt:
    problem = op.problem
    key = id(problem)
    entry = _CACHE.get(key)
    if entry is not None and entry[0]() is problem:
        # the reference hands the same bound-index arrays to every IPM
        # iteration: identical objects skip hashing them (1.6M indices on cfg4)
        same = entry[3][0] is op.bmap.lin_lower and entry[3][1] is op.bmap.lin_upper
        if same or entry[2] == _bmap_key(op.bmap):
            return entry[1]
    if entry is not None:
        _finalizer(key)
    devs = _devices(device)
    # (QPK_MULTI=1 sends even a single device through the multi-device layer: its one-GPU test)
    single = len(devs) == 1 and not os.environ.get("QPK_MULTI")
    gk = GpuKkt(problem, op.bmap, device=devs[0]) if single else MultiGpuKkt(problem, op.bmap, devs)
    try:
        ref = weakref.ref(problem, lambda _r, k=key: _finalizer(k))
    except TypeError:
        ref = lambda p=problem: p  # noqa: E731  (unweakrefable problem: keep it alive)
    _CACHE[key] = (ref, gk, _bmap_key(op.bmap), (op.bmap.lin_lower, op.bmap.lin_upper))
    return gk


def _bmap_key(bmap):
    return (len(bmap.lin_lower), len(bmap.lin_upper),
            hash(np.asarray(bmap.lin_lower).tobytes()), hash(np.asarray(bmap.lin_upper).tobytes()))


def gpu_direction(op, rhs, cfg):
    """DirectionSolver: Jacobi-PCG on the GPU (ipm.py:179-182 semantics)."""
    PcgResult, PcgBreakdownError = result_types()
    gk = operator_for(op)
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    x, info, _ = gk.pcg(rhs, cfg.tol, cfg.max_iters, cfg.tol_is_relative)
    result = PcgResult(x, int(info.iterations), float(info.final_residual_norm), bool(info.converged))
    if info.status == _native.QPK_PCG_BREAKDOWN:
        raise PcgBreakdownError(result)
    return result
