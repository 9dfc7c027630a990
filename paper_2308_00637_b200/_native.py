"""ctypes binding of libqpk.so (include/qpk.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared library is missing or no CUDA device is
visible, every entry point raises ``NativeUnavailable`` -- the solver never
silently computes on the CPU.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("QPK_LIB", Path(__file__).resolve().parent / "libqpk.so"))

QPK_OK = 0
QPK_HESS_DIAG, QPK_HESS_CSR, QPK_HESS_DENSE, QPK_HESS_LOWRANK = 0, 1, 2, 3
QPK_PCG_OK, QPK_PCG_BREAKDOWN = 0, 1
QPK_SCATTER_AUTO, QPK_SCATTER_ATOMIC, QPK_SCATTER_CSC, QPK_SCATTER_DICT, QPK_SCATTER_PANEL = 0, 1, 2, 3, 4

EXPORTED = (
    "qpk_abi_version", "qpk_last_error", "qpk_create", "qpk_destroy", "qpk_set_stream",
    "qpk_synchronize", "qpk_problem_begin", "qpk_problem_add_rows", "qpk_set_hessian_diag",
    "qpk_set_hessian_csr", "qpk_set_hessian_dense", "qpk_set_hessian_lowrank",
    "qpk_problem_finalize", "qpk_set_diagonals", "qpk_set_diagonals_dev", "qpk_jacobi",
    "qpk_apply", "qpk_apply_dev", "qpk_pcg", "qpk_pcg_dev", "qpk_query",
    "qpk_nccl_get_unique_id", "qpk_shard_init", "qpk_shard_emulate", "qpk_ipm_set_bounds", "qpk_ipm_solve",
    "qpk_set_hessian_dense_dev", "qpk_rbf_hessian_dev", "qpk_hessian_apply_dev", "qpk_dense_gemv_dev",
    "qpk_multi_create", "qpk_multi_create_emulated", "qpk_multi_destroy", "qpk_multi_devices", "qpk_multi_context", "qpk_multi_problem_begin",
    "qpk_multi_problem_add_rows", "qpk_multi_set_hessian_diag", "qpk_multi_set_hessian_csr",
    "qpk_multi_set_hessian_dense", "qpk_multi_set_hessian_lowrank", "qpk_multi_problem_finalize",
    "qpk_multi_set_diagonals", "qpk_multi_jacobi", "qpk_multi_apply", "qpk_multi_pcg", "qpk_multi_query",
)


class NativeUnavailable(RuntimeError):
    """libqpk.so is missing or cannot run (no CUDA device)."""


class NativeError(RuntimeError):
    def __init__(self, fn, code, msg):
        super().__init__(f"{fn} failed with {code}: {msg}")
        self.code = code


class PcgInfo(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
        ("status", ctypes.c_int32), ("restarts", ctypes.c_int32),
        ("applies", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("final_residual_norm", ctypes.c_double), ("threshold", ctypes.c_double),
        ("rhs_norm", ctypes.c_double), ("kernel_ms", ctypes.c_double),
        ("phase_ms", ctypes.c_double * 4),
    ]


class IpmConfig(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("mu_init", ctypes.c_double), ("mu_tol", ctypes.c_double),
                ("mu_shrink", ctypes.c_double), ("max_iters", ctypes.c_int64), ("pcg_tol", ctypes.c_double),
                ("pcg_max_iters", ctypes.c_int64), ("pcg_tol_is_relative", ctypes.c_int32),
                ("verbose", ctypes.c_int32)]


class IpmTrace(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("cg_iters", ctypes.c_int32), ("mu", ctypes.c_double),
                ("primal_inf", ctypes.c_double), ("dual_inf", ctypes.c_double), ("compl_inf", ctypes.c_double),
                ("cg_resid", ctypes.c_double), ("alpha_x", ctypes.c_double), ("alpha_lam", ctypes.c_double)]


class IpmResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32), ("cg_total", ctypes.c_int64),
                ("objective", ctypes.c_double), ("wall_ms", ctypes.c_double)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_I = ctypes.c_int
_SIGS = {
    "qpk_abi_version": ([], _I),
    "qpk_last_error": ([], ctypes.c_char_p),
    "qpk_create": ([_I, ctypes.POINTER(_P)], _I),
    "qpk_destroy": ([_P], _I),
    "qpk_set_stream": ([_P, _P], _I),
    "qpk_synchronize": ([_P], _I),
    "qpk_problem_begin": ([_P, _I64, _I64, _I64, _I64], _I),
    "qpk_problem_add_rows": ([_P, _I64, _P, _P, _P, _P, _I64, _D], _I),
    "qpk_set_hessian_diag": ([_P, _P], _I),
    "qpk_set_hessian_csr": ([_P, _P, _P, _P], _I),
    "qpk_set_hessian_dense": ([_P, _P], _I),
    "qpk_set_hessian_lowrank": ([_P, _P, _I64, _P, _P], _I),
    "qpk_set_hessian_dense_dev": ([_P, _P], _I),
    "qpk_rbf_hessian_dev": ([_P, _P, _I64, _I64, _P, _D, _P], _I),
    "qpk_hessian_apply_dev": ([_P, _P, _P], _I),
    "qpk_dense_gemv_dev": ([_P, _P, _I64, _P, _P], _I),
    "qpk_problem_finalize": ([_P, _I], _I),
    "qpk_set_diagonals": ([_P, _P, _P], _I),
    "qpk_set_diagonals_dev": ([_P, _P, _P], _I),
    "qpk_jacobi": ([_P, _P], _I),
    "qpk_apply": ([_P, _P, _P], _I),
    "qpk_apply_dev": ([_P, _P, _P], _I),
    "qpk_pcg": ([_P, _P, _D, _I, _I64, _P, ctypes.POINTER(PcgInfo), _P], _I),
    "qpk_pcg_dev": ([_P, _P, _D, _I, _I64, _P, ctypes.POINTER(PcgInfo), _P], _I),
    "qpk_query": ([_P, ctypes.c_char_p], _I64),
    "qpk_nccl_get_unique_id": ([_P], _I),
    "qpk_shard_init": ([_P, _I, _I, _P], _I),
    "qpk_shard_emulate": ([_P, _I, _I], _I),
    "qpk_ipm_set_bounds": ([_P, _P, _P, _I64, _P, _P, _I64, _P, _P], _I),
    "qpk_ipm_solve": ([_P, ctypes.POINTER(IpmConfig), _P, _P, ctypes.POINTER(IpmResult)], _I),
    "qpk_multi_create": ([_I, ctypes.POINTER(_I), ctypes.POINTER(_P)], _I),
    "qpk_multi_destroy": ([_P], _I),
    "qpk_multi_create_emulated": ([_I, _I, ctypes.POINTER(_P)], _I),
    "qpk_multi_devices": ([_P], _I),
    "qpk_multi_context": ([_P, _I], _P),
    "qpk_multi_problem_begin": ([_P, _I64, _I64, _I64, _I64], _I),
    "qpk_multi_problem_add_rows": ([_P, _I64, _P, _P, _P, _P, _I64, _D], _I),
    "qpk_multi_set_hessian_diag": ([_P, _P], _I),
    "qpk_multi_set_hessian_csr": ([_P, _P, _P, _P], _I),
    "qpk_multi_set_hessian_dense": ([_P, _P], _I),
    "qpk_multi_set_hessian_lowrank": ([_P, _P, _I64, _P, _P], _I),
    "qpk_multi_problem_finalize": ([_P, _I], _I),
    "qpk_multi_set_diagonals": ([_P, _P, _P], _I),
    "qpk_multi_jacobi": ([_P, _P], _I),
    "qpk_multi_apply": ([_P, _P, _P], _I),
    "qpk_multi_pcg": ([_P, _P, _D, _I, _I64, _P, ctypes.POINTER(PcgInfo), _P], _I),
    "qpk_multi_query": ([_P, _I, ctypes.c_char_p], _I64),
}

_lib = None


def load_library(path: Path = LIB_PATH) -> ctypes.CDLL:
    """Load libqpk.so and declare every exported signature (no CUDA calls)."""
    global _lib
    if _lib is not None:
        return _lib
    if not path.exists():
        raise NativeUnavailable(f"{path} not built; run __graft_entry__.build()")
    lib = ctypes.CDLL(str(path))
    for name, (args, ret) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ret
    _lib = lib
    return lib


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a is not None and a.size else 0


def check(fn_name: str, rc: int):
    if rc != QPK_OK:
        msg = _lib.qpk_last_error().decode(errors="replace")
        raise NativeError(fn_name, rc, msg)


class Context:
    """One libqpk context (one device).  Owns the device copy of one problem."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = ctypes.c_void_p()
        rc = lib.qpk_create(int(device), ctypes.byref(h))
        if rc != QPK_OK:
            raise NativeUnavailable(lib.qpk_last_error().decode(errors="replace"))
        self._lib = lib
        self._h = h
        self.device = device

    def close(self):
        if self._h:
            self._lib.qpk_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def call(self, name, *args):
        check(name, getattr(self._lib, name)(self._h, *args))

    def query(self, key: str) -> int:
        return int(self._lib.qpk_query(self._h, key.encode()))


class MultiContext:
    """One libqpk multi-device object (qpk_multi): several GPUs, one process."""

    def __init__(self, devices, emulate_ranks: int = 0):
        lib = load_library()
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        h = ctypes.c_void_p()
        if emulate_ranks:       # test hook: N ranks on devices[0], host-mediated collectives
            rc = lib.qpk_multi_create_emulated(int(emulate_ranks), int(devices[0]), ctypes.byref(h))
        else:
            rc = lib.qpk_multi_create(len(devices), devs, ctypes.byref(h))
        if rc != QPK_OK:
            raise NativeUnavailable(lib.qpk_last_error().decode(errors="replace"))
        self._lib = lib
        self._h = h
        self.devices = list(devices)

    def close(self):
        if self._h:
            self._lib.qpk_multi_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def call(self, name, *args):
        check(name, getattr(self._lib, name)(self._h, *args))

    def query(self, key: str, rank: int = 0) -> int:
        return int(self._lib.qpk_multi_query(self._h, int(rank), key.encode()))
