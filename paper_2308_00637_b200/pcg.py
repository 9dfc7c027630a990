"""PCG configuration and result types of the linear-solver interface.

Mirrors of ``PcgConfig``, ``PcgResult`` and ``PcgBreakdownError``
(qpipm/linalg.py:13-47).  When the reference package is importable its own
classes are used instead (``result_types``), so that a breakdown raised by the
GPU solver is caught by the reference IPM's ``except PcgBreakdownError``
(ipm.py:207-208).
"""

from __future__ import annotations

import sys
from dataclasses import dataclass

import numpy as np


class PcgBreakdownError(RuntimeError):
    """Nonpositive curvature p'(Op p) <= 0; carries the best iterate."""

    def __init__(self, result: "PcgResult"):
        super().__init__("PCG breakdown: operator is not positive definite")
        self.result = result


@dataclass(frozen=True)
class PcgConfig:
    tol: float = 1e-7
    max_iters: int = 5000
    tol_is_relative: bool = True

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")


@dataclass(frozen=True)
class PcgResult:
    solution: np.ndarray
    iterations: int
    final_residual_norm: float
    converged: bool


def result_types():
    """(PcgResult, PcgBreakdownError) of the caller: qpipm's if loaded, else ours."""
    mod = sys.modules.get("qpipm.linalg")
    if mod is not None:
        return mod.PcgResult, mod.PcgBreakdownError
    return PcgResult, PcgBreakdownError
