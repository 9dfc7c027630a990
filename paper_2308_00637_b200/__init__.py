"""B200-native Jacobi-PCG direction solver for the doubly augmented KKT system.

Drop-in for the linear-solver hook of the reference interior-point QP solver
(qpipm, arXiv 2308.00637): ``solve(problem, cfg, direction_solver=gpu_direction)``.
"""

from .direction import GpuKkt, MultiGpuKkt, gpu_direction, operator_for, set_devices
from .pcg import PcgBreakdownError, PcgConfig, PcgResult

__all__ = ["GpuKkt", "MultiGpuKkt", "gpu_direction", "operator_for", "set_devices", "PcgBreakdownError", "PcgConfig", "PcgResult"]
__version__ = "0.1.0"
