"""IPM-level parity of the drop-in: the IPM loop (the reference's, restated in
the oracle because qpipm is not installed on the GPU box) driven by the GPU
direction solver, against the reference's own IPM results (tests/golden/ipm.npz).

Gates: same status; objective and x within 1e-6 relative;
final primal/dual infeasibility within 10x the reference's or below mu_tol.
"""

import numpy as np
import pytest

import golden_io
from oracle import qp_oracle as orc
from paper_2308_00637_b200 import workloads
from paper_2308_00637_b200.direction import gpu_direction
from paper_2308_00637_b200.pcg import PcgBreakdownError, result_types

pytestmark = pytest.mark.gpu

IPM = golden_io.load("ipm")


def cfg_from(arr):
    return orc.IpmConfig(gamma=arr[0], mu_init=arr[1], mu_tol=arr[2], mu_shrink=arr[3], max_iters=int(arr[4]),
                         pcg=orc.PcgConfig(tol=arr[5], max_iters=int(arr[6]), tol_is_relative=bool(arr[7])))


@pytest.mark.parametrize("name", [str(s) for s in IPM["names"]])
def test_ipm_with_gpu_direction(name):
    pre = name + "_"
    if name == "cfg1":
        problem, _, _ = workloads.dense_qp(seed=0)
    else:
        problem = golden_io.problem_from(IPM, pre)
    cfg = cfg_from(IPM[pre + "cfg"])
    rep = orc.solve(problem, cfg, direction_solver=gpu_direction, breakdown_types=(PcgBreakdownError, result_types()[1]))
    assert rep.status == str(IPM[pre + "status"])
    obj = float(IPM[pre + "objective"])
    assert abs(rep.objective - obj) <= 1e-6 * max(abs(obj), 1.0)
    x_ref = IPM[pre + "x"]
    assert np.linalg.norm(rep.x - x_ref) <= 1e-6 * max(np.linalg.norm(x_ref), 1.0)
    primal, dual = rep.trace[-1]["primal_inf"], rep.trace[-1]["dual_inf"]
    assert primal <= max(10 * float(IPM[pre + "primal"][-1]), cfg.mu_tol)
    assert dual <= max(10 * float(IPM[pre + "dual"][-1]), cfg.mu_tol)
    # iteration counts are reported, not gated (CG chaos)
    print(f"{name}: IPM {rep.iterations} (ref {int(IPM[pre + 'iterations'])}), "
          f"CG {sum(t['cg_iters'] for t in rep.trace)} (ref {int(IPM[pre + 'cg_iters'].sum())}), "
          f"{rep.wall_time:.2f}s")
