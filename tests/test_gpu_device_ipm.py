"""The all-device IPM (qpk_ipm_solve) against the reference's own solve()
results (tests/golden/ipm.npz): same status, objective and x within 1e-6
relative, final primal/dual infeasibility within 10x the reference's or below
mu_tol; iteration counts reported, not gated."""

import numpy as np
import pytest

import golden_io
from paper_2308_00637_b200 import workloads
from paper_2308_00637_b200.ipm import IpmConfig, solve
from paper_2308_00637_b200.pcg import PcgConfig

pytestmark = pytest.mark.gpu

IPM = golden_io.load("ipm")


def cfg_from(a):
    return IpmConfig(gamma=a[0], mu_init=a[1], mu_tol=a[2], mu_shrink=a[3], max_iters=int(a[4]),
                     pcg=PcgConfig(tol=a[5], max_iters=int(a[6]), tol_is_relative=bool(a[7])))


@pytest.mark.parametrize("name", [str(s) for s in IPM["names"]])
def test_device_ipm_matches_reference(name):
    pre = name + "_"
    if name == "cfg1":
        problem, _, _ = workloads.dense_qp(seed=0)
    else:
        problem = golden_io.problem_from(IPM, pre)
    cfg = cfg_from(IPM[pre + "cfg"])
    rep = solve(problem, cfg)
    assert rep.status.value == str(IPM[pre + "status"])
    obj = float(IPM[pre + "objective"])
    assert abs(rep.objective - obj) <= 1e-6 * max(abs(obj), 1.0)
    x_ref = IPM[pre + "x"]
    assert np.linalg.norm(rep.x - x_ref) <= 1e-6 * max(np.linalg.norm(x_ref), 1.0)
    assert rep.trace[-1].primal_inf <= max(10 * float(IPM[pre + "primal"][-1]), cfg.mu_tol)
    assert rep.trace[-1].dual_inf <= max(10 * float(IPM[pre + "dual"][-1]), cfg.mu_tol)
    print(f"{name}: IPM {rep.iterations} (ref {int(IPM[pre + 'iterations'])}), CG {rep.cg_total} "
          f"(ref {int(IPM[pre + 'cg_iters'].sum())}), {rep.wall_time:.3f}s")
