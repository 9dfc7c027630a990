"""Pin the CPU oracle (oracle/qp_oracle.py) to the real reference.

The fixtures in tests/golden/ were produced by running qpipm itself
(oracle/make_golden.py).  The oracle restates the reference's operation
order, so on the same inputs it must agree BIT FOR BIT: operator applies,
Jacobi diagonals, PCG iteration counts, residual histories and solutions,
and the IPM trajectory.
"""

import numpy as np
import pytest

import golden_io
from oracle import qp_oracle as orc
from paper_2308_00637_b200 import workloads
from paper_2308_00637_b200.problem import build_operator

INST = golden_io.load("instances")
N_INST = int(INST["count"])


@pytest.mark.parametrize("i", range(N_INST))
def test_instance_bitwise(i):
    problem, state, op, pre = golden_io.instance(INST, i)
    np.testing.assert_array_equal(op.d_diag, INST[pre + "d_diag"])
    np.testing.assert_array_equal(op.q_diag_extra, INST[pre + "q_extra"])
    np.testing.assert_array_equal(orc.jacobi_diagonal(op), INST[pre + "jacobi"])
    for v, y in zip(INST[pre + "vecs"], INST[pre + "applies"]):
        np.testing.assert_array_equal(orc.apply_doubly_augmented(op, v), y)
    res = orc.compute_residuals(problem, state, op.bmap)
    rhs = orc.assemble_rhs(op, res, state)
    np.testing.assert_array_equal(rhs, INST[pre + "rhs"])
    hist = []
    cfg = orc.PcgConfig(tol=1e-10, max_iters=20000)
    try:
        out = orc.pcg_direction(op, rhs, cfg, callback=lambda k, x, rn: hist.append(rn))
        breakdown = 0
    except orc.PcgBreakdownError as exc:
        out, breakdown = exc.result, 1
    assert breakdown == int(INST[pre + "pcg_breakdown"])
    assert out.iterations == int(INST[pre + "pcg_iters"])
    assert out.converged == bool(INST[pre + "pcg_conv"])
    assert out.final_residual_norm == float(INST[pre + "pcg_final"])
    np.testing.assert_array_equal(out.solution, INST[pre + "pcg_x"])
    np.testing.assert_array_equal(np.array([np.linalg.norm(rhs)] + hist), INST[pre + "pcg_hist"])


CFG = golden_io.load("configs")
SPECS = {
    "cfg1": (workloads.dense_qp, dict(seed=0)),
    "cfg2": (workloads.svm_primal, dict(seed=2, d=40, n_samples=1500)),
    "cfg3": (workloads.rt_like, dict(seed=3, n_vox=6000, n_beam=600, density=0.02)),
    "cfg5": (workloads.random_sweep, dict(seed=5, m=20000, n=5000)),
}


def config_case(name):
    fn, kw = SPECS[name]
    assert str(CFG[name + "_kw"]) == repr(kw)
    problem, state, meta = fn(**kw)
    a = problem.a.values
    assert np.sum(a * (1 + np.arange(len(a)) % 7)) == float(CFG[name + "_checksum_a"]), "generator drifted"
    return problem, state, meta, build_operator(problem, state)


@pytest.mark.parametrize("name", sorted(SPECS))
def test_config_oracle_bitwise(name):
    problem, state, meta, op = config_case(name)
    pre = name + "_"
    np.testing.assert_array_equal(op.d_diag, CFG[pre + "d_diag"])
    np.testing.assert_array_equal(orc.jacobi_diagonal(op), CFG[pre + "jacobi"])
    for v, y in zip(CFG[pre + "vecs"], CFG[pre + "applies"]):
        np.testing.assert_array_equal(orc.apply_doubly_augmented(op, v), y)
    rhs = CFG[pre + "rhs"]
    if name == "cfg5":
        np.testing.assert_array_equal(rhs, meta["rhs"])
        cfg = orc.PcgConfig(tol=1e-300, max_iters=200)
    else:
        cfg = orc.PcgConfig(tol=1e-7, max_iters=400)
    hist = []
    out = orc.pcg_direction(op, rhs, cfg, callback=lambda k, x, rn: hist.append(rn))
    assert out.iterations == int(CFG[pre + "pcg_iters"])
    np.testing.assert_array_equal(np.array([np.linalg.norm(rhs)] + hist), CFG[pre + "pcg_hist"])
    np.testing.assert_array_equal(out.solution, CFG[pre + "pcg_x"])
