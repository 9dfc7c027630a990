"""SVM dual frontend on the GPU against the reference's outputs (tests/golden/svm.npz).

* Hessian from qpk_rbf_hessian_dev: exactly symmetric (bitwise) and within
  1e-13 absolute (entries lie in [-1, 1]) of the reference's build_svm_dual;
  the two-point known answers of test_svm.py:85-97;
* train = build_svm_dual + the device IPM (dense-H PCG every iteration) +
  extract_model: same status, alpha and objective within 1e-6 relative, bias
  within 1e-5, decision values within 1e-6 relative, same training accuracy
  (SURVEY.md 8(c) IPM tolerances);
* a larger synthetic dual (n = 2000, 31 Gram tiles per edge) against the
  oracle restatement.
"""

import math

import numpy as np
import pytest

import golden_io
from oracle import svm_oracle as so
from paper_2308_00637_b200 import svm

pytestmark = pytest.mark.gpu

SVM = golden_io.load("svm")
NAMES = [str(s) for s in SVM["names"]]


def _case(name):
    p = name + "_"
    sigma, c = SVM[p + "sigma_c"]
    data = svm.parse_libsvm(str(SVM[p + "text"]))
    return data, svm.SvmConfig(sigma=float(sigma), c=float(c)), p


@pytest.mark.parametrize("name", NAMES)
def test_device_hessian(name):
    data, cfg, p = _case(name)
    h = svm.rbf_hessian_device(data, cfg.sigma).cpu().numpy()
    assert np.array_equal(h, h.T)
    assert np.max(np.abs(h - SVM[p + "H"])) <= 1e-13


def test_two_point_structure():
    data = svm.parse_libsvm("+1 1:1\n-1 2:1\n")
    prob = svm.build_svm_dual(data, svm.SvmConfig(sigma=1.0, c=1.0))
    h = prob.hessian.to_host()
    assert h[0, 0] == 1.0 and h[1, 1] == 1.0
    assert h[0, 1] == pytest.approx(-math.exp(-1.0), rel=1e-15)
    np.testing.assert_array_equal(prob.c.values, [1.0, -1.0])
    np.testing.assert_array_equal(prob.p, [-1.0, -1.0])
    np.testing.assert_array_equal(prob.var_bounds.upper, [1.0, 1.0])


@pytest.mark.parametrize("name", NAMES)
def test_train_matches_reference(name):
    data, cfg, p = _case(name)
    rep, model = svm.train(data, cfg)
    assert rep.status.value == str(SVM[p + "status"])
    a_ref = SVM[p + "alpha"]
    assert np.linalg.norm(rep.x - a_ref) <= 1e-6 * max(np.linalg.norm(a_ref), 1.0)
    obj = float(SVM[p + "objective"])
    assert abs(rep.objective - obj) <= 1e-6 * max(abs(obj), 1.0)
    assert model is not None
    assert abs(model.bias - float(SVM[p + "bias"])) <= 1e-5
    g_ref = SVM[p + "decision"]
    g = svm.decision_values(data, cfg, rep.x)
    assert np.linalg.norm(g - g_ref) <= 1e-6 * max(np.linalg.norm(g_ref), 1.0)
    assert svm.training_accuracy(model) == float(SVM[p + "accuracy"])
    # the box and the equality constraint (test_svm.py:179-187)
    assert np.max(np.maximum(-rep.x, rep.x - cfg.c)) <= 1e-6 * cfg.c
    assert abs(rep.x @ data.labels) <= 1e-5 * len(data)
    print(f"{name}: IPM {rep.iterations} (ref {int(SVM[p + 'iterations'])}), CG {rep.cg_total}, "
          f"{rep.wall_time:.3f}s")


def test_decision_values_exact_hessian_identity():
    # g = K (a o y) = y o (H a): the device GEMV against the oracle's Gram product
    x, y = so.synthetic_dataset(21, 300, 7)
    data = svm.SvmDataset.from_dense(x, y)
    cfg = svm.SvmConfig(sigma=3.0, c=1.0)
    a = np.random.default_rng(3).random(300)
    g = svm.decision_values(data, cfg, a)
    g_ref = so.decision_values(x, y, cfg.sigma, a)
    assert np.linalg.norm(g - g_ref) <= 1e-12 * np.linalg.norm(g_ref)


def test_large_hessian_against_oracle():
    x, y = so.synthetic_dataset(22, 2000, 50)
    data = svm.SvmDataset.from_dense(x, y)
    h = svm.rbf_hessian_device(data, 25.0).cpu().numpy()
    h_ref = so.dual_hessian(x, y, 25.0)
    assert np.array_equal(h, h.T)
    assert np.max(np.abs(h - h_ref)) <= 1e-13


def test_packed_symmetric_hessian_apply():
    # n >= QPK_SYM_MIN_N: H is applied from its packed upper tiles (hess_sym);
    # n = 1100 is not a multiple of the 64-wide tile (zero padding)
    from oracle import qp_oracle as orc
    from paper_2308_00637_b200.direction import GpuKkt
    from paper_2308_00637_b200.problem import build_operator
    from paper_2308_00637_b200.workloads import _state_from_initial
    x, y = so.synthetic_dataset(23, 1100, 10)
    cfg = svm.SvmConfig(sigma=4.0, c=1.0)
    prob = svm.build_svm_dual(svm.SvmDataset.from_dense(x, y), cfg)
    host = so.dual_problem(x, y, cfg.sigma, cfg.c)
    op_h = build_operator(host, _state_from_initial(host))
    gk = GpuKkt(prob, op_h.bmap)
    assert gk.ctx.query("hess_sym") == 1
    gk.set_diagonals(op_h.d_diag, op_h.q_diag_extra)
    rng = np.random.default_rng(5)
    for _ in range(3):
        v = rng.standard_normal(op_h.dim)
        y_gpu = gk.apply(v)
        y_ref = orc.apply_doubly_augmented(op_h, v)
        assert np.linalg.norm(y_gpu - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    # PCG history against the oracle's: 1e-8 until the CPU-reorder envelope
    # leaves it, then within 10x that envelope (tests/parity.py)
    import parity
    rhs = rng.standard_normal(op_h.dim)
    cfg_p = orc.PcgConfig(tol=1e-300, max_iters=40)
    xg, info, hist = gk.pcg(rhs, 1e-300, 40, True, history=True)
    ref_hist = []
    orc.pcg_direction(op_h, rhs, cfg_p, callback=lambda k, xk, rn: ref_hist.append(rn))
    h_ref = np.array([np.linalg.norm(rhs)] + ref_hist)
    assert info.iterations == 40
    env = parity.envelope(op_h, rhs, cfg_p, h_ref)
    ok, msg = parity.check_history(hist, h_ref, env)
    assert ok, msg
    # no atomics on this path: partials are summed in a fixed order
    xg2, _, hist2 = gk.pcg(rhs, 1e-300, 40, True, history=True)
    np.testing.assert_array_equal(xg, xg2)
    np.testing.assert_array_equal(hist, hist2)
    np.testing.assert_array_equal(gk.apply(v), gk.apply(v))
    gk.close()


def test_unsymmetric_dense_hessian_is_not_packed():
    """DenseHessian documents symmetry but the reference multiplies whatever it
    is given (model.py:165-176: h.m @ v).  A dense H that is not bitwise
    symmetric must keep the row-major apply, not the mirrored upper triangle."""
    from oracle import qp_oracle as orc
    from paper_2308_00637_b200.direction import GpuKkt
    from paper_2308_00637_b200.problem import (Bounds, DenseHessian, IterateState, QpProblem, SparseMatrix,
                                               build_operator)
    rng = np.random.default_rng(31)
    n = 640
    g = rng.standard_normal((n, n))
    h = g @ g.T + n * np.eye(n)
    h[3, 500] += 0.25                                    # one entry off: H != H'
    problem = QpProblem(n=n, hessian=DenseHessian(h), p=np.zeros(n), a=SparseMatrix.empty(0, n),
                        lin_bounds=Bounds.free(0), c=SparseMatrix.empty(0, n), b=[], var_bounds=Bounds.free(n))
    z = np.zeros(0)
    state = IterateState(x=np.zeros(n), s_lA=z, s_uA=z, s_lx=z, s_ux=z, lam_e=z, lam_lA=z, lam_uA=z, lam_lx=z,
                         lam_ux=z, mu=0.5)
    op = build_operator(problem, state)
    gk = GpuKkt(problem, op.bmap)
    assert gk.ctx.query("hess_symmetric") == 0 and gk.ctx.query("hess_sym") == 0
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    v = rng.standard_normal(n)
    y_ref = orc.apply_doubly_augmented(op, v)
    assert np.linalg.norm(gk.apply(v) - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    gk.close()
    h[3, 500] -= 0.25
    h = 0.5 * (h + h.T)
    problem = QpProblem(n=n, hessian=DenseHessian(h), p=np.zeros(n), a=SparseMatrix.empty(0, n),
                        lin_bounds=Bounds.free(0), c=SparseMatrix.empty(0, n), b=[], var_bounds=Bounds.free(n))
    op = build_operator(problem, state)
    gk = GpuKkt(problem, op.bmap)
    assert gk.ctx.query("hess_symmetric") == 1 and gk.ctx.query("hess_sym") == 1
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    y_ref = orc.apply_doubly_augmented(op, v)
    assert np.linalg.norm(gk.apply(v) - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    gk.close()


def test_train_packed_matches_oracle_ipm():
    from oracle import qp_oracle as orc
    x, y = so.synthetic_dataset(24, 700, 8, sep=3.0)
    cfg = svm.SvmConfig(sigma=8.0, c=1.0)
    rep, model = svm.train(svm.SvmDataset.from_dense(x, y), cfg)
    ref = orc.solve(so.dual_problem(x, y, cfg.sigma, cfg.c), orc.IpmConfig())
    assert rep.status.value == ref.status
    assert np.linalg.norm(rep.x - ref.x) <= 1e-6 * max(np.linalg.norm(ref.x), 1.0)
    assert abs(rep.objective - ref.objective) <= 1e-6 * max(abs(ref.objective), 1.0)
    assert abs(model.bias - so.bias(x, y, cfg.sigma, cfg.c, ref.x)) <= 1e-5


@pytest.mark.parametrize("scatter", [1, 2])
def test_dense_row_split_both_scatter_modes(scatter):
    # the equality row y'alpha = 0 has n >= 2048 entries: the slot engine
    # applies it as a dense vector (top-kernel partials + k_slot_dense), in the
    # atomic (1) and CSC (2) modes; apply, Jacobi and a PCG history vs the oracle
    import parity
    from oracle import qp_oracle as orc
    from paper_2308_00637_b200.direction import GpuKkt
    from paper_2308_00637_b200.problem import build_operator
    from paper_2308_00637_b200.workloads import _state_from_initial
    x, y = so.synthetic_dataset(25, 3000, 6)
    cfg = svm.SvmConfig(sigma=3.0, c=1.0)
    prob = svm.build_svm_dual(svm.SvmDataset.from_dense(x, y), cfg)
    host = so.dual_problem(x, y, cfg.sigma, cfg.c)
    op_h = build_operator(host, _state_from_initial(host))
    gk = GpuKkt(prob, op_h.bmap, scatter=scatter)
    assert gk.ctx.query("dense_rows") == 1 and gk.ctx.query("scatter") == scatter
    gk.set_diagonals(op_h.d_diag, op_h.q_diag_extra)
    assert parity.rel_err(gk.jacobi(), orc.jacobi_diagonal(op_h)) <= parity.APPLY_TOL
    rng = np.random.default_rng(6)
    v = rng.standard_normal(op_h.dim)
    assert parity.rel_err(gk.apply(v), orc.apply_doubly_augmented(op_h, v)) <= parity.APPLY_TOL
    rhs = rng.standard_normal(op_h.dim)
    cfg_p = orc.PcgConfig(tol=1e-10, max_iters=300)
    xg, info, hist = gk.pcg(rhs, cfg_p.tol, cfg_p.max_iters, True, history=True)
    ref_hist = []
    ref = orc.pcg_direction(op_h, rhs, cfg_p, callback=lambda k, xk, rn: ref_hist.append(rn))
    h_ref = np.array([np.linalg.norm(rhs)] + ref_hist)
    ok, msg = parity.check_history(hist, h_ref, parity.envelope(op_h, rhs, cfg_p, h_ref))
    assert ok, msg
    assert parity.rel_err(xg, ref.solution) <= 1e-6
    gk.close()
