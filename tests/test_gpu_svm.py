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
