"""SVM dual frontend, host side (no GPU).

* the CPU restatement (oracle/svm_oracle.py) is pinned bit for bit to the
  reference's own outputs in tests/golden/svm.npz (oracle/make_golden_svm.py
  ran qpipm.svm): Gram Hessian, IPM solution, bias, decision values;
* this package's host logic -- LIBSVM parsing with the reference's errors
  (test_svm.py:23-56 cases), rbf_kernel, predict -- against the same fixtures;
* the device entry points refuse to run without CUDA (no CPU fallback).
"""

import math

import numpy as np
import pytest

import golden_io
from oracle import qp_oracle as orc
from oracle import svm_oracle as so
from paper_2308_00637_b200 import _native, svm

SVM = golden_io.load("svm")
NAMES = [str(s) for s in SVM["names"]]


def _case(name):
    p = name + "_"
    sigma, c = SVM[p + "sigma_c"]
    return SVM[p + "x"], SVM[p + "y"], float(sigma), float(c), p


@pytest.mark.parametrize("name", NAMES)
def test_oracle_hessian_bitwise(name):
    x, y, sigma, c, p = _case(name)
    h = so.dual_hessian(x, y, sigma)
    np.testing.assert_array_equal(h, SVM[p + "H"])
    assert np.array_equal(h, h.T)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_ipm_and_model_bitwise(name):
    x, y, sigma, c, p = _case(name)
    rep = orc.solve(so.dual_problem(x, y, sigma, c), orc.IpmConfig())
    assert rep.status == str(SVM[p + "status"])
    assert rep.iterations == int(SVM[p + "iterations"])
    np.testing.assert_array_equal(rep.x, SVM[p + "alpha"])
    np.testing.assert_array_equal(so.decision_values(x, y, sigma, rep.x), SVM[p + "decision"])
    assert so.bias(x, y, sigma, c, rep.x) == float(SVM[p + "bias"])


@pytest.mark.parametrize("name", NAMES)
def test_parse_libsvm_reads_fixture_text(name):
    x, y, _, _, p = _case(name)
    data = svm.parse_libsvm(str(SVM[p + "text"]))
    np.testing.assert_array_equal(data.dense_matrix(), x)
    np.testing.assert_array_equal(data.labels, y)
    assert len(data) == len(y)


@pytest.mark.parametrize("name", NAMES)
def test_predict_matches_reference(name):
    x, y, sigma, c, p = _case(name)
    data = svm.parse_libsvm(str(SVM[p + "text"]))
    alpha = SVM[p + "alpha"]
    model = svm.SvmModel(alpha=alpha, bias=float(SVM[p + "bias"]), support_indices=SVM[p + "support"],
                         dataset=data, config=svm.SvmConfig(sigma=sigma, c=c))
    for vals, s_ref, lab_ref in zip(SVM[p + "probes"], SVM[p + "probe_scores"], SVM[p + "probe_labels"]):
        score, lab = svm.predict(model, svm.SparseVector(np.arange(len(vals)), vals))
        assert score == pytest.approx(float(s_ref), rel=1e-12, abs=1e-12)
        assert lab == int(lab_ref)


# test_svm.py:23-56 -- parser behaviour
def test_parse_basic_format():
    data = svm.parse_libsvm("+1 1:0.5 3:1\n-1 2:2")
    assert len(data) == 2 and data.n_features == 3
    np.testing.assert_array_equal(data.labels, [1.0, -1.0])
    np.testing.assert_array_equal(data.samples[0].indices, [0, 2])
    np.testing.assert_array_equal(data.samples[1].values, [2.0])


@pytest.mark.parametrize("text, match", [
    ("", "no samples"),
    ("+2 1:1", "line 1: non-binary label"),
    ("+1 1:1\nabc 1:1", "line 2: label 'abc' is not numeric"),
    ("+1 1-1", "line 1: malformed feature '1-1'"),
    ("+1 1:x", "malformed feature"),
    ("+1 2:1 2:3", "not strictly increasing"),
    ("+1 0:1", "not strictly increasing"),
])
def test_parse_errors(text, match):
    with pytest.raises(svm.SvmParseError, match=match):
        svm.parse_libsvm(text)


def test_parse_bytes_and_blank_lines():
    data = svm.parse_libsvm(b"\n+1 1:1\n\n   \n-1 2:1\n")
    assert len(data) == 2 and data.n_features == 2


def test_rbf_kernel_known_answers():
    a = svm.SparseVector([0], [1.0])
    b = svm.SparseVector([1], [1.0])
    assert svm.rbf_kernel(a, a, 1.0) == 1.0
    assert svm.rbf_kernel(a, b, 1.0) == pytest.approx(math.exp(-1.0))      # |a-b|^2 = 2 = 2 sigma
    assert svm.rbf_kernel(a, b, 2.0) == pytest.approx(math.exp(-0.5))


def test_config_validation():
    with pytest.raises(ValueError):
        svm.SvmConfig(sigma=0.0, c=1.0)
    with pytest.raises(ValueError):
        svm.SvmConfig(sigma=1.0, c=-1.0)


def test_build_rejects_single_class_and_cap():
    data = svm.parse_libsvm("+1 1:1\n+1 1:2")
    with pytest.raises(ValueError, match="each class"):
        svm.build_svm_dual(data, svm.SvmConfig(sigma=1.0, c=1.0))


def test_device_path_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    data = svm.parse_libsvm("+1 1:1\n-1 2:1\n")
    with pytest.raises(_native.NativeUnavailable):
        svm.build_svm_dual(data, svm.SvmConfig(sigma=1.0, c=1.0))
    with pytest.raises(_native.NativeUnavailable):
        svm.decision_values(data, svm.SvmConfig(sigma=1.0, c=1.0), np.ones(2))
