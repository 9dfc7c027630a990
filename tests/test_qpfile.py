"""QP file dialect (qpipm/cli.py:37-183) against the reference's own parser.

tests/golden/qpfile.npz (oracle/make_golden_qpfile.py) holds documents the
reference wrote (cli.qp_document) or hand-written ones with nulls, duplicate
COO entries and absent optional members, and the arrays the reference's
parse_qp_document built from them: this package's parser must build the same
arrays bit for bit; the writer must round-trip; errors name the member like
the reference's (test_cli.py:44-55).  The GPU test solves each file with the
device IPM against the reference's solve().
"""

import json

import numpy as np
import pytest

import golden_io
from paper_2308_00637_b200 import qpfile
from paper_2308_00637_b200.problem import DenseHessian

G = golden_io.load("qpfile")
NAMES = [str(s) for s in G["names"]]


def _check(prob, pre):
    for m in ("a", "c"):
        mat = getattr(prob, m)
        np.testing.assert_array_equal(mat.row_offsets, G[pre + m + "_ro"])
        np.testing.assert_array_equal(mat.col_indices, G[pre + m + "_ci"])
        np.testing.assert_array_equal(mat.values, G[pre + m + "_v"])
    np.testing.assert_array_equal(prob.p, G[pre + "p"])
    np.testing.assert_array_equal(prob.b, G[pre + "b"])
    if G[pre + "bounds"].shape[1]:
        np.testing.assert_array_equal(np.stack([prob.lin_bounds.lower, prob.lin_bounds.upper]), G[pre + "bounds"])
    np.testing.assert_array_equal(np.stack([prob.var_bounds.lower, prob.var_bounds.upper]), G[pre + "vbounds"])
    h = prob.hessian
    assert type(h).__name__ == str(G[pre + "hkind"])
    if type(h).__name__ == "DiagonalHessian":
        np.testing.assert_array_equal(h.d, G[pre + "h_d"])
    elif type(h).__name__ == "SparseHessian":
        np.testing.assert_array_equal(h.m.row_offsets, G[pre + "h_ro"])
        np.testing.assert_array_equal(h.m.col_indices, G[pre + "h_ci"])
        np.testing.assert_array_equal(h.m.values, G[pre + "h_v"])
    else:
        np.testing.assert_array_equal(h.h0_diag, G[pre + "h_h0"])
        np.testing.assert_array_equal(h.u, G[pre + "h_u"])
        np.testing.assert_array_equal(h.w, G[pre + "h_w"])


@pytest.mark.parametrize("name", NAMES)
def test_parse_matches_reference(name):
    _check(qpfile.parse_qp_document(json.loads(str(G[name + "_text"]))), name + "_")


@pytest.mark.parametrize("name", NAMES)
def test_round_trip(name, tmp_path):
    prob = qpfile.parse_qp_document(json.loads(str(G[name + "_text"])))
    path = tmp_path / "p.json"
    path.write_text(json.dumps(qpfile.qp_document(prob)))
    _check(qpfile.load_qp_file(str(path)), name + "_")


BASE = {"n": 2, "hessian": {"kind": "diagonal", "d": [1, 1]}, "p": [0, 0]}


@pytest.mark.parametrize("patch, match", [
    ({"p": None}, "'p'"),
    ({"hessian": {"kind": "dense"}}, "hessian.kind"),
    ({"hessian": {"d": [1, 1]}}, "'hessian' must be an object with a 'kind'"),
    ({"hessian": {"kind": "diagonal", "d": [1]}}, "hessian.d"),
    ({"n": -1}, "'n' must be a nonnegative integer"),
    ({"n": True}, "'n' must be a nonnegative integer"),
    ({"p": [0, None]}, "'p' contains null at position 1"),
    ({"p": [0, "x"]}, "'p' contains non-numeric entry at position 1"),
    ({"l": [0], "u": [1, 2]}, "'l' and 'u' have different lengths"),
    ({"l": [0], "u": [1], "A": {"rows": [0], "cols": [5], "vals": [1]}}, "coordinate index out of range"),
    ({"l": [0], "u": [1], "A": {"rows": [0], "vals": [1]}}, "'A' is missing 'cols'"),
    ({"l": [0], "u": [1], "A": {"rows": [0, 0], "cols": [0], "vals": [1]}}, "lengths differ"),
    ({"hessian": {"kind": "bfgs", "h0_diag": [1, 1], "w": [1], "u": [[1]]}}, "n-row array"),
])
def test_errors_name_the_member(patch, match):
    doc = dict(BASE)
    for k, v in patch.items():
        if v is None:
            doc.pop(k)
        else:
            doc[k] = v
    with pytest.raises(qpfile.QpFileError, match=match):
        qpfile.parse_qp_document(doc)


def test_root_and_io_errors(tmp_path):
    with pytest.raises(qpfile.QpFileError, match="root must be an object"):
        qpfile.parse_qp_document([1, 2])
    with pytest.raises(qpfile.QpFileError, match="cannot read"):
        qpfile.load_qp_file(str(tmp_path / "missing.json"))
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    with pytest.raises(qpfile.QpFileError, match="not valid JSON"):
        qpfile.load_qp_file(str(bad))


def test_dense_hessian_has_no_file_form():
    prob = qpfile.parse_qp_document(BASE)
    dense = type(prob)(n=2, hessian=DenseHessian(np.eye(2)), p=prob.p, a=prob.a, lin_bounds=prob.lin_bounds,
                       c=prob.c, b=prob.b, var_bounds=prob.var_bounds)
    with pytest.raises(qpfile.QpFileError, match="dense Hessians"):
        qpfile.qp_document(dense)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_solve_file_matches_reference(name, tmp_path):
    path = tmp_path / "p.json"
    path.write_text(str(G[name + "_text"]))
    rep = qpfile.solve_file(str(path))
    assert rep.status.value == str(G[name + "_status"])
    x_ref = G[name + "_x"]
    assert np.linalg.norm(rep.x - x_ref) <= 1e-6 * max(np.linalg.norm(x_ref), 1.0)
    obj = float(G[name + "_objective"])
    assert abs(rep.objective - obj) <= 1e-6 * max(abs(obj), 1.0)
