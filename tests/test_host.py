"""Host-side logic: mirror containers, generators, oracle self-consistency."""

import numpy as np
import pytest

from oracle import qp_oracle as orc
from paper_2308_00637_b200 import workloads
from paper_2308_00637_b200.pcg import PcgConfig
from paper_2308_00637_b200.problem import DimensionError, SparseMatrix, build_operator


def test_sparse_matrix_validation():
    SparseMatrix(2, 3, [0, 1, 3], [2, 0, 2], [1.0, 2.0, 3.0])
    with pytest.raises(ValueError):
        SparseMatrix(2, 3, [0, 2, 3], [2, 0, 1], [1.0, 2.0, 3.0])    # 2 then 0 inside row 0
    with pytest.raises(ValueError):
        SparseMatrix(1, 3, [0, 2], [1, 1], [1.0, 2.0])                # duplicate
    with pytest.raises(ValueError):
        SparseMatrix(1, 3, [0, 1], [3], [1.0])                        # out of range
    with pytest.raises(DimensionError):
        SparseMatrix(2, 3, [0, 1], [0], [1.0])
    m = SparseMatrix.from_dense([[0, 1.0, 0], [2.0, 0, 3.0]])
    np.testing.assert_array_equal(m.row_offsets, [0, 1, 3])
    np.testing.assert_array_equal(m.col_indices, [1, 0, 2])


def test_row_submatrix_arrays():
    rng = np.random.default_rng(0)
    dense = np.where(rng.random((9, 7)) < 0.4, rng.standard_normal((9, 7)), 0.0)
    m = SparseMatrix.from_dense(dense)
    rows = np.array([8, 0, 3, 3])
    ro, ci, v = m.row_submatrix_arrays(rows)
    sub = np.zeros((len(rows), 7))
    for i in range(len(rows)):
        sub[i, ci[ro[i]:ro[i + 1]]] = v[ro[i]:ro[i + 1]]
    np.testing.assert_array_equal(sub, dense[rows])


def test_pcg_config_validation():
    with pytest.raises(ValueError):
        PcgConfig(tol=0.0)
    with pytest.raises(ValueError):
        PcgConfig(max_iters=0)


def test_generators_are_deterministic_and_shaped():
    p1, s1, m1 = workloads.random_sweep(seed=3, m=500, n=100)
    p2, s2, m2 = workloads.random_sweep(seed=3, m=500, n=100)
    np.testing.assert_array_equal(p1.a.col_indices, p2.a.col_indices)
    np.testing.assert_array_equal(m1["rhs"], m2["rhs"])
    assert p1.a.nnz == 500 * 16
    cols = p1.a.col_indices.reshape(500, 16)
    assert np.all(np.diff(cols, axis=1) > 0)
    op = build_operator(p1, s1)
    np.testing.assert_array_equal(op.d_diag, s1.s_lA)       # d_diag = w (kkt.py:200)
    p, s, meta = workloads.svm_primal(seed=2, d=10, n_samples=50)
    assert p.a.nnz == 50 * 12 and p.n == 61
    p, s, meta = workloads.rt_like(seed=3, n_vox=1000, n_beam=50, density=0.05)
    assert p.hessian.m.n_rows == 50
    assert np.all(np.isfinite(p.p))
    p, s, meta = workloads.dense_qp(seed=0, n=20, m=40)
    assert p.a.nnz == 800


def test_oracle_operator_is_symmetric_positive_definite(rng):
    p, s, meta = workloads.svm_primal(seed=2, d=8, n_samples=40)
    op = build_operator(p, s)
    for _ in range(20):
        u, v = rng.standard_normal(op.dim), rng.standard_normal(op.dim)
        ku, kv = orc.apply_doubly_augmented(op, u), orc.apply_doubly_augmented(op, v)
        assert abs(u @ kv - v @ ku) <= 1e-10 * (1 + abs(u @ kv))
        assert v @ kv > 0


def test_operator_cache_identity_and_content(monkeypatch):
    """operator_for (direction.py): one device operator per live problem; the
    same bound-index arrays skip hashing, equal contents in new arrays reuse
    the operator, different bounds rebuild it (no device needed: GpuKkt is
    stubbed)."""
    from types import SimpleNamespace

    from paper_2308_00637_b200 import direction

    built = []

    class FakeKkt:
        def __init__(self, problem, bmap, device=0):
            built.append(bmap)

        def close(self):
            pass

    monkeypatch.setattr(direction, "GpuKkt", FakeKkt)
    monkeypatch.setattr(direction, "_CACHE", {})
    problem = SimpleNamespace()
    lo, up = np.array([0, 2, 5]), np.array([1, 3])
    op = SimpleNamespace(problem=problem, bmap=SimpleNamespace(lin_lower=lo, lin_upper=up))
    gk = direction.operator_for(op)
    assert direction.operator_for(op) is gk and len(built) == 1
    key_fn = direction._bmap_key
    monkeypatch.setattr(direction, "_bmap_key", lambda b: (_ for _ in ()).throw(AssertionError("hashed")))
    assert direction.operator_for(op) is gk          # same array objects: no hashing
    monkeypatch.setattr(direction, "_bmap_key", key_fn)
    op2 = SimpleNamespace(problem=problem, bmap=SimpleNamespace(lin_lower=lo.copy(), lin_upper=up.copy()))
    assert direction.operator_for(op2) is gk and len(built) == 1
    op3 = SimpleNamespace(problem=problem, bmap=SimpleNamespace(lin_lower=np.array([0, 2]), lin_upper=up))
    assert direction.operator_for(op3) is not gk and len(built) == 2
