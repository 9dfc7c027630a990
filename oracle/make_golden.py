"""Generate tests/golden/*.npz by running the REAL reference (qpipm) here.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference is
mounted read-only at /root/reference:

    python oracle/make_golden.py

It imports ``qpipm`` from /root/reference/pkg/src and the reference's own test
generators from /root/reference/pkg/tests/oracles.py, and records, for the
same seeded instances the reference's tests use, the reference's outputs:
operator applies, Jacobi diagonals, right-hand sides, PCG results with full
residual histories (via pcg's callback, linalg.py:71, 108-109) and IPM
results.  The fixtures travel to the GPU box (the reference does not); the
CPU oracle (oracle/qp_oracle.py) is pinned against them in
tests/test_oracle_golden.py and the CUDA path in tests/test_gpu_parity.py.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import qpipm.ipm as ref_ipm  # noqa: E402
import qpipm.kkt as ref_kkt  # noqa: E402
import qpipm.linalg as ref_linalg  # noqa: E402
import qpipm.model as ref_model  # noqa: E402
from oracles import random_interior_state, random_problem  # noqa: E402  (reference tests)

from paper_2308_00637_b200 import workloads  # noqa: E402

OUT = ROOT / "tests" / "golden"


# ----------------------------------------------------------------------------
def pack_problem(prefix, problem, out):
    out[prefix + "n"] = np.int64(problem.n)
    for name, m in (("a", problem.a), ("c", problem.c)):
        out[f"{prefix}{name}_shape"] = np.array([m.n_rows, m.n_cols], dtype=np.int64)
        out[f"{prefix}{name}_ro"] = np.asarray(m.row_offsets, dtype=np.int64)
        out[f"{prefix}{name}_ci"] = np.asarray(m.col_indices, dtype=np.int64)
        out[f"{prefix}{name}_v"] = np.asarray(m.values, dtype=np.float64)
    h = problem.hessian
    kind = type(h).__name__
    out[prefix + "hkind"] = np.array(kind)
    if kind == "DiagonalHessian":
        out[prefix + "h_d"] = h.d
    elif kind == "SparseHessian":
        out[prefix + "h_ro"] = h.m.row_offsets
        out[prefix + "h_ci"] = h.m.col_indices
        out[prefix + "h_v"] = h.m.values
    elif kind == "DenseHessian":
        out[prefix + "h_m"] = h.m
    else:
        out[prefix + "h_h0"] = h.h0_diag
        out[prefix + "h_u"] = h.u
        out[prefix + "h_w"] = h.w
    out[prefix + "p"] = problem.p
    out[prefix + "b"] = problem.b
    out[prefix + "lin_lo"] = problem.lin_bounds.lower
    out[prefix + "lin_hi"] = problem.lin_bounds.upper
    out[prefix + "var_lo"] = problem.var_bounds.lower
    out[prefix + "var_hi"] = problem.var_bounds.upper


STATE_KEYS = ("x", "s_lA", "s_uA", "s_lx", "s_ux", "lam_e", "lam_lA", "lam_uA", "lam_lx", "lam_ux")


def pack_state(prefix, state, out):
    for k in STATE_KEYS:
        out[prefix + "st_" + k] = getattr(state, k)
    out[prefix + "st_mu"] = np.float64(state.mu)


def to_ref_problem(p):
    """package mirror QpProblem -> reference QpProblem (same fields)."""
    h = p.hessian
    kind = type(h).__name__
    if kind == "DiagonalHessian":
        rh = ref_model.DiagonalHessian(h.d)
    elif kind == "SparseHessian":
        rh = ref_model.SparseHessian(_ref_sparse(h.m))
    elif kind == "DenseHessian":
        rh = ref_model.DenseHessian(h.m)
    else:
        rh = ref_model.QuasiNewtonHessian(h.h0_diag, h.u, h.w)
    return ref_model.QpProblem(
        n=p.n, hessian=rh, p=p.p, a=_ref_sparse(p.a),
        lin_bounds=ref_model.Bounds(p.lin_bounds.lower, p.lin_bounds.upper),
        c=_ref_sparse(p.c), b=p.b,
        var_bounds=ref_model.Bounds(p.var_bounds.lower, p.var_bounds.upper))


def _ref_sparse(m):
    # bypass the reference constructor's per-row Python loop for big matrices:
    # the arrays were validated by the package's vectorised constructor
    obj = object.__new__(ref_model.SparseMatrix)
    object.__setattr__(obj, "n_rows", m.n_rows)
    object.__setattr__(obj, "n_cols", m.n_cols)
    object.__setattr__(obj, "row_offsets", np.asarray(m.row_offsets, dtype=np.int64))
    object.__setattr__(obj, "col_indices", np.asarray(m.col_indices, dtype=np.int64))
    object.__setattr__(obj, "values", np.asarray(m.values, dtype=np.float64))
    return obj


def to_ref_state(s):
    return ref_kkt.IterateState(**{k: np.array(getattr(s, k), dtype=np.float64) for k in STATE_KEYS}, mu=s.mu)


def record_operator(prefix, op, rng_vec, out, n_vec=3, pcg_cfg=None, hist_cap=None, rhs=None):
    out[prefix + "d_diag"] = op.d_diag
    out[prefix + "q_extra"] = op.q_diag_extra
    out[prefix + "jacobi"] = ref_kkt.jacobi_diagonal(op)
    vs = rng_vec.standard_normal((n_vec, op.dim))
    out[prefix + "vecs"] = vs
    out[prefix + "applies"] = np.stack([ref_kkt.apply_doubly_augmented(op, v) for v in vs])
    if pcg_cfg is not None:
        hist = []
        try:
            inv = 1.0 / ref_kkt.jacobi_diagonal(op)
            res = ref_linalg.pcg(lambda v: ref_kkt.apply_doubly_augmented(op, v), lambda v: inv * v,
                                 rhs, pcg_cfg, callback=lambda k, x, rn: hist.append(rn))
            out[prefix + "pcg_breakdown"] = np.int64(0)
        except ref_linalg.PcgBreakdownError as exc:
            res = exc.result
            out[prefix + "pcg_breakdown"] = np.int64(1)
        out[prefix + "rhs"] = rhs
        out[prefix + "pcg_x"] = res.solution
        out[prefix + "pcg_iters"] = np.int64(res.iterations)
        out[prefix + "pcg_final"] = np.float64(res.final_residual_norm)
        out[prefix + "pcg_conv"] = np.int64(res.converged)
        h = np.array([np.linalg.norm(rhs)] + hist)
        out[prefix + "pcg_hist"] = h if hist_cap is None else h[:hist_cap]


# ----------------------------------------------------------------------------
def make_instances():
    """The 50 seeded QPs of the reference acceptance suite (test_acceptance.py:30-43)
    plus the 8-instance sets of test_kkt.py, with the reference's outputs."""
    out = {}
    rng_vec = np.random.default_rng(424)
    cfg = ref_linalg.PcgConfig(tol=1e-10, max_iters=20000)
    names = []
    for seed in range(50):
        rng = np.random.default_rng(7000 + seed)
        problem = random_problem(rng, n=int(rng.integers(2, 31)), m_a=int(rng.integers(0, 21)),
                                 m_e=int(rng.integers(0, 6)))
        state = random_interior_state(rng, problem)
        names.append(("acc", seed, problem, state))
    rng = np.random.default_rng(20240817)        # conftest.py:5-7 fixture seed
    for k in range(8):
        problem = random_problem(rng)
        state = random_interior_state(rng, problem)
        names.append(("kkt", k, problem, state))
    for hk in ("diagonal", "sparse", "bfgs"):    # one of each Hessian kind, larger
        rng = np.random.default_rng({"diagonal": 11, "sparse": 12, "bfgs": 13}[hk])
        problem = random_problem(rng, n=40, m_a=30, m_e=4, hessian_kind=hk)
        state = random_interior_state(rng, problem)
        names.append(("kind_" + hk, 0, problem, state))
    out["count"] = np.int64(len(names))
    for i, (tag, seed, problem, state) in enumerate(names):
        pre = f"i{i}_"
        out[pre + "tag"] = np.array(f"{tag}:{seed}")
        pack_problem(pre, problem, out)
        pack_state(pre, state, out)
        op = ref_kkt.build_operator(problem, state)
        res = ref_kkt.compute_residuals(problem, state)
        rhs = ref_kkt.assemble_rhs(op, res, state)
        record_operator(pre, op, rng_vec, out, pcg_cfg=cfg, rhs=rhs)
    np.savez_compressed(OUT / "instances.npz", **out)
    print("instances:", len(names))


def make_configs():
    """Scaled-down BASELINE configs (same generators, smaller sizes) with the
    reference's operator outputs and PCG residual histories; cfg1 at full size."""
    out = {}
    specs = {
        "cfg1": dict(fn=workloads.dense_qp, kw=dict(seed=0)),
        "cfg2": dict(fn=workloads.svm_primal, kw=dict(seed=2, d=40, n_samples=1500)),
        "cfg3": dict(fn=workloads.rt_like, kw=dict(seed=3, n_vox=6000, n_beam=600, density=0.02)),
        "cfg5": dict(fn=workloads.random_sweep, kw=dict(seed=5, m=20000, n=5000)),
    }
    rng_vec = np.random.default_rng(99)
    for name, spec in specs.items():
        problem, state, meta = spec["fn"](**spec["kw"])
        rp = to_ref_problem(problem)
        rs = to_ref_state(state)
        op = ref_kkt.build_operator(rp, rs)
        if name == "cfg5":
            rhs = meta["rhs"]
            cfg = ref_linalg.PcgConfig(tol=1e-300, max_iters=200)
        else:
            rhs = ref_kkt.assemble_rhs(op, ref_kkt.compute_residuals(rp, rs), rs)
            cfg = ref_linalg.PcgConfig(tol=1e-7, max_iters=400)
        pre = name + "_"
        out[pre + "kw"] = np.array(repr(spec["kw"]))
        out[pre + "checksum_a"] = np.float64(np.sum(problem.a.values * (1 + np.arange(problem.a.nnz) % 7)))
        t0 = time.perf_counter()
        record_operator(pre, op, rng_vec, out, n_vec=2, pcg_cfg=cfg, rhs=rhs)
        print(name, "dim", op.dim, "pcg iters", int(out[pre + "pcg_iters"]), f"{time.perf_counter() - t0:.1f}s")
    np.savez_compressed(OUT / "configs.npz", **out)


def make_ipm():
    """IPM-level goldens: analytic QPs, random QPs, cfg1 at the pinned tolerances."""
    out = {}
    cases = []
    # test_ipm.py:189-206 / test_acceptance.py:46-58 analytic problems
    cases.append(("active_bound", ref_model.box_qp(ref_model.DiagonalHessian([1.0]), [0.0], [1.0], [10.0]),
                  ref_ipm.IpmConfig(max_iters=100)))
    cases.append(("interior_optimum", ref_model.box_qp(ref_model.DiagonalHessian([1.0]), [-2.0], [0.0], [10.0]),
                  ref_ipm.IpmConfig(max_iters=100)))
    cases.append(("equality", ref_model.QpProblem(
        n=2, hessian=ref_model.DiagonalHessian([1.0, 1.0]), p=[0.0, 0.0],
        a=ref_model.SparseMatrix.empty(0, 2), lin_bounds=ref_model.Bounds.free(0),
        c=ref_model.SparseMatrix.from_coo(1, 2, [0, 0], [0, 1], [1.0, 1.0]),
        b=[1.0], var_bounds=ref_model.Bounds.box([-10.0, -10.0], [10.0, 10.0])), ref_ipm.IpmConfig(max_iters=100)))
    for seed in range(5):                         # test_ipm.py:250-260
        p = random_problem(np.random.default_rng(100 + seed), n=8, m_a=4, m_e=1)
        cases.append((f"random_{seed}", p, ref_ipm.IpmConfig()))
    problem, _, _ = workloads.dense_qp(seed=0)
    cases.append(("cfg1", to_ref_problem(problem),
                  ref_ipm.IpmConfig(mu_tol=1e-8, pcg=ref_linalg.PcgConfig(tol=1e-10))))
    out["names"] = np.array([c[0] for c in cases])
    for name, problem, cfg in cases:
        t0 = time.perf_counter()
        rep = ref_ipm.solve(problem, cfg)
        pre = name + "_"
        if name != "cfg1":
            pack_problem(pre, problem, out)
        out[pre + "cfg"] = np.array([cfg.gamma, cfg.mu_init, cfg.mu_tol, cfg.mu_shrink, cfg.max_iters,
                                     cfg.pcg.tol, cfg.pcg.max_iters, float(cfg.pcg.tol_is_relative)])
        out[pre + "x"] = rep.x
        out[pre + "objective"] = np.float64(rep.objective)
        out[pre + "status"] = np.array(rep.status.value)
        out[pre + "iterations"] = np.int64(rep.iterations)
        out[pre + "cg_iters"] = np.array([t.cg_iters for t in rep.trace], dtype=np.int64)
        out[pre + "primal"] = np.array([t.primal_inf for t in rep.trace])
        out[pre + "dual"] = np.array([t.dual_inf for t in rep.trace])
        out[pre + "mu"] = np.array([t.mu for t in rep.trace])
        print(name, rep.status.value, rep.iterations, f"obj {rep.objective:.12e}", f"{time.perf_counter() - t0:.1f}s")
    np.savez_compressed(OUT / "ipm.npz", **out)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    which = sys.argv[1:] or ["instances", "configs", "ipm"]
    if "instances" in which:
        make_instances()
    if "configs" in which:
        make_configs()
    if "ipm" in which:
        make_ipm()
