"""Parity at BASELINE scale: the very code paths the bench lines run.

* cfg2-cfg5 built at FULL size (BASELINE.json configs[1..4], the seeds
  bench.py uses): Jacobi and operator apply <= 1e-12 against the oracle
  (kkt.py:211-239), operator symmetry u'Kv = v'Ku, and the first 20 PCG
  residuals (linalg.py:99-130) within the north star's literal 1e-8 of the
  oracle's -- no reorder envelope is needed this early in a solve.
* long per-CTA tile streams on a small problem (QPK_TILE_GRID caps the tile
  grid): ring-stage reuse, the descriptor batch refill (from 32 tiles per CTA)
  and the L2 prefetch (from 128 tiles per CTA) under parity assertions.
* the explicit-residual restart branch (linalg.py:112-125): a case where the
  recurrence residual passes the threshold and the true residual does not.
"""

import os

import numpy as np
import pytest

import parity
from oracle import qp_oracle as orc
from paper_2308_00637_b200 import _native, workloads
from paper_2308_00637_b200.direction import GpuKkt
from paper_2308_00637_b200.problem import build_operator

pytestmark = pytest.mark.gpu

FULL = {
    "cfg2": (workloads.svm_primal, dict(seed=2), _native.QPK_SCATTER_PANEL),
    "cfg3": (workloads.rt_like, dict(seed=3), _native.QPK_SCATTER_DICT),
    "cfg4": (workloads.rt_like, dict(seed=4, n_vox=2_000_000, n_beam=100_000, density=0.001),
             _native.QPK_SCATTER_DICT),
    "cfg5": (workloads.random_sweep, dict(seed=5), _native.QPK_SCATTER_ATOMIC),
}


def oracle_history(op, rhs, cfg):
    hist = []
    res = orc.pcg_direction(op, rhs, cfg, callback=lambda k, xk, rn: hist.append(rn))
    return res, np.array([np.linalg.norm(rhs)] + hist)


@pytest.mark.slow
@pytest.mark.parametrize("name", sorted(FULL))
def test_full_scale_apply_jacobi_history(name):
    fn, kw, want_mode = FULL[name]
    problem, state, meta = fn(**kw)
    op = build_operator(problem, state)
    gk = GpuKkt(problem, op.bmap)                       # AUTO: the format the bench runs
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    assert gk.ctx.query("scatter") == want_mode
    if name == "cfg4":
        assert gk.ctx.query("hess_tiled") == 1
        assert gk.ctx.query("dict_blocks") // gk.ctx.query("tile_grid") >= 128
    rng = np.random.default_rng(77)
    jac, ref_jac = gk.jacobi(), orc.jacobi_diagonal(op)
    assert np.max(np.abs(jac - ref_jac) / np.abs(ref_jac)) <= parity.APPLY_TOL
    u, v = rng.standard_normal(op.dim), rng.standard_normal(op.dim)
    ku, kv = gk.apply(u), gk.apply(v)
    assert parity.rel_err(ku, orc.apply_doubly_augmented(op, u)) <= parity.APPLY_TOL
    assert parity.rel_err(kv, orc.apply_doubly_augmented(op, v)) <= parity.APPLY_TOL
    # size-independent property: K is symmetric
    assert abs(v @ ku - u @ kv) <= 1e-11 * np.linalg.norm(v) * np.linalg.norm(ku)
    rhs = meta["rhs"] if "rhs" in meta else rng.standard_normal(op.dim)
    cfg = orc.PcgConfig(tol=1e-300, max_iters=20)
    ref, ref_hist = oracle_history(op, rhs, cfg)
    x, info, hist = gk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    assert info.iterations == ref.iterations == 20 and info.applies == 21
    dev = np.max(np.abs(hist - ref_hist) / ref_hist)
    assert dev <= parity.HIST_TOL, f"{name}: residual history deviates by {dev:.3e}"
    assert parity.rel_err(x, ref.solution) <= 1e-8
    assert abs(info.final_residual_norm - ref.final_residual_norm) <= 1e-8 * ref.final_residual_norm
    print(f"{name}: apply {parity.rel_err(ku, orc.apply_doubly_augmented(op, u)):.2e}, history dev {dev:.2e}")
    gk.close()


@pytest.mark.parametrize("grid,l2pf", [(2, 3), (3, 0), (3, 3)])
def test_long_tile_streams(monkeypatch, grid, l2pf):
    """~170-250 tiles per CTA on a 40k-voxel problem (cfg4 runs ~380): every ring
    stage is reused dozens of times (mbarrier parity wait) and the producer
    refills its descriptor batch; with and without the optional L2 prefetch
    beyond the ring (QPK_TILE_L2PF)."""
    monkeypatch.setenv("QPK_TILE_GRID", str(grid))
    monkeypatch.setenv("QPK_TILE_L2PF", str(l2pf))
    problem, state, meta = workloads.rt_like(seed=9, n_vox=40_000, n_beam=1000, density=0.02)
    op = build_operator(problem, state)
    gk = GpuKkt(problem, op.bmap, scatter=_native.QPK_SCATTER_DICT)
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    assert gk.ctx.query("scatter") == _native.QPK_SCATTER_DICT and gk.ctx.query("tile_cta_acc") == 1
    assert gk.ctx.query("tile_grid") == grid
    per_cta = gk.ctx.query("dict_blocks") // grid
    assert per_cta >= 128 and gk.ctx.query("tile_l2pf") == l2pf, per_cta
    assert parity.rel_err(gk.jacobi(), orc.jacobi_diagonal(op)) <= parity.APPLY_TOL
    rng = np.random.default_rng(13)
    for _ in range(3):
        v = rng.standard_normal(op.dim)
        assert parity.rel_err(gk.apply(v), orc.apply_doubly_augmented(op, v)) <= parity.APPLY_TOL
    rhs = rng.standard_normal(op.dim)
    cfg = orc.PcgConfig(tol=1e-300, max_iters=60)
    ref, ref_hist = oracle_history(op, rhs, cfg)
    x, info, hist = gk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    ok, msg = parity.check_history(hist, ref_hist, parity.envelope(op, rhs, cfg, ref_hist))
    assert ok, msg
    x2, _, hist2 = gk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    np.testing.assert_array_equal(x, x2)
    np.testing.assert_array_equal(hist, hist2)
    gk.close()


@pytest.mark.parametrize("mode", [_native.QPK_SCATTER_AUTO, _native.QPK_SCATTER_ATOMIC, _native.QPK_SCATTER_CSC,
                                  _native.QPK_SCATTER_DICT])
def test_restart_branch(mode, monkeypatch):
    """linalg.py:112-125: with tol 1e-15 the recurrence residual reaches the
    threshold while the true residual has not; the solver must re-check with
    an extra apply, restart the direction from the true residual and go on.
    The oracle takes 98 iterations with 14 extra applies on this instance."""
    problem, state, meta = workloads.random_sweep(seed=8, m=3000, n=800, log10_w_spread=0)
    op = build_operator(problem, state)
    rhs = meta["rhs"]
    cfg = orc.PcgConfig(tol=1e-15, max_iters=5000)
    applies = [0]
    inv = 1.0 / orc.jacobi_diagonal(op)

    def counted(v):
        applies[0] += 1
        return orc.apply_doubly_augmented(op, v)

    ref = orc.pcg(counted, lambda r: inv * r, rhs, cfg)
    ref_restarts = applies[0] - ref.iterations - 1           # final check converged: no extra final apply
    assert ref.converged and ref_restarts > 0
    variants = {"cluster": {"QPK_ENGINE": "0"}, "persistent": {"QPK_ENGINE": "0", "QPK_NO_CLUSTER": "1"},
                "engine": {"QPK_ENGINE": "1"}}
    for engine, env in variants.items():
        monkeypatch.delenv("QPK_NO_CLUSTER", raising=False)
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        gk = GpuKkt(problem, op.bmap, scatter=mode)
        gk.set_diagonals(op.d_diag, op.q_diag_extra)
        x, info, hist = gk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
        assert info.restarts > 0, (engine, info.restarts)
        assert info.converged and info.status == _native.QPK_PCG_OK
        true_r = np.linalg.norm(rhs - orc.apply_doubly_augmented(op, x))
        assert true_r <= 1.5 * info.threshold, (true_r, info.threshold)
        assert info.final_residual_norm <= info.threshold
        assert parity.rel_err(x, ref.solution) <= 1e-6
        assert info.applies == info.iterations + info.restarts + 1
        print(f"mode {mode} engine {engine}: {info.iterations} iterations, {info.restarts} restarts "
              f"(oracle {ref.iterations}, {ref_restarts})")
        gk.close()


@pytest.mark.slow
@pytest.mark.parametrize("mode", [_native.QPK_SCATTER_AUTO, _native.QPK_SCATTER_DICT])
def test_full_scale_cfg3_eight_emulated_ranks(mode):
    """cfg3 at full size through the N = 8 sharded engine on one GPU
    (qpk_multi_create_emulated: host-mediated collectives, no kernel waits on a
    peer): every rank tiles its row shard and its slice of the Hessian rows;
    apply, Jacobi and the first 20 residuals against the oracle."""
    from paper_2308_00637_b200.direction import MultiGpuKkt
    problem, state, meta = workloads.rt_like(seed=3)
    op = build_operator(problem, state)
    mk = MultiGpuKkt(problem, op.bmap, devices=[0], scatter=mode, emulate_ranks=8)
    fmt = [(mk.ctx.query("scatter", r), mk.ctx.query("hess_tiled", r)) for r in range(8)]
    print("per-rank (format, Hessian tiles):", fmt)
    # (AUTO decides per rank: a 1/8 shard of cfg3 is below the tile format's size threshold -> CSC)
    if mode == _native.QPK_SCATTER_DICT:
        assert all(f == (_native.QPK_SCATTER_DICT, 1) for f in fmt)
    mk.set_diagonals(op.d_diag, op.q_diag_extra)
    rng = np.random.default_rng(77)
    jac, ref_jac = mk.jacobi(), orc.jacobi_diagonal(op)
    assert np.max(np.abs(jac - ref_jac) / np.abs(ref_jac)) <= parity.APPLY_TOL
    v = rng.standard_normal(op.dim)
    assert parity.rel_err(mk.apply(v), orc.apply_doubly_augmented(op, v)) <= parity.APPLY_TOL
    rhs = rng.standard_normal(op.dim)
    cfg = orc.PcgConfig(tol=1e-300, max_iters=20)
    ref, ref_hist = oracle_history(op, rhs, cfg)
    x, info, hist = mk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    assert info.iterations == 20
    dev = np.max(np.abs(hist - ref_hist) / ref_hist)
    assert dev <= parity.HIST_TOL, dev
    assert parity.rel_err(x, ref.solution) <= 1e-8
    mk.close()
