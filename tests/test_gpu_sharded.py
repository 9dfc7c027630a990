"""The sharded (NCCL) engine on one GPU: world_size 1 runs every collective of
the multi-GPU slot (grouped all-reduce of [y_top | scalars], all-reduce of
[r'r, r'z], the separate decision kernel) through a real NCCL communicator.
Parity as tests/parity.py, against the golden fixtures / oracle."""

import os
import socket

import numpy as np
import pytest

import golden_io
import parity
from oracle import qp_oracle as orc
from paper_2308_00637_b200 import _native, workloads
from paper_2308_00637_b200.problem import build_operator
from paper_2308_00637_b200.sharded import ShardedKkt

pytestmark = pytest.mark.gpu

CFG = golden_io.load("configs")
SPECS = {
    "cfg2": (workloads.svm_primal, dict(seed=2, d=40, n_samples=1500)),
    "cfg3": (workloads.rt_like, dict(seed=3, n_vox=6000, n_beam=600, density=0.02)),
    "cfg5": (workloads.random_sweep, dict(seed=5, m=20000, n=5000)),
}


@pytest.fixture(scope="module")
def group():
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield None


@pytest.mark.parametrize("mode", [_native.QPK_SCATTER_ATOMIC, _native.QPK_SCATTER_CSC, _native.QPK_SCATTER_DICT,
                                  _native.QPK_SCATTER_PANEL])
@pytest.mark.parametrize("name", sorted(SPECS))
def test_sharded_world1_parity(group, name, mode):
    fn, kw = SPECS[name]
    problem, state, meta = fn(**kw)
    op = build_operator(problem, state)
    pre = name + "_"
    sk = ShardedKkt(problem, op.bmap, device=0, scatter=mode)
    assert sk.ctx.query("world") == 1 and sk.ctx.query("engine") == 1
    sk.set_diagonals(op.d_diag, op.q_diag_extra)
    assert parity.rel_err(sk.jacobi(), CFG[pre + "jacobi"]) <= parity.APPLY_TOL
    for v, y in zip(CFG[pre + "vecs"], CFG[pre + "applies"]):
        assert parity.rel_err(sk.apply(v), y) <= parity.APPLY_TOL
    rhs = CFG[pre + "rhs"]
    cfg = orc.PcgConfig(tol=1e-300, max_iters=200) if name == "cfg5" else orc.PcgConfig(tol=1e-7, max_iters=400)
    x, info, hist = sk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    env = parity.envelope(op, rhs, cfg, CFG[pre + "pcg_hist"])
    ok, msg = parity.check_history(hist, CFG[pre + "pcg_hist"], env)
    assert ok, msg
    if int(CFG[pre + "pcg_conv"]):
        assert info.converged
        assert parity.rel_err(x, CFG[pre + "pcg_x"]) <= 1e-5
    sk.close()


# ------------------------------------------------ one process, several GPUs --
@pytest.mark.parametrize("mode", [_native.QPK_SCATTER_AUTO, _native.QPK_SCATTER_CSC, _native.QPK_SCATTER_DICT])
@pytest.mark.parametrize("name", sorted(SPECS))
def test_multi_device_context_world1(name, mode):
    """qpk_multi (one process driving a device list; include/qpk.h) with a
    one-device list: the row-sharding layer, the NCCL communicator created
    from the device threads and every collective of the sharded slot run on
    the one GPU this box has.  Global vectors in and out, no torch.distributed."""
    from paper_2308_00637_b200.direction import MultiGpuKkt
    fn, kw = SPECS[name]
    problem, state, meta = fn(**kw)
    op = build_operator(problem, state)
    pre = name + "_"
    mk = MultiGpuKkt(problem, op.bmap, devices=[0], scatter=mode)
    assert mk.ctx.query("world") == 1 and mk.ctx.query("engine") == 1
    assert mk.ctx.query("row_lo") == 0 and mk.ctx.query("row_hi") == op.m
    mk.set_diagonals(op.d_diag, op.q_diag_extra)
    assert parity.rel_err(mk.jacobi(), CFG[pre + "jacobi"]) <= parity.APPLY_TOL
    for v, y in zip(CFG[pre + "vecs"], CFG[pre + "applies"]):
        assert parity.rel_err(mk.apply(v), y) <= parity.APPLY_TOL
    rhs = CFG[pre + "rhs"]
    cfg = orc.PcgConfig(tol=1e-300, max_iters=200) if name == "cfg5" else orc.PcgConfig(tol=1e-7, max_iters=400)
    x, info, hist = mk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    ok, msg = parity.check_history(hist, CFG[pre + "pcg_hist"], parity.envelope(op, rhs, cfg, CFG[pre + "pcg_hist"]))
    assert ok, msg
    if int(CFG[pre + "pcg_conv"]):
        assert info.converged and parity.rel_err(x, CFG[pre + "pcg_x"]) <= 1e-5
    # a second problem on the same object (communicator reused, shard rebuilt)
    mk.close()


def test_hook_through_multi_device_layer(monkeypatch):
    """gpu_direction(op, rhs, cfg) with QPK_DEVICES / QPK_MULTI selecting the
    multi-device layer: same PcgResult as the single-GPU operator."""
    from paper_2308_00637_b200 import direction
    from paper_2308_00637_b200.pcg import PcgConfig
    problem, state, meta = workloads.rt_like(seed=3, n_vox=6000, n_beam=600, density=0.02)
    op = build_operator(problem, state)
    rhs = CFG["cfg3_rhs"]
    cfg = PcgConfig(tol=1e-7, max_iters=400)
    direction.set_devices(None)
    single = direction.gpu_direction(op, rhs, cfg)
    monkeypatch.setenv("QPK_MULTI", "1")
    direction.set_devices([0])
    try:
        multi = direction.gpu_direction(op, rhs, cfg)
        assert isinstance(direction.operator_for(op), direction.MultiGpuKkt)
    finally:
        direction.set_devices(None)
    assert multi.converged == single.converged
    assert parity.rel_err(multi.solution, single.solution) <= 1e-6
    assert parity.rel_err(multi.solution, CFG["cfg3_pcg_x"]) <= 1e-5


def test_multi_device_rejects_duplicate_devices():
    with pytest.raises(_native.NativeUnavailable, match="listed twice"):
        _native.MultiContext([0, 0])


# ------------------------------------- N > 1 partition logic, rank by rank --
class EmulatedRank:
    """Rank `rank` of `world` without a communicator (qpk_shard_emulate): its row
    shard of B, its slice of the top block and of the Hessian rows; apply and
    Jacobi return the rank's un-reduced share.  Ranks run one after the other
    on the one GPU; the test sums their shares on the host."""

    def __init__(self, problem, bmap, world, rank, scatter):
        from paper_2308_00637_b200 import sharded
        from paper_2308_00637_b200.direction import GpuKkt, _csr_arrays
        self.n = int(problem.n)
        segs = sharded.b_row_segments(problem, bmap)
        self.lo, self.hi = sharded.partition_rows(sharded.b_row_nnz(segs), world)[rank]
        self.ctx = _native.Context(0)
        self.ctx.call("qpk_shard_emulate", world, rank)
        self.ctx.call("qpk_problem_begin", self.n, 0, self.hi - self.lo, 0)
        base = 0
        for mat, rows, sign in segs:
            count = mat.n_rows if rows is None else len(rows)
            a, b = max(self.lo, base), min(self.hi, base + count)
            if a < b:
                sel = (np.arange(a - base, b - base, dtype=np.int64) if rows is None
                       else np.ascontiguousarray(rows[a - base:b - base]))
                ro, ci, v = _csr_arrays(mat)
                self.ctx.call("qpk_problem_add_rows", int(mat.n_rows), _native.ptr(ro), _native.ptr(ci),
                              _native.ptr(v), _native.ptr(sel), len(sel), float(sign))
            base += count
        GpuKkt._set_hessian(self, problem.hessian)
        self.ctx.call("qpk_problem_finalize", int(scatter))

    def share(self, fn, d_diag, q_extra, v=None):
        d = np.ascontiguousarray(d_diag[self.lo:self.hi])
        q = np.ascontiguousarray(q_extra, dtype=np.float64)
        self.ctx.call("qpk_set_diagonals", _native.ptr(d), _native.ptr(q))
        out = np.empty(self.n + self.hi - self.lo)
        if fn == "jacobi":
            self.ctx.call("qpk_jacobi", _native.ptr(out))
        else:
            vl = np.ascontiguousarray(np.concatenate([v[:self.n], v[self.n + self.lo:self.n + self.hi]]))
            self.ctx.call("qpk_apply", _native.ptr(vl), _native.ptr(out))
        return out


EMU = {
    "rt_tiled_H": (workloads.rt_like, dict(seed=7, n_vox=10000, n_beam=1000, density=0.04), _native.QPK_SCATTER_DICT),
    "rt_csc": (workloads.rt_like, dict(seed=3, n_vox=6000, n_beam=600, density=0.02), _native.QPK_SCATTER_CSC),
    "random_diagH": (workloads.random_sweep, dict(seed=5, m=20000, n=5000), _native.QPK_SCATTER_ATOMIC),
    "svm_panel": (workloads.svm_primal, dict(seed=2, d=40, n_samples=1500), _native.QPK_SCATTER_AUTO),
}


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name", sorted(EMU))
def test_partition_logic_rank_by_rank(name, world):
    """The N > 1 layout on one GPU, one rank at a time: the ranks' shares of K v
    (top block: a sum over ranks, what the all-reduce forms; bottom block: the
    shards side by side) must give the oracle's apply -- every replicated term
    (diag(Q) u, each Hessian row) is owned by exactly one rank -- and the same
    for the Jacobi diagonal (diag(H) + q is added by every rank after the
    reduction, so it is taken out of all shares but one)."""
    fn, kw, mode = EMU[name]
    problem, state, meta = fn(**kw)
    op = build_operator(problem, state)
    rng = np.random.default_rng(41)
    v = rng.standard_normal(op.dim)
    top = np.zeros(op.n)
    bottom = np.zeros(op.m)
    jtop = np.zeros(op.n)
    jbottom = np.zeros(op.m)
    tiled = 0
    for rank in range(world):
        er = EmulatedRank(problem, op.bmap, world, rank, mode)
        assert er.ctx.query("world") == world and er.ctx.query("rank") == rank
        tiled += er.ctx.query("hess_tiled")
        y = er.share("apply", op.d_diag, op.q_diag_extra, v)
        top += y[:op.n]
        bottom[er.lo:er.hi] = y[op.n:]
        j = er.share("jacobi", op.d_diag, op.q_diag_extra)
        jtop += j[:op.n]
        jbottom[er.lo:er.hi] = j[op.n:]
        er.ctx.close()
    if name == "rt_tiled_H":
        assert tiled == world                          # every rank tiles its slice of the Hessian rows
    y_ref = orc.apply_doubly_augmented(op, v)
    assert parity.rel_err(np.concatenate([top, bottom]), y_ref) <= parity.APPLY_TOL
    jac_ref = orc.jacobi_diagonal(op)
    diag_part = orc.hessian_diagonal(problem.hessian) + op.q_diag_extra
    jtop -= (world - 1) * diag_part
    assert np.max(np.abs(np.concatenate([jtop, jbottom]) - jac_ref) / np.abs(jac_ref)) <= 1e-11


@pytest.mark.parametrize("fold", ["1", "0"])
def test_sharded_tile_slot_with_and_without_folded_scalars(monkeypatch, fold):
    """Sharded tile format: [r'r, r'z] ride in the slot's one all-reduce (default;
    the bottom block's share through |r - a y|^2 = r'r - 2a r'y + a^2 y'y), or
    take the second all-reduce + decision kernel (QPK_SHARD_FOLD=0).  Both must
    hold the literal 1e-8 on the first 60 residuals of an RT-like system at 3
    emulated ranks, and agree on the solution."""
    from paper_2308_00637_b200.direction import MultiGpuKkt
    monkeypatch.setenv("QPK_SHARD_FOLD", fold)
    problem, state, meta = workloads.rt_like(seed=7, n_vox=20000, n_beam=2000, density=0.02)
    op = build_operator(problem, state)
    rhs = np.random.default_rng(5).standard_normal(op.dim)
    cfg = orc.PcgConfig(tol=1e-300, max_iters=60)
    ref_hist = []
    ref = orc.pcg_direction(op, rhs, cfg, callback=lambda k, xk, rn: ref_hist.append(rn))
    ref_hist = np.array([np.linalg.norm(rhs)] + ref_hist)
    mk = MultiGpuKkt(problem, op.bmap, devices=[0], scatter=_native.QPK_SCATTER_DICT, emulate_ranks=3)
    mk.set_diagonals(op.d_diag, op.q_diag_extra)
    x, info, hist = mk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    launches = mk.ctx.query("kernel_launches")
    mk.close()
    ok, msg = parity.check_history(hist, ref_hist, parity.envelope(op, rhs, cfg, ref_hist))
    assert ok, msg
    assert parity.rel_err(x, ref.solution) <= 1e-6
    print(f"fold={fold}: max history deviation {np.max(np.abs(hist - ref_hist) / ref_hist):.2e}, launches {launches}")


@pytest.mark.parametrize("ranks", [2, 3])
@pytest.mark.parametrize("mode", [_native.QPK_SCATTER_AUTO, _native.QPK_SCATTER_CSC, _native.QPK_SCATTER_DICT])
@pytest.mark.parametrize("name", sorted(SPECS))
def test_sharded_engine_with_emulated_ranks(name, mode, ranks):
    """The WHOLE N > 1 sharded engine on one GPU (qpk_multi_create_emulated):
    N contexts on device 0, each with its row shard, its slice of the top
    block and of the Hessian rows, driven by N host threads; the slot's
    collectives ([y_top | 4 scalars], [r'r, r'z], ||rhs||^2, the Jacobi
    partial) are mediated by the host (stream sync, barrier, sum in rank
    order), so no kernel of one rank waits on another.  Same gates as the
    single-GPU parity tests."""
    from paper_2308_00637_b200.direction import MultiGpuKkt
    fn, kw = SPECS[name]
    problem, state, meta = fn(**kw)
    op = build_operator(problem, state)
    pre = name + "_"
    mk = MultiGpuKkt(problem, op.bmap, devices=[0], scatter=mode, emulate_ranks=ranks)
    assert mk.ctx.query("world") == ranks and mk.ctx.query("rank", ranks - 1) == ranks - 1
    bounds = [(mk.ctx.query("row_lo", r), mk.ctx.query("row_hi", r)) for r in range(ranks)]
    assert bounds[0][0] == 0 and bounds[-1][1] == op.m and all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
    mk.set_diagonals(op.d_diag, op.q_diag_extra)
    assert parity.rel_err(mk.jacobi(), CFG[pre + "jacobi"]) <= parity.APPLY_TOL
    for v, y in zip(CFG[pre + "vecs"], CFG[pre + "applies"]):
        assert parity.rel_err(mk.apply(v), y) <= parity.APPLY_TOL
    rhs = CFG[pre + "rhs"]
    cfg = orc.PcgConfig(tol=1e-300, max_iters=200) if name == "cfg5" else orc.PcgConfig(tol=1e-7, max_iters=400)
    x, info, hist = mk.pcg(rhs, cfg.tol, cfg.max_iters, True, history=True)
    ok, msg = parity.check_history(hist, CFG[pre + "pcg_hist"], parity.envelope(op, rhs, cfg, CFG[pre + "pcg_hist"]))
    assert ok, msg
    if int(CFG[pre + "pcg_conv"]):
        assert info.converged and parity.rel_err(x, CFG[pre + "pcg_x"]) <= 1e-5
    mk.close()
