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
