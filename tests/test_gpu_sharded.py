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
