"""Check the packed-symmetric dense-H apply at the svm_dual bench size against
the oracle, and time the solver's apply (GPU box)."""
import sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import qp_oracle as orc, svm_oracle as so
from paper_2308_00637_b200 import svm
from paper_2308_00637_b200.direction import GpuKkt
from paper_2308_00637_b200.problem import build_operator
from paper_2308_00637_b200.workloads import _state_from_initial, svm_dual_data

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
x, y = svm_dual_data(seed=6, n=n, d=100)
cfg = svm.SvmConfig(sigma=100.0, c=1.0)
prob = svm.build_svm_dual(svm.SvmDataset.from_dense(x, y), cfg)
host = so.dual_problem(x, y, cfg.sigma, cfg.c)
op = build_operator(host, _state_from_initial(host))
gk = GpuKkt(prob, op.bmap)
print("hess_sym", gk.ctx.query("hess_sym"), "dense_rows", gk.ctx.query("dense_rows"), "scatter", gk.ctx.query("scatter"))
gk.set_diagonals(op.d_diag, op.q_diag_extra)
v = np.random.default_rng(1).standard_normal(op.dim)
yg = gk.apply(v)
t0 = time.perf_counter(); yr = orc.apply_doubly_augmented(op, v); t1 = time.perf_counter()
print("apply rel err", np.linalg.norm(yg - yr) / np.linalg.norm(yr), f"(oracle apply {t1 - t0:.2f}s)")
jg = gk.jacobi(); jr = orc.jacobi_diagonal(op)
print("jacobi rel err", np.max(np.abs(jg - jr) / jr))
xg, info, hist = gk.pcg(np.random.default_rng(2).standard_normal(op.dim), 1e-300, 100, True)
print("pcg 100 it: kernel ms", info.kernel_ms, "phases ms", list(info.phase_ms))
