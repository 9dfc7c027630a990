"""Debug helper: DICT-mode PCG on one golden instance (tile CTA accumulation on/off via QPK_NO_CACC)."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import golden_io
from paper_2308_00637_b200 import _native
from paper_2308_00637_b200.direction import GpuKkt
INST = golden_io.load("instances")
i = int(sys.argv[1]) if len(sys.argv) > 1 else 4
problem, state, op, pre = golden_io.instance(INST, i)
gk = GpuKkt(op.problem, op.bmap, scatter=_native.QPK_SCATTER_DICT)
gk.set_diagonals(op.d_diag, op.q_diag_extra)
print("cacc", gk.ctx.query("tile_cta_acc"), "blocks", gk.ctx.query("dict_blocks"), "htiled", gk.ctx.query("hess_tiled"))
x, info, hist = gk.pcg(INST[pre + "rhs"], 1e-10, 60, True, history=True)
print("conv", info.converged, info.iterations, info.restarts)
print("gpu", hist[:14])
print("ref", INST[pre + "pcg_hist"][:14])
from oracle import qp_oracle as orc
rhs = INST[pre + "rhs"]
for k in (1, 2):
    x1, info1, _ = gk.pcg(rhs, 1e-300, k, True, history=False)
    ref = orc.pcg_direction(op, rhs, orc.PcgConfig(tol=1e-300, max_iters=k))
    print("iters", k, "x rel err", np.linalg.norm(x1 - ref.solution) / np.linalg.norm(ref.solution))
v = np.random.default_rng(0).standard_normal(op.dim)
print("apply rel err", np.linalg.norm(gk.apply(v) - orc.apply_doubly_augmented(op, v)) / np.linalg.norm(orc.apply_doubly_augmented(op, v)))
jac = gk.jacobi(); rj = orc.jacobi_diagonal(op)
print("jac rel err", np.max(np.abs(jac - rj) / rj))
