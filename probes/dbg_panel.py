"""Debug helper: panel-mode PCG on the golden instances, repeated, against CSC."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import golden_io
from paper_2308_00637_b200 import _native
from paper_2308_00637_b200.direction import GpuKkt
INST = golden_io.load("instances")
bad = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    for i in range(int(INST["count"])):
        problem, state, op, pre = golden_io.instance(INST, i)
        out = []
        for mode in (_native.QPK_SCATTER_PANEL, _native.QPK_SCATTER_PANEL):
            gk = GpuKkt(op.problem, op.bmap, scatter=mode)
            gk.set_diagonals(op.d_diag, op.q_diag_extra)
            x, info, hist = gk.pcg(INST[pre + "rhs"], 1e-10, 20000, True, history=True)
            out.append((x, hist, info.converged, info.iterations, gk.ctx.query("panel_ew"), gk.ctx.query("panel_direct"),
                        gk.ctx.query("panel_kp"), gk.ctx.query("scatter")))
            gk.close()
        if not (np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])):
            bad += 1
            k = int(np.argmax(out[0][1][:min(len(out[0][1]), len(out[1][1]))] != out[1][1][:min(len(out[0][1]), len(out[1][1]))]))
            print("rep", rep, "inst", i, "nondeterministic", out[0][2:], out[1][2:], "first hist diff at", k, op.dim, op.m, type(problem.hessian).__name__)
print("done bad", bad)
