"""Where the e2e gap of gpu_direction goes (host buffers in, host result out):
set_diagonals (H2D of d, q), qpk_pcg (H2D rhs, Jacobi, solve, D2H x) against the
solve's device time.  python probes/e2e_split.py cfg4 [iters]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2308_00637_b200.direction import operator_for  # noqa: E402

name = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
problem, op, rhs, meta = bench.make_workload(name, 1.0)
gk = operator_for(op)
for rep in range(4):
    t0 = time.perf_counter()
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    t1 = time.perf_counter()
    x, info, _ = gk.pcg(rhs, 1e-300, iters, True)
    t2 = time.perf_counter()
    print(f"{name}: set_diagonals {1e3 * (t1 - t0):.2f} ms, pcg call {1e3 * (t2 - t1):.2f} ms "
          f"(device solve {info.kernel_ms:.2f} ms) -> host overhead {1e3 * (t2 - t0) - info.kernel_ms:.2f} ms "
          f"of {1e3 * (t2 - t0):.2f} ms", flush=True)
