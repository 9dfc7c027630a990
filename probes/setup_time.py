"""Host setup cost of one device operator (the e2e gap of --ipm): workload
generation, build_operator, and GpuKkt construction with the library's own
phase split (QPK_TIMING=1).  python probes/setup_time.py cfg4"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("QPK_TIMING", "1")
import bench  # noqa: E402
from paper_2308_00637_b200.direction import GpuKkt  # noqa: E402

for name in sys.argv[1].split(","):
    t0 = time.time()
    problem, op, rhs, meta = bench.make_workload(name, 1.0)
    t1 = time.time()
    gk = GpuKkt(problem, op.bmap)
    t2 = time.time()
    gk.set_diagonals(op.d_diag, op.q_diag_extra)
    gk.jacobi()
    t3 = time.time()
    print(f"{name}: workload {t1 - t0:.2f} s, GpuKkt {t2 - t1:.2f} s, first diagonals+jacobi {t3 - t2:.2f} s", flush=True)
    gk.close()
