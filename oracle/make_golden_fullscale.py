"""Full-scale IPM goldens: the REAL reference's solve() on BASELINE configs at
their full sizes (cfg2, cfg3, cfg4), defaults (mu_tol 1e-6, CG tol 1e-7).

TEST INFRASTRUCTURE ONLY.  Run in the build container (needs oracle/_ref,
placed by oracle/build_ref.py from /root/reference); each config takes
10-60 minutes of CPU:

    python oracle/make_golden_fullscale.py cfg3 [cfg2 cfg4]

Writes tests/golden/ipm_full_<cfg>.npz: the reference's x, objective, status,
iteration counts and per-iteration infeasibilities.  tests/test_gpu_fullscale_ipm.py
compares the device IPM and the hook-driven reference loop against them.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import build_ref, refbridge  # noqa: E402
from paper_2308_00637_b200 import workloads  # noqa: E402

SPECS = {
    "cfg2": (workloads.svm_primal, dict(seed=2)),
    "cfg3": (workloads.rt_like, dict(seed=3)),
    "cfg4": (workloads.rt_like, dict(seed=4, n_vox=2_000_000, n_beam=100_000, density=0.001)),
}


def main():
    qp = build_ref.import_qpipm()
    for name in sys.argv[1:]:
        fn, kw = SPECS[name]
        problem, _, meta = fn(**kw)
        rp = refbridge.ref_problem(problem)
        cfg = qp.ipm.IpmConfig()
        t0 = time.perf_counter()
        rep = qp.ipm.solve(rp, cfg, verbose=True)
        dt = time.perf_counter() - t0
        out = {
            "kw": np.array(repr(kw)), "x": rep.x, "objective": np.float64(rep.objective),
            "status": np.array(rep.status.value), "iterations": np.int64(rep.iterations),
            "cg_iters": np.array([t.cg_iters for t in rep.trace], dtype=np.int64),
            "primal": np.array([t.primal_inf for t in rep.trace]),
            "dual": np.array([t.dual_inf for t in rep.trace]),
            "compl": np.array([t.compl_inf for t in rep.trace]),
            "mu": np.array([t.mu for t in rep.trace]),
            "cfg": np.array([cfg.gamma, cfg.mu_init, cfg.mu_tol, cfg.mu_shrink, cfg.max_iters, cfg.pcg.tol,
                             cfg.pcg.max_iters, float(cfg.pcg.tol_is_relative)]),
            "wall_s": np.float64(dt),
        }
        np.savez_compressed(ROOT / "tests" / "golden" / f"ipm_full_{name}.npz", **out)
        print(f"{name}: {rep.status.value} in {rep.iterations} IPM / {int(out['cg_iters'].sum())} CG iterations, "
              f"objective {rep.objective:.13e}, {dt:.0f} s", flush=True)


if __name__ == "__main__":
    main()
