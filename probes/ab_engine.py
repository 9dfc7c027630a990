"""A/B timing of libqpk.so build variants on the bench workloads (one process,
each workload generated once).  Usage on the GPU box:

    QPK_ENGINE=1 python probes/ab_engine.py cfg5,cfg3 lib1.so,lib2.so [iters]
"""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2308_00637_b200 import _native  # noqa: E402
from paper_2308_00637_b200.direction import GpuKkt  # noqa: E402


def main():
    names = sys.argv[1].split(",")
    libs = sys.argv[2].split(",")
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    modes = [int(m) for m in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["1", "2"])]
    for name in names:
        t0 = time.time()
        problem, op, rhs, meta = bench.make_workload(name, 1.0)
        print(f"# {name}: generated in {time.time() - t0:.1f}s  N={op.dim}", flush=True)
        for lib in libs:
            _native._lib = None
            _native.load_library(Path(lib))
            for mode in modes:
                gk = GpuKkt(problem, op.bmap, scatter=mode)
                gk.set_diagonals(op.d_diag, op.q_diag_extra)
                info = _native.PcgInfo()
                x = np.empty(op.dim)
                best = None
                for rep in range(3):
                    gk.ctx.call("qpk_pcg", _native.ptr(rhs), 1e-300, 1, iters, _native.ptr(x),
                                _native.ctypes.byref(info), None)
                    t = info.kernel_ms / iters
                    best = t if best is None else min(best, t)
                ph = [round(v * 1e3 / iters, 1) for v in info.phase_ms]
                print(f"{name} {Path(lib).name} scatter={mode} engine={gk.ctx.query('engine')} "
                      f"grid={gk.ctx.query('grid_engine')}: {1e3 / best:.0f} it/s ({best * 1e3:.1f} us/it) "
                      f"phases {ph} iters {info.iterations}", flush=True)
                gk.close()


if __name__ == "__main__":
    main()
