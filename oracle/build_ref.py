"""Recipe for oracle/_ref: the UNMODIFIED reference package, made importable.

TEST INFRASTRUCTURE ONLY.  The reference (`qpipm`, pure Python, no build step
of its own) is mounted read-only at /root/reference in the build container and
does not exist on the GPU box.  This recipe places its package directory under
the git-ignored `oracle/_ref/` (never in history; it travels to the GPU box
with the snapshot like a built .so), so that

* tests/test_gpu_reference_hook.py can run the reference's own
  `qpipm.ipm.solve(problem, cfg, direction_solver=gpu_direction)` on the GPU,
* `bench.py --impl reference` and the `cpu_baseline` leg time the reference's
  own `qpipm.linalg.pcg` / `qpipm.kkt` (cpu_baseline.kind = "reference").

Nothing under paper_2308_00637_b200/ imports it.  `__graft_entry__.build()`
calls `ensure()`; on the GPU box (no /root/reference) the prebuilt copy is used.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/src/qpipm")
REF_TESTS = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parent / "_ref"


def ensure(verbose: bool = True) -> bool:
    """Refresh oracle/_ref/qpipm from the mounted reference when it is there.
    Returns True when oracle/_ref/qpipm is importable afterwards."""
    if SRC.is_dir():
        DST.mkdir(parents=True, exist_ok=True)
        target = DST / "qpipm"
        if target.exists():
            shutil.rmtree(target)
        shutil.copytree(SRC, target, ignore=shutil.ignore_patterns("__pycache__"))
        if verbose:
            print(f"oracle/_ref: qpipm placed from {SRC}", flush=True)
    return (DST / "qpipm" / "ipm.py").exists()


def available() -> bool:
    return (DST / "qpipm" / "ipm.py").exists()


def import_qpipm():
    """Import the reference from oracle/_ref (raises ImportError if absent)."""
    if not available():
        raise ImportError("oracle/_ref/qpipm missing: run `python oracle/build_ref.py` where /root/reference exists")
    if str(DST) not in sys.path:
        sys.path.insert(0, str(DST))
    import qpipm  # noqa: F401
    import qpipm.ipm, qpipm.kkt, qpipm.linalg, qpipm.model  # noqa: F401,E401
    return sys.modules["qpipm"]


if __name__ == "__main__":
    ok = ensure()
    print("oracle/_ref available:", ok)
