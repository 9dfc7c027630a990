"""C-ABI checks that need no GPU: libqpk.so loads, exports exactly the symbols
include/qpk.h declares, and the Python binding declares every one of them."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2308_00637_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "qpk.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qpk_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not _native.LIB_PATH.exists():
        import __graft_entry__
        __graft_entry__.build()
    return _native.load_library()


def test_header_declares_the_binding():
    assert header_functions() == sorted(_native.EXPORTED)


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (qpk_[a-z_0-9]+)", out))
    assert exported == set(header_functions())


def test_abi_version_and_error_channel(lib):
    assert lib.qpk_abi_version() == 1
    assert isinstance(lib.qpk_last_error(), bytes)


def _gpu_visible():
    import torch
    return torch.cuda.is_available()


def test_create_without_gpu_fails_loudly(lib):
    """No CUDA device here: the context must refuse, never fall back to CPU."""
    if _gpu_visible():
        pytest.skip("a GPU is visible")
    with pytest.raises(_native.NativeUnavailable):
        _native.Context(0)


def test_solver_entry_raises_without_gpu(lib):
    if _gpu_visible():
        pytest.skip("a GPU is visible")
    import numpy as np
    from paper_2308_00637_b200 import workloads
    from paper_2308_00637_b200.direction import gpu_direction
    from paper_2308_00637_b200.pcg import PcgConfig
    from paper_2308_00637_b200.problem import build_operator
    problem, state, meta = workloads.random_sweep(seed=1, m=40, n=100)
    op = build_operator(problem, state)
    with pytest.raises(_native.NativeUnavailable):
        gpu_direction(op, np.ones(op.dim), PcgConfig())
