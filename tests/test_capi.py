"""The C-ABI library builds, loads without a GPU and exports every symbol
include/jhsvd_b200.h declares; host-only entry points are checked against
the reference goldens."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1401_2720_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "jhsvd_b200.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void)\s+(jh_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = _declared()
    assert "jh_block_sweep" in names and len(names) >= 10


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1401_2720_b200 as J

    with pytest.raises(J.NativeUnavailable):
        J.block_jacobi(np.eye(4), None, J.SolverConfig(block_width=2))
    with pytest.raises(J.NativeUnavailable):
        J.gram(np.eye(4))


def test_host_safe_bounds_match_reference(kernels_golden):
    lib = _lib.load_library()
    for n in (1, 2, 3, 255, 256, 257, 512, 4096, 16384, 131072, 1 << 20):
        a, b = ctypes.c_double(), ctypes.c_double()
        lib.jh_safe_bounds(n, ctypes.byref(a), ctypes.byref(b))
        assert (a.value, b.value) == tuple(kernels_golden[f"safe_{n}"]), n


def test_workspace_size():
    lib = _lib.load_library()
    assert lib.jh_sweep_workspace_bytes(16384, 32, 0) >= 512 * 32 * 32 * 8 * 2
    assert lib.jh_sweep_workspace_bytes(16384, 30, 0) == -1
