"""The branch-free FP64 division / square root fast paths used in the inner
Jacobi (csrc/jh_fastmath.cuh) must equal the IEEE operators bit for bit
whenever they report themselves in range (probe kernel in the dev-only
library, tools/dev)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(a, b):
    import torch

    from paper_1401_2720_b200 import _lib
    from tools.dev import devlib

    _lib.require_cuda()
    lib = devlib.load()
    ta = torch.as_tensor(a, dtype=torch.float64, device="cuda")
    tb = torch.as_tensor(b, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    _lib.check(lib.jh_probe_fastmath(ta.data_ptr(), tb.data_ptr(), ta.numel(), cnt.data_ptr(),
                                     _lib.stream_handle()), "probe_fastmath")
    return [int(x) for x in cnt.cpu().tolist()]


def test_fast_paths_match_ieee_random_wide_range():
    rng = np.random.default_rng(0)
    n = 1 << 24
    for _ in range(4):
        a = rng.standard_normal(n) * np.exp2(rng.integers(-1000, 1000, n))
        b = rng.standard_normal(n) * np.exp2(rng.integers(-1000, 1000, n))
        c = _run(a, b)
        assert c[0] == 0 and c[2] == 0, c


def test_fast_paths_match_ieee_solver_ranges():
    # operands as they occur in the rotation: moderate exponents, near-equal
    # values, tiny and huge ratios, exact squares
    rng = np.random.default_rng(1)
    n = 1 << 24
    x = rng.random(n) + 0.5
    y = x * (1 + rng.standard_normal(n) * 1e-12)
    cases = [
        (rng.standard_normal(n), rng.standard_normal(n)),
        (x - y, 2.0 * rng.standard_normal(n) * 1e-9),
        (np.ones(n), rng.random(n) * 1e8 + 1.0),
        (np.floor(rng.random(n) * 2 ** 26) ** 2, np.floor(rng.random(n) * 2 ** 26) + 1.0),
        (rng.random(n) * 2 ** 27, rng.random(n) * 2 ** -27 + 2 ** -60),
    ]
    for a, b in cases:
        c = _run(a, b)
        assert c[0] == 0 and c[2] == 0, c


def test_special_values_rejected_not_wrong():
    a = np.array([0.0, -0.0, 1e-310, np.inf, 1.0, 1.0, 5e-324, 1e300, 2.0], dtype=np.float64)
    b = np.array([1.0, 3.0, 2.0, 1.0, 0.0, np.inf, 1.0, 1e-300, 1e-310], dtype=np.float64)
    c = _run(a, b)
    assert c[0] == 0 and c[2] == 0, c
