"""Robust 2-norms (DRDSSQ, the paper's Appendix A) -- drop-in for the
reference ``jhsvd.robustnorm`` (pkg/src/jhsvd/robustnorm.py).

The sums of squares run on the GPU (``jh_robust_norms``: one CTA per vector,
the reference's leaves of ``chunk`` in-order fma chains combined along its
fixed binary tree, with the power-of-two-scaled three-partition fallback),
so results are bitwise the reference's.  The scalar helpers (common form,
scaled addition, scale exponents, safe bounds) are the library's own host
code, the same source the kernels inline (``csrc/jh_robust.cuh``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

EPS = 2.0 ** -53
MU = 2.0 ** -1022                       # smallest normal (robustnorm.py:34-45)
NU = math.ldexp(2.0 - 2.0 ** -52, 1022)  # half the largest double
GAMMA = 1.0 - EPS
DELTA = 1.0 + EPS
#: elements per reduction-tree leaf; part of the result's definition
DEFAULT_CHUNK = 256


@dataclass(frozen=True)
class FpParams:
    mu: float = MU
    nu: float = NU
    eps: float = EPS
    gamma: float = GAMMA
    delta: float = DELTA


@dataclass(frozen=True)
class ScaledSquare:
    """value * 2**scale_exp; the common form keeps 0.5 <= value < 2 with an
    even scale exponent (zero is (0, 0.0))."""

    scale_exp: int
    value: float

    def to_float(self) -> float:
        return math.ldexp(self.value, self.scale_exp)


ZERO = ScaledSquare(0, 0.0)


def reduction_depth(n: int) -> int:
    """Depth of the fixed reduction tree over n terms (robustnorm.py:72-89)."""
    if n < 1:
        raise ValueError("vector length must be at least 1")
    return max(1, (n - 1).bit_length())


def safe_bounds(n: int) -> tuple[float, float]:
    """Inclusive magnitudes [mu_tilde, nu_hat] whose squares and tree sums of
    n terms can neither underflow nor overflow (robustnorm.py:104-113)."""
    if n < 1:
        raise ValueError("vector length must be at least 1")
    lib = _lib.load_library()
    a, b = ctypes.c_double(), ctypes.c_double()
    lib.jh_safe_bounds(int(n), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def scale_exponent(f: float, t: float, direction: str) -> int:
    """'up': smallest j with 2**j f >= t; 'down': largest j with
    2**j f <= t (robustnorm.py:125-136)."""
    if not (f > 0.0 and t > 0.0 and math.isfinite(f) and math.isfinite(t)):
        raise ValueError("scale_exponent needs positive finite inputs")
    if direction not in ("up", "down"):
        raise ValueError(f"direction must be 'up' or 'down', got {direction!r}")
    return int(_lib.load_library().jh_scale_exponent(f, t, 1 if direction == "up" else 0))


def common_form(s: ScaledSquare) -> ScaledSquare:
    """Exact renormalisation to 0.5 <= value < 2, even exponent
    (robustnorm.py:165-170)."""
    if s.value < 0.0 or not math.isfinite(s.value):
        raise ValueError(f"scaled square value {s.value} is not a finite nonneg real")
    j, v = ctypes.c_int64(), ctypes.c_double()
    _lib.load_library().jh_common_form(int(s.scale_exp), float(s.value), ctypes.byref(j),
                                       ctypes.byref(v))
    return ScaledSquare(j.value, v.value)


def add_scaled(a: ScaledSquare, b: ScaledSquare) -> ScaledSquare:
    """Sum of two common-form scaled squares, the smaller rescaled exactly to
    the larger's scale; not re-normalised (robustnorm.py:173-178)."""
    j, v = ctypes.c_int64(), ctypes.c_double()
    _lib.load_library().jh_add_scaled(int(a.scale_exp), float(a.value), int(b.scale_exp),
                                      float(b.value), ctypes.byref(j), ctypes.byref(v))
    return ScaledSquare(j.value, v.value)


def _as_vector(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 1:
        raise ValueError("expected a one-dimensional vector")
    if not np.all(np.isfinite(x)):
        raise ValueError("input vector contains NaN or infinity")
    return x


def _device_norms(x: np.ndarray, chunk: int, force_scaled: bool):
    import torch

    lib = _lib.require_cuda()
    if chunk < 1:
        raise ValueError("chunk must be positive")
    xd = torch.from_numpy(x).cuda()
    out_j = torch.zeros(2, dtype=torch.int64, device="cuda")
    out_v = torch.zeros(2, dtype=torch.float64, device="cuda")
    _lib.check(lib.jh_robust_norms(xd.data_ptr(), max(x.size, 1), x.size, 1, int(chunk),
                                   1 if force_scaled else 0, out_j.data_ptr(),
                                   out_v.data_ptr(), out_j[1:].data_ptr(), out_v[1:].data_ptr(),
                                   _lib.stream_handle()), "robust_norms")
    j = out_j.cpu().tolist()
    v = out_v.cpu().tolist()
    return int(j[0]), float(v[0]), int(j[1]), float(v[1])


def sum_squares(x, chunk: int = DEFAULT_CHUNK, force_scaled: bool = False) -> ScaledSquare:
    """Sum of squares as a common-form ScaledSquare (robustnorm.py:324-328);
    force_scaled skips the plain fast path."""
    j, v, _, _ = _device_norms(_as_vector(x), chunk, force_scaled)
    return ScaledSquare(j, v)


def norm2(x, chunk: int = DEFAULT_CHUNK, force_scaled: bool = False) -> tuple[int, float]:
    """2-norm as (js, sigma) with ||x|| = sigma / 2**js (robustnorm.py:331-334)."""
    _, _, js, s = _device_norms(_as_vector(x), chunk, force_scaled)
    return js, s


def norm2_value(x, chunk: int = DEFAULT_CHUNK, force_scaled: bool = False) -> float:
    """The 2-norm collapsed to a double (inf if it exceeds the range)."""
    js, sigma = norm2(x, chunk=chunk, force_scaled=force_scaled)
    return math.ldexp(sigma, -js)
