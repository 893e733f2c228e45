"""Guarded trigonometric / hyperbolic Jacobi rotation parameters -- drop-in
for the rotation API of the reference ``jhsvd.rotation``
(pkg/src/jhsvd/rotation.py:48-124).

``compute_rotation`` evaluates the inner kernel's own device function
(``rotation_core`` in ``csrc/jh_common.cuh``: the cs2 formula with the 5/4,
sqrt(eps) and sqrt(2/eps) guards) on the GPU through ``jh_rotations``, so
the parameters are bit for bit the ones the solver applies.
``compute_rotations`` is the batched form.  The departure diagnostics and
the Table B.1 survey (rotation.py:127-244) are out of scope (SURVEY.md
section 2, row 3): they are not on the solve path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

TRIG = "trig"
HYPERBOLIC = "hyp"


class HyperbolicDomainError(ArithmeticError):
    """|coth 2phi| < 1: the pivot pair lost J-definiteness upstream."""


@dataclass(frozen=True)
class PivotGram:
    """Entries of the 2x2 pivot Gram matrix."""

    h_pp: float
    h_qq: float
    h_pq: float


@dataclass(frozen=True)
class RotationParams:
    kind: str            # TRIG or HYPERBOLIC
    cs: float            # cos(phi) or cosh(phi)
    tn: float            # tan(phi) or tanh(phi)
    proper: bool         # cs != 1: the rotation changes column scales
    swap: bool = False   # sorting permutation applied after the rotation


def compute_rotations(h, t):
    """Batched rotation parameters: h (n, 3) rows (h_pp, h_qq, h_pq), t (n,)
    +1 trigonometric / -1 hyperbolic.  Returns (cs, tn, ok) arrays; ok is
    False where a hyperbolic pair has |coth 2phi| < 1."""
    import torch

    lib = _lib.require_cuda()
    hd = torch.as_tensor(np.ascontiguousarray(h, dtype=np.float64).reshape(-1, 3), device="cuda")
    td = torch.as_tensor(np.ascontiguousarray(t, dtype=np.float64).reshape(-1), device="cuda")
    if hd.shape[0] != td.shape[0]:
        raise ValueError("h and t must have the same number of rows")
    out = torch.empty_like(hd)
    _lib.check(lib.jh_rotations(hd.data_ptr(), td.data_ptr(), hd.shape[0], out.data_ptr(),
                                _lib.stream_handle()), "rotations")
    o = out.cpu().numpy()
    return o[:, 0].copy(), o[:, 1].copy(), o[:, 2] != 0.0


def compute_rotation(g: PivotGram, kind: str) -> RotationParams:
    """Rotation parameters diagonalising the 2x2 pivot Gram matrix
    (rotation.py:105-124); h_pq must be nonzero, h_pp and h_qq positive."""
    if not (g.h_pp > 0.0 and g.h_qq > 0.0):
        raise ValueError("pivot Gram diagonal must be positive")
    if g.h_pq == 0.0:
        raise ValueError("h_pq is zero; the pair is already orthogonal")
    if kind not in (TRIG, HYPERBOLIC):
        raise ValueError(f"kind must be {TRIG!r} or {HYPERBOLIC!r}")
    cs, tn, ok = compute_rotations([[g.h_pp, g.h_qq, g.h_pq]], [1.0 if kind == TRIG else -1.0])
    if not ok[0]:
        raise HyperbolicDomainError(
            "hyperbolic pivot with |coth 2phi| < 1; J-definiteness was lost upstream")
    return RotationParams(kind=kind, cs=float(cs[0]), tn=float(tn[0]), proper=bool(cs[0] != 1.0))
