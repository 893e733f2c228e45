"""Block-pair task kernels on the GPU (drop-in for ``jhsvd.blockkernel``).

Reference: ``pkg/src/jhsvd/blockkernel.py``.  Each wrapper accepts host
(numpy, Fortran order preferred) or device (torch CUDA) matrices, runs the
sm_100a kernel through the C ABI and returns the same kind it was given.
Results are bitwise the reference's: every kernel replays the reference's
operation order (see ``csrc/jh_common.cuh``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .strategy import PStrategy, as_table, validate_pstrategy

#: row-chunk height of the reference Gram accumulation (blockkernel.py:27);
#: chunking never reorders a chain, so it only documents the reference.
GRAM_CHUNK = 64
EPS = 2.0 ** -53


class RankDeficiencyError(ArithmeticError):
    """A pivot column (or Cholesky pivot) signalled numerical rank loss
    (blockkernel.py:30-35); ``index`` is 1-based."""

    def __init__(self, message, index):
        super().__init__(message)
        self.index = index


class JDefinitenessError(ArithmeticError):
    """A hyperbolic pivot pair lost J-definiteness (blockkernel.py:38-39)."""


@dataclass(frozen=True)
class Signature:
    """J = diag(I, -I) encoded by the number of +1 entries (blockkernel.py:42-60)."""

    n: int
    n_plus: int

    def __post_init__(self):
        if not (0 <= self.n_plus <= self.n):
            raise ValueError("n_plus must lie in [0, n]")

    def sign(self, column: int) -> int:
        return 1 if column <= self.n_plus else -1

    def as_vector(self) -> np.ndarray:
        j = np.ones(self.n)
        j[self.n_plus:] = -1.0
        return j


@dataclass(frozen=True)
class BlockTaskResult:
    r_out: object
    v_acc: object
    rotations: int
    proper_rotations: int
    inner_sweeps: int


def _torch():
    import torch

    return torch


def gram(gpair):
    """Gram matrix of a tall block-column pair (m x c, m >= c)."""
    from . import _dev

    lib = _lib.require_cuda()
    torch = _torch()
    as_np = not _dev.is_torch(gpair)
    g = _dev.to_colmajor(gpair)
    c, m = g.shape
    if m < c:
        raise ValueError(f"need at least as many rows as columns, got {m}x{c}")
    h = torch.empty((c, c), dtype=torch.float64, device=g.device)
    _lib.check(lib.jh_gram(g.data_ptr(), m, m, c, h.data_ptr(), _lib.stream_handle()), "gram")
    return _dev.from_colmajor(h, as_np)


def cholesky_in_place(h):
    """H = L L^T (forward-looking, lower triangle); returns R = L^T with zero
    strict lower triangle.  The input is not modified."""
    from . import _dev

    lib = _lib.require_cuda()
    torch = _torch()
    as_np = not _dev.is_torch(h)
    hf = _dev.to_colmajor(h, copy=True)
    c = hf.shape[0]
    if hf.shape != (c, c):
        raise ValueError("cholesky needs a square matrix")
    r = torch.empty_like(hf)
    info = torch.zeros(1, dtype=torch.int32, device=hf.device)
    _lib.check(lib.jh_cholesky(hf.data_ptr(), c, r.data_ptr(), info.data_ptr(),
                               _lib.stream_handle()), "cholesky")
    bad = int(info.item())
    if bad:
        raise RankDeficiencyError(
            f"nonpositive Cholesky pivot at index {bad}: "
            "the block-pair is numerically rank deficient", index=bad)
    return _dev.from_colmajor(r, as_np)


def inner_jacobi(r, colmap, signature: Signature, strategy: PStrategy, max_sweeps: int,
                 eps_factor: float = 1.0) -> BlockTaskResult:
    """Orthogonalize the square factor r by pointwise Jacobi rotations
    (blockkernel.py:346-400); tolerance eps * sqrt(order) * eps_factor."""
    from . import _dev

    lib = _lib.require_cuda()
    torch = _torch()
    as_np = not _dev.is_torch(r)
    rt = _dev.to_colmajor(r, copy=True)
    c = rt.shape[0]
    if rt.shape != (c, c):
        raise ValueError("the shortened factor must be square")
    if strategy.n != c:
        raise ValueError(f"strategy order {strategy.n} != factor order {c}")
    bad = validate_pstrategy(strategy)
    if bad:
        raise ValueError("invalid inner strategy: " + bad[0])
    if max_sweeps < 1:
        raise ValueError("max_sweeps must be at least 1")
    colmap = np.asarray(colmap, dtype=np.int64)
    if colmap.shape != (c,):
        raise ValueError("colmap must list one global index per local column")
    if np.any(np.diff(colmap) <= 0):
        raise ValueError("colmap must be strictly increasing (keeps J partitioned)")
    signs = torch.tensor([signature.sign(int(g)) for g in colmap], dtype=torch.int8,
                         device=rt.device)
    steps = torch.from_numpy(np.array(as_table(strategy))).to(rt.device)
    v = torch.empty_like(rt)
    out = torch.zeros(5, dtype=torch.int64, device=rt.device)
    tol_c = EPS * math.sqrt(c) * eps_factor
    _lib.check(lib.jh_inner_jacobi(rt.data_ptr(), v.data_ptr(), c, steps.data_ptr(),
                                   signs.data_ptr(), tol_c, int(max_sweeps), out.data_ptr(),
                                   _lib.stream_handle()), "inner_jacobi")
    rot, proper, sweeps, status, badc = (int(x) for x in out.cpu().tolist())
    if status == 2:
        raise RankDeficiencyError(
            f"zero column norm at local column {badc} (global {int(colmap[badc - 1])})",
            index=badc)
    if status == 3:
        raise JDefinitenessError(f"hyperbolic pivot at local column {badc} has |coth 2phi| < 1")
    return BlockTaskResult(r_out=_dev.from_colmajor(rt, as_np),
                           v_acc=_dev.from_colmajor(v, as_np), rotations=rot,
                           proper_rotations=proper, inner_sweeps=sweeps)


def postmultiply(apair, vacc):
    """apair @ vacc with per-entry in-order fma accumulation
    (blockkernel.py:407-428)."""
    from . import _dev

    lib = _lib.require_cuda()
    torch = _torch()
    as_np = not (_dev.is_torch(apair) or _dev.is_torch(vacc))
    a = _dev.to_colmajor(apair)
    v = _dev.to_colmajor(vacc)
    c, m = a.shape
    if v.shape[1] != c or v.shape[0] != v.shape[1]:
        raise ValueError(f"shape mismatch: {(m, c)} @ {(v.shape[1], v.shape[0])}")
    out = torch.empty_like(a)
    _lib.check(lib.jh_gemm(a.data_ptr(), m, m, c, v.data_ptr(), c, c, out.data_ptr(), m,
                           _lib.stream_handle()), "postmultiply")
    return _dev.from_colmajor(out, as_np)


def qr_peeloff(gpair):
    """Upper-triangular factor of a tall block-column pair by per-chunk
    Householder QRs merged with Givens peel-off stages (blockkernel.py:223-244);
    nonnegative diagonal.  The row count must be a multiple of the column
    count (even, <= 256 on the GPU)."""
    from . import _dev

    lib = _lib.require_cuda()
    torch = _torch()
    as_np = not _dev.is_torch(gpair)
    a = _dev.to_colmajor(gpair)
    c, m = (int(x) for x in a.shape)
    if m % c or m < c:
        raise ValueError(f"row count {m} must be a positive multiple of {c}")
    if c % 2 or c > 256:
        raise NotImplementedError("qr_peeloff runs on the GPU for even widths up to 256")
    r = torch.empty((c, c), dtype=torch.float64, device=a.device)
    _lib.check(lib.jh_qr_peeloff(a.data_ptr(), m, m, c, r.data_ptr(), _lib.stream_handle()),
               "qr_peeloff")
    return _dev.from_colmajor(r, as_np)
