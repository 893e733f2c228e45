"""Single-GPU two-level blocked one-sided Jacobi (H)SVD (drop-in for ``jhsvd.driver``).

Reference: ``pkg/src/jhsvd/driver.py``.  The matrix is split into
b = n / (w/2) block-columns; every p-step of the outer strategy pairs them
off into b/2 independent tasks (shorten, pointwise Jacobi, post-multiply),
here executed by the fused sm_100a kernels of ``csrc/jh_pstep.cu`` (one
``jh_block_sweep`` call enqueues a whole block sweep).  The host reads back
one pair of counters per sweep and stops after a sweep without proper
rotations, or at the sweep limit, exactly like the reference.  Results are
bitwise those of the reference for the same inputs.

Data stay on the device: G (m x n) and V (n x n) are column-major FP64
torch tensors; host numpy inputs are uploaded once and results copied back
once.  ``workers`` is accepted for API compatibility and ignored (the GPU is
the parallelism; the reference's results do not depend on it either).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _dev, _lib
from .blockkernel import (
    EPS,
    JDefinitenessError,
    RankDeficiencyError,
    Signature,
)
from .strategy import PStrategy, as_table, make_strategy

FULL_BLOCK = "full-block"
BLOCK_ORIENTED = "block-oriented"
VARIANTS = (FULL_BLOCK, BLOCK_ORIENTED)
SHORTENINGS = ("cholesky", "qr")
# widths above 64 run the general-purpose per-task path (jh_pstep.cu sweep_wide)
MAX_GPU_BLOCK_WIDTH = 8190


class UnsafeScalingError(ValueError):
    """Column norms outside the safe range; rescale the input first
    (driver.py:42-43)."""


@dataclass(frozen=True)
class SolverConfig:
    """Solver knobs, identical to the reference's (driver.py:46-80)."""

    block_width: int = 32
    variant: str = FULL_BLOCK
    max_block_sweeps: int = 30
    max_inner_sweeps: int = 30
    outer_strategy: str = "rrow"
    inner_strategy: str = "rrow"
    accumulate_v: bool = True
    solve_v: bool = False
    shortening: str = "cholesky"
    eps_factor: float = 1.0

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}")
        if self.shortening not in SHORTENINGS:
            raise ValueError(f"shortening must be one of {SHORTENINGS}")
        if self.block_width < 2 or self.block_width % 2:
            raise ValueError("block_width must be an even number >= 2")
        if self.max_block_sweeps < 1 or self.max_inner_sweeps < 1:
            raise ValueError("sweep limits must be at least 1")

    @property
    def inner_sweep_limit(self) -> int:
        return 1 if self.variant == BLOCK_ORIENTED else self.max_inner_sweeps


@dataclass(frozen=True)
class HsvdResult:
    sigma: object
    u: object
    v: object
    signature: Signature
    stats: tuple
    block_sweeps: int
    converged: bool

    @property
    def eigenvalues(self):
        """sigma_i**2 * j_i, the implicit eigenvalues of G J G^T."""
        jv = self.signature.as_vector()
        if _dev.is_torch(self.sigma):
            import torch

            return self.sigma ** 2 * torch.as_tensor(jv, device=self.sigma.device)
        return self.sigma ** 2 * jv


# ---------------------------------------------------------------------------
# device plumbing


class SweepEngine:
    """Device-resident state for repeated block sweeps of one problem shape:
    pivot tables, task workspace and the per-sweep counters."""

    def __init__(self, m: int, n: int, nv: int, cfg: SolverConfig,
                 outer: PStrategy, inner: PStrategy, n_plus: int,
                 engine: Optional[int] = None, outer_table=None, gblock=None):
        """``engine`` (bitwise equal, see jh_block_sweep): 0 per-p-step
        kernels, 1 per-p-step Gram / inner kernels with the V update paired
        over two p-steps and mixed into the G update launch (default when V
        is accumulated and the pivot table pairs block-columns in 4-cycles,
        e.g. rrow; engine 0 otherwise).  ``outer_table`` (int32[steps][b/2][2],
        0-based) replaces the strategy's table (sharded solves run local
        sub-tables); ``gblock`` maps local block-columns to global ones for
        the J signature."""
        import torch

        self.lib = _lib.require_cuda()
        dev = _dev.device()
        w = cfg.block_width
        if w > MAX_GPU_BLOCK_WIDTH:
            raise ValueError(f"block_width {w} > {MAX_GPU_BLOCK_WIDTH} is not supported on the GPU")
        if cfg.shortening == "qr" and (w not in (16, 32, 64) or m % w):
            raise NotImplementedError(
                "QR peel-off shortening runs on the GPU for block widths 16, 32 and 64 "
                "with m a multiple of the width")
        self.shortening = 1 if cfg.shortening == "qr" else 0
        self.m, self.n, self.nv, self.w = m, n, nv, w
        self.cfg = cfg
        self.outer = outer
        self.n_plus = int(n_plus)
        table = np.array(as_table(outer) if outer_table is None else outer_table,
                         dtype=np.int32, order="C")
        self.table = table
        self.outer_dev = torch.from_numpy(table).to(dev)
        self.inner_dev = torch.from_numpy(np.array(as_table(inner))).to(dev)
        self.nsteps = int(table.shape[0])
        self.tasks = int(table.shape[1])  # pairs per p-step
        self._last_rot = self._last_proper = 0
        self.gblock_dev = (torch.from_numpy(np.ascontiguousarray(gblock, dtype=np.int32)).to(dev)
                           if gblock is not None else None)
        if engine is None or nv == 0:
            engine = 1 if nv > 0 else 0
        self.plan_dev = self._cycle_plan(table) if engine == 1 else None
        self.engine = engine if self.plan_dev is not None else 0
        nbytes = int(self.lib.jh_sweep_workspace_bytes(n, w, self.nsteps))
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.counters = torch.empty(4, dtype=torch.int64, device=dev)
        self.tasks_rotated: list[int] = []
        self.tol_c = EPS * math.sqrt(w) * cfg.eps_factor

    def _cycle_plan(self, table: np.ndarray):
        """Device copy of the 4-cycle plan of the pivot table (None when the
        table lacks the structure or the width is not 32)."""
        import torch

        b = 2 * table.shape[1]
        nints = int(self.lib.jh_cycle_plan_ints(b, table.shape[0])) if self.w == 32 else 0
        if nints <= 0:
            return None
        plan = np.empty(nints, dtype=np.int32)
        if self.lib.jh_cycle_plan(table.ctypes.data, b, table.shape[0], plan.ctypes.data) != 0:
            return None
        return torch.from_numpy(plan).to(_dev.device())

    def sweep(self, G, V, first_step: int = 0, nsteps: Optional[int] = None,
              n_plus: Optional[int] = None, counters=None):
        """Enqueue p-steps [first_step, first_step + nsteps) of the pivot table
        on G (n, m) / V (n, nv) column-major tensors; returns the device
        counter tensor (rotations, proper, error key, tasks rotated).
        ``n_plus`` overrides the signature's +1 count; ``counters`` (int64[4],
        initialised by the caller) accumulates instead of this engine's own."""
        if counters is None:
            counters = self.counters
            counters.zero_()
            counters[2].fill_(-1)
        ns = self.nsteps - first_step if nsteps is None else nsteps
        rc = self.lib.jh_block_sweep(
            G.data_ptr(), self.m, self.m, self.n,
            V.data_ptr() if V is not None else None, self.nv, self.nv,
            self.w, self.outer_dev.data_ptr(), self.nsteps,
            self.plan_dev.data_ptr() if self.plan_dev is not None else None,
            self.gblock_dev.data_ptr() if self.gblock_dev is not None else None,
            self.engine, self.shortening, int(first_step), int(ns),
            self.inner_dev.data_ptr(), self.n_plus if n_plus is None else int(n_plus),
            self.cfg.inner_sweep_limit, self.tol_c,
            self.ws.data_ptr(), self.ws.numel(), counters.data_ptr(),
            _lib.stream_handle())
        _lib.check(rc, "jh_block_sweep")
        return counters

    def raise_error(self, key: int) -> None:
        key &= (1 << 64) - 1
        pstep, task = key >> 38, (key >> 16) & 0x3FFFFF
        status, index = (key >> 13) & 7, key & 0x1FFF
        bw = self.w // 2
        p, q = (int(x) for x in self.table[pstep, task])
        gcol = (p * bw + index) if index <= bw else (q * bw + index - bw)
        if status == 1:
            raise RankDeficiencyError(
                f"nonpositive Cholesky pivot at index {index}: "
                "the block-pair is numerically rank deficient", index=index)
        if status == 2:
            raise RankDeficiencyError(
                f"zero column norm at local column {index} (global {gcol})", index=index)
        raise JDefinitenessError(
            f"hyperbolic pivot at local column {index} has |coth 2phi| < 1")

    def one_sweep(self, G, V, n_plus: Optional[int] = None) -> tuple[int, int]:
        """One block sweep; returns (rotations, proper) and raises like the
        reference on numerical failure.  Late sweeps (after a sweep in which
        fewer than half the tasks rotated, or fewer than a tenth of the
        rotations were proper) run engine 0 even where engine 1 applies: with
        few rotating tasks the per-p-step update beats pairing V over two
        p-steps (config 3, sweeps 8-10: 974 / 724 / 645 vs 992 / 786 / 708
        ms, profiles/r02/README.md).  Both engines give the same bits."""
        late = bool(self.tasks_rotated) and (
            self.tasks_rotated[-1] < 0.5 * self.nsteps * self.tasks
            or self._last_proper < 0.1 * self._last_rot)
        engine = self.engine
        if late and engine == 1:
            self.engine = 0
        try:
            out = self.sweep(G, V, n_plus=n_plus)
        finally:
            self.engine = engine
        rot, proper, key, nrot = (int(x) for x in out.cpu().tolist())
        if key != -1:
            self.raise_error(key)
        self.tasks_rotated.append(nrot)
        self._last_rot, self._last_proper = rot, proper
        return rot, proper

    def run(self, G, V, early_stop: Optional[Callable[[], bool]] = None,
            n_plus: Optional[int] = None):
        """Sweep loop of run_block_jacobi_inplace (driver.py:176-200)."""
        stats: list[tuple[int, int]] = []
        converged = False
        self.tasks_rotated: list[int] = []
        for _ in range(self.cfg.max_block_sweeps):
            rot, proper = self.one_sweep(G, V, n_plus)
            stats.append((rot, proper))
            if proper == 0:
                converged = True
                break
            if early_stop is not None and early_stop():
                break
        return stats, converged


def _check_blocking(m: int, n: int, w: int, allow_tall: bool) -> None:
    if m != n and not (allow_tall and m > n):
        raise ValueError("the working factor must be square")
    if n % w or n < w:
        raise ValueError(f"order {n} must be a positive multiple of block_width {w}")


def run_block_jacobi_inplace(g, v, signature: Signature, cfg: SolverConfig, workers: int = 1,
                             outer: Optional[PStrategy] = None,
                             inner: Optional[PStrategy] = None,
                             early_stop: Optional[Callable[[], bool]] = None,
                             *, allow_tall: bool = False):
    """Sweep loop of the blocked Jacobi (driver.py:125-200); g (and v, when
    given) are updated in place.  Returns (per-sweep stats, converged).

    Device tensors that are column-major (``g.t().is_contiguous()``) are
    updated in place on the device; numpy arrays are uploaded, processed and
    written back."""
    m, n = (int(s) for s in g.shape)
    w = cfg.block_width
    _check_blocking(m, n, w, allow_tall)
    b = n // (w // 2)
    if outer is None:
        outer = make_strategy(cfg.outer_strategy, b)
    if inner is None:
        inner = make_strategy(cfg.inner_strategy, w)
    if outer.n != b or inner.n != w:
        raise ValueError("strategy orders do not match the blocking")
    _lib.require_cuda()
    Gd = _dev.to_colmajor(g)
    Vd = _dev.to_colmajor(v) if v is not None else None
    nv = int(Vd.shape[1]) if Vd is not None else 0
    eng = SweepEngine(m, n, nv, cfg, outer, inner, signature.n_plus)
    stats, converged = eng.run(Gd, Vd, early_stop)
    _write_back(g, Gd)
    if v is not None:
        _write_back(v, Vd)
    return stats, converged


def _write_back(orig, dev_t) -> None:
    if _dev.is_torch(orig):
        if orig.t().data_ptr() != dev_t.data_ptr() or not orig.t().is_contiguous():
            orig.copy_(dev_t.t())
    else:
        orig[...] = dev_t.cpu().numpy().T


def solve_for_v(r, w):
    """Solve the upper-triangular system R V = W column by column
    (driver.py:214-227)."""
    import torch

    lib = _lib.require_cuda()
    as_np = not (_dev.is_torch(r) or _dev.is_torch(w))
    rt = _dev.to_colmajor(r)
    wt = _dev.to_colmajor(w)
    n = rt.shape[0]
    if rt.shape != (n, n) or wt.shape[1] != n:
        raise ValueError("shape mismatch in triangular solve")
    diag = torch.diagonal(rt)
    zero = torch.nonzero(diag == 0.0)
    if zero.numel():
        raise ZeroDivisionError(f"zero diagonal entry at index {int(zero[0, 0]) + 1}")
    out = torch.empty_like(wt)
    _lib.check(lib.jh_back_substitute(rt.data_ptr(), n, wt.data_ptr(), wt.shape[0],
                                      out.data_ptr(), _lib.stream_handle()), "solve_for_v")
    return _dev.from_colmajor(out, as_np)


def _safe_bounds(n: int) -> tuple[float, float]:
    import ctypes

    lib = _lib.load_library()
    a, b = ctypes.c_double(), ctypes.c_double()
    lib.jh_safe_bounds(n, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def _check_scaling_dev(G, m: int, n: int) -> None:
    import torch

    lib = _lib.require_cuda()
    bad = torch.full((1,), -1, dtype=torch.int64, device=G.device)
    _lib.check(lib.jh_check_scaling(G.data_ptr(), m, m, n, bad.data_ptr(),
                                    _lib.stream_handle()), "check_column_scaling")
    col = int(bad.item())
    if col != -1:
        mu_tilde, nu_hat = _safe_bounds(m)
        js = torch.zeros(1, dtype=torch.int64, device=G.device)
        s = torch.zeros(1, dtype=torch.float64, device=G.device)
        lib.jh_column_norms(G[col - 1].data_ptr(), m, m, 1, js.data_ptr(), s.data_ptr(),
                            _lib.stream_handle())
        sv = float(s.item())
        nrm = math.ldexp(sv, -int(js.item())) if sv else 0.0
        raise UnsafeScalingError(
            f"column {col} has norm {nrm:.3e} outside the safe range "
            f"[{mu_tilde:.3e}, {math.sqrt(nu_hat):.3e}]; rescale the input factor")


def check_column_scaling(g) -> None:
    """Reject factors whose column norms could over- or underflow the Gram
    formation (driver.py:99-112)."""
    G = _dev.to_colmajor(g)
    _check_scaling_dev(G, int(G.shape[1]), int(G.shape[0]))


def _sigma_u_dev(G, m: int, n: int):
    import torch

    lib = _lib.require_cuda()
    sigma = torch.empty(n, dtype=torch.float64, device=G.device)
    U = torch.empty_like(G)
    bad = torch.full((1,), -1, dtype=torch.int64, device=G.device)
    _lib.check(lib.jh_sigma_u(G.data_ptr(), m, m, n, sigma.data_ptr(), U.data_ptr(), m,
                              bad.data_ptr(), _lib.stream_handle()), "extract_sigma")
    col = int(bad.item())
    if col != -1:
        raise RankDeficiencyError(f"column {col} of the factor is zero", col)
    return sigma, U


def extract_sigma(g):
    """Robust column norms of the transformed factor (driver.py:230-238)."""
    as_np = not _dev.is_torch(g)
    G = _dev.to_colmajor(g)
    sigma, _ = _sigma_u_dev(G, int(G.shape[1]), int(G.shape[0]))
    return _dev.vector_out(sigma, as_np)


def _class_sort_order(sigma, n_plus: int):
    """Non-increasing within the + class, then within the - class
    (driver.py:241-248); stable like numpy's argsort(kind='stable')."""
    import torch

    n = sigma.shape[0]
    idx = torch.arange(n, device=sigma.device)
    parts = []
    for lo, hi in ((0, n_plus), (n_plus, n)):
        if hi > lo:
            _, o = torch.sort(-sigma[lo:hi], stable=True)
            parts.append(idx[lo:hi][o])
    return torch.cat(parts) if parts else idx


class Solver:
    """Reusable single-GPU solver for one problem shape (keeps the pivot
    tables and workspace on the device between calls)."""

    def __init__(self, n: int, cfg: SolverConfig = SolverConfig(),
                 signature: Optional[Signature] = None, m: Optional[int] = None):
        self.m = n if m is None else m
        self.n = n
        self.cfg = cfg
        self.signature = signature if signature is not None else Signature(n, n)
        if self.signature.n != n:
            raise ValueError("signature order does not match the matrix")
        _check_blocking(self.m, n, cfg.block_width, allow_tall=True)
        b = n // (cfg.block_width // 2)
        outer = make_strategy(cfg.outer_strategy, b)
        inner = make_strategy(cfg.inner_strategy, cfg.block_width)
        nv = n if (cfg.accumulate_v and not cfg.solve_v) else 0
        self.engine = SweepEngine(self.m, n, nv, cfg, outer, inner, self.signature.n_plus)

    def solve_device(self, G0):
        """Solve on a device factor G0 given as an (n, m) column-major tensor
        (not modified).  Returns device (sigma, U (n, m), V (n, n) | None,
        stats, converged), all sorted per class like the reference."""
        import torch

        m, n, cfg = self.m, self.n, self.cfg
        if not bool(torch.isfinite(G0).all()):
            raise ValueError("the input factor contains NaN or infinity")
        _check_scaling_dev(G0, m, n)
        work = G0.clone()
        keep = None
        if cfg.solve_v:
            if m != n:
                raise ValueError("solving for V needs a square upper-triangular factor")
            # G0 rows are columns of g: g lower part nonzero <=> triu(G0, 1) != 0
            if bool(torch.triu(G0, 1).ne(0).any()):
                raise ValueError("solving for V needs an upper-triangular input factor; "
                                 "accumulate V instead")
            keep = G0
        V = torch.eye(n, dtype=torch.float64, device=G0.device) if cfg.accumulate_v else None
        # with solve_v the accumulated V would be discarded: do not form it
        stats, converged = self.engine.run(work, V if self.engine.nv else None)
        if cfg.solve_v:
            V = torch.empty((n, n), dtype=torch.float64, device=G0.device)
            lib = _lib.require_cuda()
            _lib.check(lib.jh_back_substitute(keep.data_ptr(), n, work.data_ptr(), n,
                                              V.data_ptr(), _lib.stream_handle()),
                       "solve_for_v")
        sigma, U = _sigma_u_dev(work, m, n)
        order = _class_sort_order(sigma, self.signature.n_plus)
        sigma = sigma[order]
        U = U.index_select(0, order)
        if V is not None:
            V = V.index_select(0, order)
        return sigma, U, V, stats, converged


def block_jacobi(g, signature: Optional[Signature] = None, cfg: SolverConfig = SolverConfig(),
                 workers: int = 1, *, allow_tall: bool = False) -> HsvdResult:
    """Blocked one-sided Jacobi (H)SVD of a square full-rank factor
    (driver.py:251-313).  Singular values come sorted non-increasingly
    inside each signature class (+ class first) with U and V permuted
    consistently; g = U diag(sigma) V^T for J = I.

    Host numpy input -> numpy outputs; CUDA tensor input -> CUDA tensor
    outputs; CPU tensor input (pinned for speed) -> CPU tensor outputs.  ``allow_tall`` (an extension; the reference is square-only)
    accepts m > n factors."""
    mode = _dev.out_mode(g)
    shape = tuple(int(s) for s in g.shape)
    if len(shape) != 2 or (shape[1] != shape[0] and not (allow_tall and shape[0] > shape[1])):
        raise ValueError("the input factor must be square")
    m, n = shape
    if signature is None:
        signature = Signature(n, n)
    if signature.n != n:
        raise ValueError("signature order does not match the matrix")
    if n % cfg.block_width or n < cfg.block_width:
        raise ValueError(f"order {n} must be a positive multiple of block_width "
                         f"{cfg.block_width}")
    G0 = _dev.to_colmajor(g)
    solver = Solver(n, cfg, signature, m=m)
    sigma, U, V, stats, converged = solver.solve_device(G0)
    return HsvdResult(
        sigma=_dev.vector_out(sigma, mode),
        u=_dev.from_colmajor(U, mode),
        v=_dev.from_colmajor(V, mode) if V is not None else None,
        signature=signature,
        stats=tuple(stats),
        block_sweeps=len(stats),
        converged=converged,
    )
