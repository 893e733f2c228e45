"""ctypes front-end of the C oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg use
this module, and only as the checker / CPU baseline.  It restates, on top of
``jhsvd_oracle.c``, the reference driver logic:

* ``run_block_jacobi_inplace`` / ``block_jacobi`` -- reference
  ``pkg/src/jhsvd/driver.py:125-313``;
* ``run_distributed`` -- reference ``pkg/src/jhsvd/distsim.py:216-424``
  (workers simulated sequentially, exchange by the given mapping);
* kernel wrappers -- reference ``blockkernel.py`` / ``robustnorm.py``.

Pivot tables are inputs (int32[steps][n/2][2], 0-based); the strategy
generator they come from is pinned separately against reference digests.
Matrices are numpy arrays in Fortran (column-major) order, like the
reference.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path
from types import SimpleNamespace
from typing import Callable, Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libjhsvd_oracle.so"
EPS = 2.0 ** -53

_lib = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_p = ctypes.c_void_p


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.or_gram.argtypes = [_p, _i64, _i64, _i32, _p]
        L.or_cholesky.argtypes = [_p, _i32]
        L.or_cholesky.restype = _i32
        L.or_inner_jacobi.argtypes = [_p, _p, _i32, _p, _i32, _p, _d, _i32, _p]
        L.or_postmultiply.argtypes = [_p, _i64, _i64, _i32, _p, _p, _i64]
        L.or_qr_peeloff.argtypes = [_p, _i64, _i64, _i32, _p]
        L.or_qr_peeloff.restype = _i32
        L.or_back_substitute.argtypes = [_p, _i32, _p, _i32, _p]
        L.or_norm2.argtypes = [_p, _i64, _i32, _p, _p]
        L.or_safe_bounds.argtypes = [_i64, _p, _p]
        L.or_rotation.argtypes = [_d, _d, _d, _d, _p]
        L.or_block_sweep.argtypes = [_p, _i64, _i64, _i64, _p, _i64, _i64, _i32, _p, _i32,
                                     _p, _i64, _i32, _d, _i32, _i32, _p, _p, _p]
        L.or_block_sweep.restype = _i32
        L.or_max_threads.restype = _i32
        L.or_gen_butterfly.argtypes = [_p, _i64, _i64, _i64, _p, _i64, ctypes.c_uint64, _i32, _d]
        L.or_gen_butterfly.restype = _i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class OracleError(ArithmeticError):
    """Raised with .kind in {'rank', 'jdef'} and .index (1-based)."""

    def __init__(self, kind: str, index: int, msg: str = ""):
        super().__init__(msg or f"{kind} failure at index {index}")
        self.kind = kind
        self.index = index


# ---------------------------------------------------------------------------
# kernel wrappers


def gram(g) -> np.ndarray:
    g = _f64(g)
    m, c = g.shape
    h = np.zeros((c, c), order="F")
    lib().or_gram(_ptr(g), m, m, c, _ptr(h))
    return h


def cholesky_in_place(h) -> np.ndarray:
    hf = _f64(h).copy(order="F")
    c = hf.shape[0]
    info = lib().or_cholesky(_ptr(hf), c)
    if info:
        raise OracleError("rank", info)
    r = np.zeros_like(hf)
    for j in range(c):
        r[: j + 1, j] = hf[j, : j + 1]
    return r


def inner_jacobi(r, signs, table, max_sweeps, eps_factor=1.0):
    """(r_out, v_acc, rotations, proper, sweeps); signs: +-1 per column."""
    r = _f64(r).copy(order="F")
    c = r.shape[0]
    v = np.eye(c, order="F")
    tab = np.ascontiguousarray(table, dtype=np.int32)
    sg = np.ascontiguousarray(signs, dtype=np.int8)
    out = np.zeros(5, dtype=np.int64)
    tol_c = EPS * math.sqrt(c) * eps_factor
    lib().or_inner_jacobi(_ptr(r), _ptr(v), c, _ptr(tab), tab.shape[0], _ptr(sg),
                          tol_c, max_sweeps, _ptr(out))
    if out[3] == 1:
        raise OracleError("rank", int(out[4]) + 1)
    if out[3] == 2:
        raise OracleError("jdef", int(out[4]) + 1)
    return r, v, int(out[0]), int(out[1]), int(out[2])


def postmultiply(a, v) -> np.ndarray:
    a = _f64(a)
    v = _f64(v)
    m, c = a.shape
    out = np.empty((m, c), order="F")
    lib().or_postmultiply(_ptr(a), m, m, c, _ptr(v), _ptr(out), m)
    return out


def qr_peeloff(g) -> np.ndarray:
    g = _f64(g)
    m, c = g.shape
    if m % c or m < c:
        raise ValueError(f"row count {m} must be a positive multiple of {c}")
    r = np.zeros((c, c), order="F")
    lib().or_qr_peeloff(_ptr(g), m, m, c, _ptr(r))
    return r


def solve_for_v(r, w) -> np.ndarray:
    r = _f64(r)
    w = _f64(w)
    n = r.shape[0]
    if np.any(np.diag(r) == 0.0):
        raise ZeroDivisionError("zero diagonal entry")
    out = np.empty_like(w)
    lib().or_back_substitute(_ptr(r), n, _ptr(w), w.shape[1], _ptr(out))
    return out


def norm2(x, force_scaled=False) -> tuple[int, float]:
    x = np.ascontiguousarray(x, dtype=np.float64)
    js = np.zeros(1, dtype=np.int64)
    s = np.zeros(1)
    lib().or_norm2(_ptr(x), x.shape[0], int(force_scaled), _ptr(js), _ptr(s))
    return int(js[0]), float(s[0])


def safe_bounds(n: int) -> tuple[float, float]:
    a = np.zeros(1)
    b = np.zeros(1)
    lib().or_safe_bounds(n, _ptr(a), _ptr(b))
    return float(a[0]), float(b[0])


def rotation(hpp, hqq, hpq, t):
    out = np.zeros(3)
    lib().or_rotation(hpp, hqq, hpq, t, _ptr(out))
    return float(out[0]), float(out[1]), bool(out[2])


# ---------------------------------------------------------------------------
# driver (reference driver.py)


def _cfg(cfg):
    d = dict(block_width=32, variant="full-block", max_block_sweeps=30, max_inner_sweeps=30,
             accumulate_v=True, solve_v=False, shortening="cholesky", eps_factor=1.0)
    if cfg is not None:
        for k in list(d):
            if hasattr(cfg, k):
                d[k] = getattr(cfg, k)
            elif isinstance(cfg, dict) and k in cfg:
                d[k] = cfg[k]
    ns = SimpleNamespace(**d)
    ns.inner_limit = 1 if ns.variant == "block-oriented" else ns.max_inner_sweeps
    return ns


def block_sweep(g, v, n_plus, cfg, outer_tab, inner_tab, threads=0, nsteps=None, gblock=None,
                err_out=None):
    """One block sweep (or its first ``nsteps`` p-steps) in place; returns
    (rotations, proper).  Raises OracleError like the reference.  ``gblock``
    (int32 per local block-column) gives the global block index for the J
    signature of sharded solves; with ``err_out`` (list) the failure (status,
    1-based index, p-step, task) is appended instead of raised."""
    c = _cfg(cfg)
    m, n = g.shape
    w = c.block_width
    tab = np.ascontiguousarray(outer_tab, dtype=np.int32)
    itab = np.ascontiguousarray(inner_tab, dtype=np.int32)
    ns = tab.shape[0] if nsteps is None else int(nsteps)
    counts = np.zeros(2, dtype=np.int64)
    err = np.zeros(3, dtype=np.int64)
    tol_c = EPS * math.sqrt(w) * c.eps_factor
    vp = _ptr(v) if v is not None else None
    nv = v.shape[0] if v is not None else 0
    gb = np.ascontiguousarray(gblock, dtype=np.int32) if gblock is not None else None
    st = lib().or_block_sweep(_ptr(g), m, m, n, vp, nv, nv, w, _ptr(tab), ns, _ptr(itab),
                              int(n_plus), c.inner_limit, tol_c,
                              0 if c.shortening == "cholesky" else 1, int(threads),
                              _ptr(counts), _ptr(err), _ptr(gb) if gb is not None else None)
    if st and err_out is not None:
        err_out.append((int(st), int(err[0]), int(err[1]), int(err[2])))
        return int(counts[0]), int(counts[1])
    if st == 1 or st == 2:
        raise OracleError("rank", int(err[0]))
    if st == 3:
        raise OracleError("jdef", int(err[0]))
    return int(counts[0]), int(counts[1])


def run_block_jacobi_inplace(g, v, n_plus, cfg, outer_tab, inner_tab, threads=0,
                             early_stop: Optional[Callable[[], bool]] = None):
    """driver.py:125-200; g (m x n, F-order) and v updated in place."""
    c = _cfg(cfg)
    stats = []
    converged = False
    for _ in range(c.max_block_sweeps):
        rot, proper = block_sweep(g, v, n_plus, cfg, outer_tab, inner_tab, threads)
        stats.append((rot, proper))
        if proper == 0:
            converged = True
            break
        if early_stop is not None and early_stop():
            break
    return stats, converged


def extract_sigma(g) -> np.ndarray:
    sig = np.empty(g.shape[1])
    for i in range(g.shape[1]):
        js, s = norm2(g[:, i])
        if s == 0.0:
            raise OracleError("rank", i + 1)
        sig[i] = math.ldexp(s, -js)
    return sig


def class_sort_order(sigma, n_plus) -> np.ndarray:
    order = np.arange(sigma.size)
    plus, minus = order[:n_plus], order[n_plus:]
    plus = plus[np.argsort(-sigma[plus], kind="stable")]
    minus = minus[np.argsort(-sigma[minus], kind="stable")]
    return np.concatenate((plus, minus))


def block_jacobi(g, n_plus, cfg, outer_tab, inner_tab, threads=0):
    """driver.py:251-313 (input checks omitted: the oracle is fed valid
    inputs).  Returns a namespace with sigma, u, v, stats, block_sweeps,
    converged."""
    c = _cfg(cfg)
    g0 = _f64(g)
    n = g0.shape[1]
    work = g0.copy(order="F")
    keep = g0.copy(order="F") if c.solve_v else None
    v = np.eye(n, order="F") if c.accumulate_v else None
    stats, conv = run_block_jacobi_inplace(work, v, n_plus, cfg, outer_tab, inner_tab, threads)
    if c.solve_v:
        v = solve_for_v(keep, work)
    sigma = extract_sigma(work)
    u = work / sigma
    order = class_sort_order(sigma, n_plus)
    return SimpleNamespace(
        sigma=sigma[order], u=np.asfortranarray(u[:, order]),
        v=None if v is None else np.asfortranarray(v[:, order]),
        stats=tuple(stats), block_sweeps=len(stats), converged=conv)


# ---------------------------------------------------------------------------
# distributed outer level (distsim.py:216-424), workers simulated in turn


def local_n_plus(n_plus, p, q, bw):
    """distsim.py:427-433 (1-based block indices)."""
    lo_p, hi_p = (p - 1) * bw, p * bw
    lo_q, hi_q = (q - 1) * bw, q * bw
    return max(0, min(n_plus, hi_p) - lo_p) + max(0, min(n_plus, hi_q) - lo_q)


def run_distributed(g, n_plus, gw, cfg, assignments, nested_outer_tab, inner_tab,
                    threads=0):
    """assignments[s][i] = 1-based (p, q) block pair of worker i at step s.
    Returns (sigma, u, v, stats, converged)."""
    c = _cfg(cfg)
    gm = _f64(g)
    m, n = gm.shape
    bw = n // (2 * gw)
    ln = 2 * bw
    nsteps = len(assignments)
    want_v = c.accumulate_v or c.solve_v
    local_cfg = dict(block_width=c.block_width, variant=c.variant,
                     max_block_sweeps=1 if c.variant == "block-oriented" else c.max_block_sweeps,
                     max_inner_sweeps=c.max_inner_sweeps, accumulate_v=not c.solve_v,
                     solve_v=False, shortening=c.shortening, eps_factor=c.eps_factor)

    def blk(b):
        return slice((b - 1) * bw, b * bw)

    gx, vx = [], []
    for i in range(gw):
        p, q = assignments[0][i]
        gx.append(np.asfortranarray(np.hstack((gm[:, blk(p)], gm[:, blk(q)]))))
        if want_v:
            vv = np.zeros((n, ln), order="F")
            vv[blk(p), :bw] = np.eye(bw)
            vv[blk(q), bw:] = np.eye(bw)
            vx.append(vv)
        else:
            vx.append(None)
    stats = []
    converged = False
    for _sweep in range(c.max_block_sweeps):
        rot_t = proper_t = 0
        for s in range(nsteps):
            for i in range(gw):
                p, q = assignments[s][i]
                h = gram(gx[i])
                r = cholesky_in_place(h)
                work = r.copy(order="F")
                vhat = np.eye(ln, order="F") if not c.solve_v else None
                lst, _ = run_block_jacobi_inplace(work, vhat, local_n_plus(n_plus, p, q, bw),
                                                  local_cfg, nested_outer_tab, inner_tab,
                                                  threads)
                if c.solve_v:
                    vhat = solve_for_v(r, work)
                rot_t += sum(a for a, _ in lst)
                proper_t += sum(b for _, b in lst)
                if any(a for a, _ in lst):
                    gx[i] = postmultiply(gx[i], vhat)
                    if vx[i] is not None:
                        vx[i] = postmultiply(vx[i], vhat)
            # exchange: every worker keeps one block-column, receives the other
            nxt = assignments[(s + 1) % nsteps]
            held = {}
            for i in range(gw):
                p, q = assignments[s][i]
                held[p] = (gx[i][:, :bw], None if vx[i] is None else vx[i][:, :bw])
                held[q] = (gx[i][:, bw:], None if vx[i] is None else vx[i][:, bw:])
            for i in range(gw):
                np_, nq = nxt[i]
                gx[i] = np.asfortranarray(np.hstack((held[np_][0], held[nq][0])))
                if vx[i] is not None:
                    vx[i] = np.asfortranarray(np.hstack((held[np_][1], held[nq][1])))
        stats.append((rot_t, proper_t))
        if proper_t == 0:
            converged = True
            break
    gf = np.empty_like(gm)
    vf = np.empty((n, n), order="F") if want_v else None
    for i in range(gw):
        p, q = assignments[0][i]
        gf[:, blk(p)] = gx[i][:, :bw]
        gf[:, blk(q)] = gx[i][:, bw:]
        if vf is not None:
            vf[:, blk(p)] = vx[i][:, :bw]
            vf[:, blk(q)] = vx[i][:, bw:]
    sigma = extract_sigma(gf)
    u = gf / sigma
    order = class_sort_order(sigma, n_plus)
    return SimpleNamespace(sigma=sigma[order], u=np.asfortranarray(u[:, order]),
                           v=None if vf is None else np.asfortranarray(vf[:, order]),
                           stats=tuple(stats), block_sweeps=len(stats), converged=converged)


def gen_butterfly(sigma, m=None, n_plus=None, seed=0, passes=2, tanh_max=0.1) -> np.ndarray:
    """Host twin of the GPU input generator jh_gen_butterfly (gen_butterfly.c):
    G = Q [diag(sigma); 0] W^T, m x n, Fortran order."""
    sig = np.ascontiguousarray(sigma, dtype=np.float64)
    n = sig.size
    m = n if m is None else int(m)
    n_plus = n if n_plus is None else int(n_plus)
    g = np.empty((m, n), order="F")
    rc = lib().or_gen_butterfly(_ptr(g), m, m, n, _ptr(sig), n_plus, seed, passes, tanh_max)
    if rc:
        raise ValueError(f"or_gen_butterfly: unsupported shape (status {rc})")
    return g


def max_threads() -> int:
    return int(lib().or_max_threads())


def threads_default() -> int:
    return int(os.environ.get("JHSVD_ORACLE_THREADS", "0")) or max_threads()
