"""Synthetic test factors with prescribed spectra (reference ``jhsvd.testgen``).

``gen_spectrum`` / ``canonical_sort`` / ``relative_error`` / ``gen_factor``
restate the reference (pkg/src/jhsvd/testgen.py:21-146) exactly: the
spectra and reflectors come from numpy's PCG64 with the same draws, and the
host ``gen_factor`` repeats the reference's numpy operations, so on the same
BLAS its output is bitwise the reference's (tests/golden/testgen.npz).

``gen_factor_device`` is the same construction on the GPU: the same random
draws (host PCG64, identical unit reflector vectors and hyperbolic
rotations, in the reference's order), the O(n^3) reflector applications in
FP64 on the device.  It differs from the host factor only by rounding
(~1e-15 relative) and makes the reference's hour-long host generation at
n = 8192 take seconds.  ``gen_factor_orth_device`` (G = Q diag(sigma) W^T
with Haar Q, W from a seeded QR) builds the tall and the 16384 inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .blockkernel import Signature


@dataclass(frozen=True)
class SpectrumSpec:
    type: int
    n: int
    seed: int

    def __post_init__(self):
        if self.type not in (1, 2, 3, 4):
            raise ValueError("spectrum type must be 1, 2, 3 or 4")
        if self.type in (1, 2) and self.n < 16:
            raise ValueError("types 1 and 2 pin the first 16 entries; need n >= 16")
        if self.n < 1:
            raise ValueError("spectrum length must be positive")


def _nonzero_normal(rng, size, scale):
    out = rng.normal(0.0, scale, size)
    while True:
        zeros = out == 0.0
        if not zeros.any():
            return out
        out[zeros] = rng.normal(0.0, scale, int(zeros.sum()))


def gen_spectrum(spec: SpectrumSpec) -> np.ndarray:
    """Pseudorandom eigenvalues (testgen.py:50-68): types 1/2 pin 16 entries
    at 0.5 (+1 for type 2) and draw the rest N(0, 0.1); types 3/4 are
    uniform in [1e-7, 10 max(n/1024, 1)], type 3 with random signs."""
    rng = np.random.Generator(np.random.PCG64(spec.seed))
    n = spec.n
    k = max(n / 1024.0, 1.0)
    if spec.type in (1, 2):
        lam = np.empty(n)
        lam[:16] = 0.5
        lam[16:] = _nonzero_normal(rng, n - 16, 0.1)
        if spec.type == 2:
            lam = 1.0 + lam
        return lam
    mags = rng.uniform(1e-7, 10.0 * k, n)
    if spec.type == 4:
        return mags
    signs = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    return signs * mags


def canonical_sort(lam) -> tuple[np.ndarray, int]:
    """Positives descending, then negatives by magnitude descending."""
    lam = np.asarray(lam, dtype=np.float64)
    if (lam == 0.0).any():
        raise ValueError("eigenvalues must be nonzero")
    plus = np.sort(lam[lam > 0.0])[::-1]
    minus = np.sort(lam[lam < 0.0])
    return np.concatenate((plus, minus)), plus.size


def relative_error(sigma, signature: Signature, lam) -> float:
    """Eq. 6.1: max |sigma_i^2 j_i - lambda_i| / |lambda_i| (testgen.py:136-146)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    lam_sorted, n_plus = canonical_sort(lam)
    if sigma.size != lam_sorted.size:
        raise ValueError("sigma and lambda lengths differ")
    if n_plus != signature.n_plus:
        raise ValueError("signature does not match the signs of lambda")
    implied = sigma ** 2 * signature.as_vector()
    return float(np.max(np.abs(implied - lam_sorted) / np.abs(lam_sorted)))


def _apply_reflectors(rng, g: np.ndarray, count: int) -> None:
    """g <- Q g with Q a product of `count` random Householder reflectors
    (testgen.py:82-88)."""
    n = g.shape[0]
    for _ in range(count):
        v = rng.normal(size=n)
        v /= np.linalg.norm(v)
        g -= 2.0 * np.outer(v, v @ g)


def _mix_j_orthogonal(rng, g: np.ndarray, n_plus: int, tanh_max: float) -> None:
    """g <- g W^T for a J-orthogonal W (testgen.py:91-114): reflectors inside
    each signature class, then 2n hyperbolic rotations across the boundary."""
    n = g.shape[0]
    for lo, hi in ((0, n_plus), (n_plus, n)):
        width = hi - lo
        if width < 2:
            continue
        block = np.asfortranarray(g[:, lo:hi].T)
        _apply_reflectors(rng, block, width)
        g[:, lo:hi] = block.T
    if 0 < n_plus < n:
        for _ in range(2 * n):
            i = int(rng.integers(0, n_plus))
            j = int(rng.integers(n_plus, n))
            th = tanh_max * (2.0 * rng.random() - 1.0)
            ch = 1.0 / math.sqrt(1.0 - th * th)
            gi = g[:, i].copy()
            gj = g[:, j].copy()
            g[:, i] = ch * (gi + th * gj)
            g[:, j] = ch * (th * gi + gj)


def gen_factor(lam, seed: int, tanh_max: float = 0.1) -> tuple[np.ndarray, Signature]:
    """Factor G = Q diag(sqrt|lam_sorted|) W^T whose hyperbolic singular
    values are sqrt|lam| (testgen.py:117-133); host numpy, O(n^3)."""
    lam_sorted, n_plus = canonical_sort(lam)
    n = lam_sorted.size
    rng = np.random.Generator(np.random.PCG64(seed))
    g = np.zeros((n, n), order="F")
    np.fill_diagonal(g, np.sqrt(np.abs(lam_sorted)))
    _apply_reflectors(rng, g, n)
    _mix_j_orthogonal(rng, g, n_plus, tanh_max)
    return np.asfortranarray(g), Signature(n, n_plus)


def _unit_reflectors(rng, length: int, count: int, batch: int = 256):
    """The unit reflector vectors of _apply_reflectors, drawn in the same
    order (one rng.normal(size=length) per reflector), in batches."""
    done = 0
    while done < count:
        k = min(batch, count - done)
        vs = np.empty((k, length))
        for i in range(k):
            v = rng.normal(size=length)
            v /= np.linalg.norm(v)
            vs[i] = v
        yield vs
        done += k


def gen_factor_device(lam, seed: int, tanh_max: float = 0.1):
    """``gen_factor`` on the GPU: (G, signature) with G the column-major
    device storage (an (n, n) tensor whose row i is column i of the factor).
    Same draws and operation order as the reference; the reflector
    applications run as FP64 rank-1 updates on the device."""
    import torch

    lam_sorted, n_plus = canonical_sort(lam)
    n = lam_sorted.size
    rng = np.random.Generator(np.random.PCG64(seed))
    dev = torch.device("cuda")
    # gt = g^T (row i of gt = column i of g)
    gt = torch.diag(torch.as_tensor(np.sqrt(np.abs(lam_sorted)), device=dev))
    # g <- H g  <=>  gt <- gt H:  gt -= 2 (gt v) v^T
    for vs in _unit_reflectors(rng, n, n):
        vd = torch.as_tensor(vs, device=dev)
        for v in vd:
            gt.addr_(gt @ v, v, alpha=-2.0)
    # class blocks: g[:, lo:hi] <- (H block^T)^T, i.e. gt[lo:hi] <- H gt[lo:hi]
    for lo, hi in ((0, n_plus), (n_plus, n)):
        width = hi - lo
        if width < 2:
            continue
        blk = gt[lo:hi]
        for vs in _unit_reflectors(rng, width, width):
            vd = torch.as_tensor(vs, device=dev)
            for v in vd:
                blk.addr_(v, v @ blk, alpha=-2.0)
    if 0 < n_plus < n:
        for _ in range(2 * n):
            i = int(rng.integers(0, n_plus))
            j = int(rng.integers(n_plus, n))
            th = tanh_max * (2.0 * rng.random() - 1.0)
            ch = 1.0 / math.sqrt(1.0 - th * th)
            gi = gt[i].clone()
            gj = gt[j].clone()
            gt[i] = ch * (gi + th * gj)
            gt[j] = ch * (th * gi + gj)
    return gt.contiguous(), Signature(n, n_plus)


def random_orthogonal_device(n: int, seed: int, m: int | None = None):
    """m x n (default n x n) matrix with orthonormal columns, FP64 on the GPU."""
    import torch

    m = n if m is None else m
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    q, r = torch.linalg.qr(a)
    # sign-fix so the distribution is Haar and the result deterministic
    q *= torch.sign(torch.diagonal(r)).unsqueeze(0)
    return q


def gen_factor_orth_device(sigma, seed: int, m: int | None = None):
    """G = Q diag(sigma) W^T (m x n, FP64, on the GPU, Haar Q and W) returned
    in column-major storage as an (n, m) tensor."""
    import torch

    sig = torch.as_tensor(np.ascontiguousarray(sigma, dtype=np.float64), device="cuda")
    n = sig.numel()
    m = n if m is None else m
    q = random_orthogonal_device(n, seed, m)
    w = random_orthogonal_device(n, seed + 1)
    # (n, m) storage of G = Q diag(s) W^T is G^T = W diag(s) Q^T
    gt = (w * sig.unsqueeze(0)) @ q.t()
    del q, w
    return gt.contiguous()


def gen_factor_butterfly_device(sigma, seed: int, m: int | None = None,
                                n_plus: int | None = None, passes: int = 2,
                                tanh_max: float = 0.1):
    """G = Q [diag(sigma); 0] W^T on the GPU (``jh_gen_butterfly``): Q, W
    random Givens butterflies, plus J-orthogonal hyperbolic layers when
    ``n_plus == n/2``.  Returns the column-major device storage, an (n, m)
    tensor whose row i is column i of G.  Bitwise equal to the host twin
    ``oracle/gen_butterfly.c`` (see ``workloads.py``)."""
    import torch

    from . import _lib

    lib = _lib.require_cuda()
    sig = torch.as_tensor(np.ascontiguousarray(sigma, dtype=np.float64), device="cuda")
    n = int(sig.numel())
    m = n if m is None else int(m)
    n_plus = n if n_plus is None else int(n_plus)
    nbytes = int(lib.jh_gen_workspace_bytes(m, n, n_plus, passes))
    if nbytes < 0:
        raise ValueError("jh_gen_butterfly needs m >= n powers of two and n_plus in {n, n/2}")
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    gt = torch.empty((n, m), dtype=torch.float64, device="cuda")
    _lib.check(lib.jh_gen_butterfly(gt.data_ptr(), m, m, n, sig.data_ptr(), n_plus, seed,
                                    passes, tanh_max, ws.data_ptr(), nbytes,
                                    _lib.stream_handle()), "gen_butterfly")
    return gt


def workload_input_device(wl):
    """(device storage (n, m), prescribed sigma in generator order, n_plus)
    of a ``workloads.Workload``."""
    sigma, n_plus = wl.sigma_nplus()
    gt = gen_factor_butterfly_device(sigma, wl.gen_seed, m=wl.m, n_plus=n_plus,
                                     passes=wl.passes, tanh_max=wl.tanh_max)
    return gt, sigma, n_plus
