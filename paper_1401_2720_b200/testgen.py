"""Synthetic test factors with prescribed spectra (reference ``jhsvd.testgen``).

``gen_spectrum`` / ``canonical_sort`` / ``relative_error`` restate the
reference (pkg/src/jhsvd/testgen.py:21-146) exactly: the spectra come from
numpy's PCG64 with the same draws, so they are bitwise the reference's.
``gen_factor_device`` builds G = Q diag(sqrt|lambda|) W^T on the GPU with
FP64 Q, W from seeded Householder QR (torch.linalg.qr): the reference's
O(n^3) rank-1 reflector loop takes about an hour at n = 8192 on the host.
The device factor has the same spectrum but not the reference's bits (its
Q, W differ); parity runs use stored inputs instead.
"""

from __future__ import annotations

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


def gen_factor_device(sigma, seed: int, m: int | None = None):
    """G = Q diag(sigma) W^T (m x n, FP64, on the GPU) returned in
    column-major storage as an (n, m) tensor."""
    import torch

    sig = torch.as_tensor(np.asarray(sigma, dtype=np.float64), device="cuda")
    n = sig.numel()
    m = n if m is None else m
    q = random_orthogonal_device(n, seed, m)
    w = random_orthogonal_device(n, seed + 1)
    # (n, m) storage of G = Q diag(s) W^T is G^T = W diag(s) Q^T
    gt = (w * sig.unsqueeze(0)) @ q.t()
    del q, w
    return gt.contiguous()
