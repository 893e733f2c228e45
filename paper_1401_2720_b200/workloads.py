"""The BASELINE.json workloads as reproducible synthetic inputs.

Each configuration fixes a prescribed spectrum (host numpy, the reference's
``gen_spectrum`` draws) and the seed of the butterfly generator
``jh_gen_butterfly`` (``csrc/jh_gen.cu``): G = Q [diag(sigma); 0] W^T with Q,
W products of random Givens butterflies (and, for the hyperbolic config,
J-orthogonal hyperbolic layers).  The generator uses only correctly rounded
arithmetic in a fixed order, so its host twin (``oracle/gen_butterfly.c``,
test infrastructure) produces the same bytes; that is what lets the C oracle
solve the headline matrix end to end offline (``tools/oracle_offline.py``)
and the bench compare its result against that golden bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .testgen import SpectrumSpec, canonical_sort, gen_spectrum


@dataclass(frozen=True)
class Workload:
    name: str
    m: int
    n: int
    block_width: int
    variant: str
    strategy: str
    spectrum: str          # "type2" or "hsvd"
    spectrum_seed: int
    gen_seed: int
    passes: int = 2
    tanh_max: float = 0.1

    def lam(self) -> np.ndarray:
        """Prescribed eigenvalues of G J G^T (unsorted draw)."""
        if self.spectrum == "type2":
            return gen_spectrum(SpectrumSpec(2, self.n, self.spectrum_seed))
        if self.spectrum == "hsvd":
            # lambda = +-U(1e-7, 10 n / 1024), exactly n/2 negative
            rng = np.random.default_rng(self.spectrum_seed)
            k = max(self.n / 1024.0, 1.0)
            mags = rng.uniform(1e-7, 10.0 * k, self.n)
            signs = np.ones(self.n)
            signs[rng.permutation(self.n)[: self.n // 2]] = -1.0
            return signs * mags
        raise ValueError(self.spectrum)

    def sigma_nplus(self) -> tuple[np.ndarray, int]:
        """(prescribed sigma in generator column order, n_plus)."""
        lam_sorted, n_plus = canonical_sort(self.lam())
        return np.sqrt(np.abs(lam_sorted)), int(n_plus)

    def solver_kwargs(self) -> dict:
        return dict(block_width=self.block_width, variant=self.variant,
                    outer_strategy=self.strategy, inner_strategy=self.strategy)

    def describe(self) -> str:
        shape = f"{self.m}x{self.n}"
        spec = ("type-2 spectrum" if self.spectrum == "type2"
                else "hyperbolic, lambda = +-U(1e-7, 10n/1024), n/2 negative")
        return (f"{shape} FP64, {self.variant}, {self.strategy}, w={self.block_width}; "
                f"G = Q diag(sigma) W^T, {spec} (seed {self.spectrum_seed}), "
                f"butterfly Q/W (jh_gen_butterfly seed {self.gen_seed}, {self.passes} passes)")


CONFIG3 = Workload("config3", 16384, 16384, 32, "full-block", "rrow", "type2", 3, 3)
CONFIG4 = Workload("config4", 8192, 8192, 32, "full-block", "rrow", "hsvd", 4, 5)
CONFIG5 = Workload("config5", 131072, 8192, 32, "full-block", "rrow", "type2", 5, 7)
WORKLOADS = {w.name: w for w in (CONFIG3, CONFIG4, CONFIG5)}


def scaled(w: Workload, n: int, m: int | None = None) -> Workload:
    """The same construction at another size (tests)."""
    from dataclasses import replace

    return replace(w, name=f"{w.name}@{n}", n=n, m=n if m is None else m)
