"""Whole-solve bitwise validation against the C oracle at a BASELINE size
(run once on a GPU box; minutes of oracle time):
    python tools/validate_full.py 4   -> config 4 (8192 HSVD, n/2 negative)
    python tools/validate_full.py 2   -> config 2 (4096 graded, block-oriented)
    python tools/validate_full.py 3   -> config 3 (16384, the bench input; ~80 min of oracle)
Prints one JSON line."""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import testgen as T  # noqa: E402
from oracle import oracle as O  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    which = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    if which == 3:
        n = 16384
        lam = T.gen_spectrum(T.SpectrumSpec(2, n, 3))
        lam_sorted, n_plus = T.canonical_sort(lam)
        G0 = T.gen_factor_orth_device(np.sqrt(np.abs(lam_sorted)), seed=3)
        g = np.asfortranarray(G0.cpu().numpy().T)
        del G0
        cfg = J.SolverConfig(block_width=32)
    elif which == 4:
        n = 8192
        rng = np.random.default_rng(4)
        k = max(n / 1024.0, 1.0)
        mags = rng.uniform(1e-7, 10.0 * k, n)
        signs = np.ones(n)
        signs[rng.permutation(n)[: n // 2]] = -1.0
        G0, sig = T.gen_factor_device(signs * mags, seed=5)
        g = np.asfortranarray(G0.cpu().numpy().T)
        n_plus = sig.n_plus
        cfg = J.SolverConfig(block_width=32)
    else:
        n = 4096
        gen = torch.Generator(device="cuda").manual_seed(2)
        B = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
        B /= B.norm(dim=1, keepdim=True)
        d = torch.logspace(0, -12, n, dtype=torch.float64, device="cuda")
        g = np.asfortranarray((B * d.unsqueeze(1)).cpu().numpy().T)
        n_plus = n
        sig = J.Signature(n, n)
        cfg = J.SolverConfig(block_width=32, variant="block-oriented")
    t0 = time.time()
    res = J.block_jacobi(g, J.Signature(n, n_plus), cfg)
    t_gpu = time.time() - t0
    outer = J.as_table(J.make_strategy("rrow", n // 16))
    inner = J.as_table(J.make_strategy("rrow", 32))
    t0 = time.time()
    ref = O.block_jacobi(g, n_plus, cfg, outer, inner, threads=O.max_threads())
    t_cpu = time.time() - t0
    out = {"config": which, "n": n, "n_plus": n_plus, "sweeps": len(res.stats),
           "stats_equal": [list(s) for s in res.stats] == [list(s) for s in ref.stats],
           "sigma_bitwise": bool(np.array_equal(res.sigma, ref.sigma)),
           "u_bitwise": bool(np.array_equal(res.u, ref.u)),
           "v_bitwise": bool(np.array_equal(res.v, ref.v)),
           "sigma_sha256_16": sha(res.sigma), "gpu_wall_s": round(t_gpu, 2),
           "oracle_wall_s": round(t_cpu, 1), "oracle_threads": O.max_threads(),
           "device": torch.cuda.get_device_name(0)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
