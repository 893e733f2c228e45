"""Phase times of one public-API solve from pinned host memory (dev tool):
    python tools/e2e_breakdown.py [n]"""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import _dev, driver  # noqa: E402
from paper_1401_2720_b200.testgen import SpectrumSpec, canonical_sort, gen_factor_orth_device, \
    gen_spectrum  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    lam = gen_spectrum(SpectrumSpec(2, n, 3))
    lam_sorted, n_plus = canonical_sort(lam)
    G0 = gen_factor_orth_device(np.sqrt(np.abs(lam_sorted)), seed=3)
    host_in = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    host_in.copy_(G0)
    del G0
    g = host_in.t()
    cfg = J.SolverConfig()
    sig = J.Signature(n, n_plus)
    for rep in range(2):
        T = {}
        torch.cuda.synchronize()
        t = t_all = time.perf_counter()

        def mark(k):
            nonlocal t
            torch.cuda.synchronize()
            now = time.perf_counter()
            T[k] = round(now - t, 4)
            t = now

        Gd = _dev.to_colmajor(g)
        mark("h2d")
        solver = driver.Solver(n, cfg, sig, m=n)
        mark("solver_init")
        bool(torch.isfinite(Gd).all())
        mark("isfinite")
        driver._check_scaling_dev(Gd, n, n)
        mark("check_scaling")
        work = Gd.clone()
        V = torch.eye(n, dtype=torch.float64, device=Gd.device)
        mark("clone_eye")
        stats, conv = solver.engine.run(work, V)
        mark("sweeps")
        sigma, U = driver._sigma_u_dev(work, n, n)
        order = driver._class_sort_order(sigma, n_plus)
        sigma, U, V = sigma[order], U.index_select(0, order), V.index_select(0, order)
        mark("sigma_u_sort")
        u = _dev.from_colmajor(U, "host")
        v = _dev.from_colmajor(V, "host")
        s = _dev.vector_out(sigma, "host")
        mark("d2h")
        T["total"] = round(time.perf_counter() - t_all, 4)
        print(rep, T, flush=True)
        del u, v, s, U, V, work, Gd, solver
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
