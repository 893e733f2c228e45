"""Profiling target (dev tool): the config-3 input, then the first K p-steps
of sweep 1 on engine 1 -- the steady state of the hot kernels, without a
whole solve's 27k launches.  Run under ncu:

    ncu --set full -k regex:k_update_mix --launch-skip 20 --launch-count 1 \
        python tools/ncu_target.py [K] [n]
"""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import testgen as T, workloads as WL  # noqa: E402
from paper_1401_2720_b200.driver import Solver  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    n = int(sys.argv[2]) if len(sys.argv) > 2 else WL.CONFIG3.n
    wl = WL.CONFIG3 if n == WL.CONFIG3.n else WL.scaled(WL.CONFIG3, n)
    G0, _, n_plus = T.workload_input_device(wl)
    solver = Solver(n, J.SolverConfig(**wl.solver_kwargs()), J.Signature(n, n_plus))
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    c = solver.engine.sweep(G0, V, 0, k)
    torch.cuda.synchronize()
    print("p-steps", k, "counters", c.tolist())


if __name__ == "__main__":
    main()
