"""Profiling target for a late sweep (dev tool): the config-3 input, S whole
sweeps outside the profiler, then K p-steps of the next sweep between
cudaProfilerStart/Stop.  Run under ncu with --profile-from-start off:

    ncu --profile-from-start off --set full -k regex:k_update_mix -c 2 \
        python tools/ncu_late.py [S] [K] [overlap]
"""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import _lib, testgen as T, workloads as WL  # noqa: E402
from paper_1401_2720_b200.driver import Solver  # noqa: E402


def main():
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 9
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    overlap = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    wl = WL.CONFIG3
    n = wl.n
    G0, _, n_plus = T.workload_input_device(wl)
    solver = Solver(n, J.SolverConfig(**wl.solver_kwargs()), J.Signature(n, n_plus))
    _lib.load_library().jh_set_overlap(overlap)
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    for _ in range(s):
        print("sweep", solver.engine.one_sweep(G0, V), flush=True)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    c = solver.engine.sweep(G0, V, 0, k)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("p-steps", k, "counters", c.tolist())


if __name__ == "__main__":
    main()
