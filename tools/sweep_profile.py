"""Per-sweep time and kernel-class split of the bench.py config 3 solve
(dev tool):  [OVERLAP=1] python tools/sweep_profile.py [n]
(with OVERLAP=1 the class split is not meaningful: inner includes the update)"""

import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import _lib  # noqa: E402
from paper_1401_2720_b200.driver import Solver  # noqa: E402
from paper_1401_2720_b200.testgen import SpectrumSpec, canonical_sort, gen_factor_orth_device, \
    gen_spectrum  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    from paper_1401_2720_b200 import testgen as T, workloads as WL

    wl = WL.CONFIG3 if n == WL.CONFIG3.n else WL.scaled(WL.CONFIG3, n)
    G0, _, n_plus = T.workload_input_device(wl)
    solver = Solver(n, J.SolverConfig(), J.Signature(n, n_plus))
    eng = solver.engine
    lib = _lib.load_library()
    import os

    overlap = int(os.environ.get("OVERLAP", "0"))
    lib.jh_set_overlap(overlap)  # 0: kernels apart, so the classes separate
    G = G0.clone()
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    nsw = int(os.environ.get("SWEEPS", "30"))
    for sweep in range(nsw):
        lib.jh_profile_begin(4 * eng.nsteps + 16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rot, proper = eng.one_sweep(G, V)
        e1.record()
        torch.cuda.synchronize()
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        lib.jh_profile_end(ms, cnt)
        print(json.dumps({"sweep": sweep + 1, "ms": e0.elapsed_time(e1), "rot": rot,
                          "proper": proper, "tasks_rotated": eng.tasks_rotated[-1],
                          "gram_ms": ms[0], "inner_ms": ms[1], "update_ms": ms[2] + ms[3], "overlap": overlap}), flush=True)
        if proper == 0:
            break


if __name__ == "__main__":
    main()
