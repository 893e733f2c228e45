"""Per-sweep time and kernel-class split of the bench.py config 3 solve
(dev tool):  python tools/sweep_profile.py [n]"""

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
    lam = gen_spectrum(SpectrumSpec(2, n, 3))
    lam_sorted, n_plus = canonical_sort(lam)
    G0 = gen_factor_orth_device(np.sqrt(np.abs(lam_sorted)), seed=3)
    solver = Solver(n, J.SolverConfig(), J.Signature(n, n_plus))
    eng = solver.engine
    lib = _lib.load_library()
    lib.jh_set_overlap(0)  # kernels apart, so the classes separate
    G = G0.clone()
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    import os

    phases = os.environ.get("INNER_PHASES") == "1"
    nsw = int(os.environ.get("SWEEPS", "30"))
    for sweep in range(nsw):
        if phases:
            lib.jh_inner5_profile(1, None)
        lib.jh_profile_begin(4 * eng.nsteps + 16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rot, proper = eng.one_sweep(G, V)
        e1.record()
        torch.cuda.synchronize()
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        lib.jh_profile_end(ms, cnt)
        if phases:
            pv = (ctypes.c_uint64 * 12)()
            lib.jh_inner5_profile(0, pv)
            v = list(pv)
            nst, nt = max(v[5], 1), max(v[7], 1)
            print(json.dumps({"inner_phases": {
                "tasks": v[7], "inner_sweeps_per_task": v[6] / nt,
                "inner_steps_per_task": v[5] / nt,
                "cycles_per_step": {k: round(v[i] / nst, 1) for i, k in
                                    enumerate(["", "dots|wait_empty", "rotation|dots",
                                               "barrier1|rotation", "apply_barrier2|v_wait_full"])
                                    if i > 0},
                "load_cholesky_cycles_per_task": v[0] / nt,
                "task_cycles_avg": v[8] / nt, "task_cycles_max": v[9],
                "setup_cycles_per_task": v[10] / nt, "cholesky_cycles_per_task": v[11] / nt}}),
                  flush=True)
        print(json.dumps({"sweep": sweep + 1, "ms": e0.elapsed_time(e1), "rot": rot,
                          "proper": proper, "tasks_rotated": eng.tasks_rotated[-1],
                          "gram_ms": ms[0], "inner_ms": ms[1], "update_ms": ms[2] + ms[3]}), flush=True)
        if proper == 0:
            break


if __name__ == "__main__":
    main()
