"""Kernel-class split of one worker of the sharded solve (dev tool): the
config-3 input, worker 0's first cross segment at g GPUs, run alone on the
GPU with the kernels kept apart.

    python tools/worker_profile.py [g] [n]
"""

import ctypes
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import _lib, sharded as SH, testgen as T, workloads as WL  # noqa: E402
from paper_1401_2720_b200.driver import SweepEngine  # noqa: E402


def main():
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    n = int(sys.argv[2]) if len(sys.argv) > 2 else WL.CONFIG3.n
    wl = WL.CONFIG3 if n == WL.CONFIG3.n else WL.scaled(WL.CONFIG3, n)
    G0, _, n_plus = T.workload_input_device(wl)
    cfg = J.SolverConfig(**wl.solver_kwargs())
    w = cfg.block_width
    plan = SH.shard_plan(J.make_strategy(wl.strategy, n // (w // 2)), g)
    seg = plan.segments[0]
    slots = list(plan.held(seg.config, 0))
    tab, _ = SH._local_table(plan, seg, slots)
    gb = SH._gblock(plan, slots)
    bwc = plan.sb * (w // 2)
    Gl = torch.cat([G0[sc * bwc:(sc + 1) * bwc] for sc in slots]).contiguous()
    Vl = torch.zeros((2 * bwc, n), dtype=torch.float64, device="cuda")
    eng = SweepEngine(wl.m, 2 * bwc, n, cfg, None, J.make_strategy(cfg.inner_strategy, w), n_plus,
                      outer_table=tab, gblock=gb)
    lib = _lib.load_library()
    out = {"g": g, "tasks_per_pstep": int(tab.shape[1]), "psteps": int(tab.shape[0]),
           "engine": eng.engine}
    for overlap in (1, 0):
        lib.jh_set_overlap(overlap)
        G, V = Gl.clone(), Vl.clone()
        lib.jh_profile_begin(4096)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.sweep(G, V)
        e1.record()
        torch.cuda.synchronize()
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        lib.jh_profile_end(ms, cnt)
        k = tab.shape[0]
        out[f"overlap{overlap}"] = {"ms_per_pstep": e0.elapsed_time(e1) / k,
                                    "gram_ms": ms[0] / k, "inner_ms": ms[1] / k,
                                    "update_ms": (ms[2] + ms[3]) / k}
    lib.jh_set_overlap(1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
