"""Whole-solve A/B of the sweep engines under the board's power limit (dev
tool): config-3 input, the full solve with engine 0 (per-p-step update of
G and V) and engine 1 (V paired over two p-steps, mixed into the G update
launch), per-sweep ms and energy (NVML).

    python tools/engine_ab.py [n] [engines, e.g. 1,0,1,0]
"""
import json
import sys
from pathlib import Path

import pynvml
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import testgen as T, workloads as WL  # noqa: E402
from paper_1401_2720_b200.driver import Solver  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    engines = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,0,1,0").split(",")]
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    wl = WL.CONFIG3 if n == WL.CONFIG3.n else WL.scaled(WL.CONFIG3, n)
    G0, _, npl = T.workload_input_device(wl)
    s = Solver(n, J.SolverConfig(**wl.solver_kwargs()), J.Signature(n, npl))
    eng = s.engine
    default = eng.engine
    for e in engines:
        eng.engine = e if e == 0 else default
        G = G0.clone()
        V = torch.eye(n, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        e_start = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ms, stats = [], []
        eng.tasks_rotated = []
        joules_sweep = []
        for _ in range(eng.cfg.max_block_sweeps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            j0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
            e0.record()
            rot, proper = eng.one_sweep(G, V)
            e1.record()
            torch.cuda.synchronize()
            joules_sweep.append(round((pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - j0) / 1e3, 1))
            ms.append(round(e0.elapsed_time(e1), 1))
            stats.append((rot, proper))
            if proper == 0:
                break
        joules = (pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - e_start) / 1e3
        print(json.dumps({"engine": e, "total_s": round(sum(ms) / 1e3, 3), "joules": joules,
                          "ms_per_sweep": ms, "joules_per_sweep": joules_sweep,
                          "tasks_rotated": list(eng.tasks_rotated), "sweeps": len(ms)}),
              flush=True)
        del G, V
    eng.engine = default


if __name__ == "__main__":
    main()
