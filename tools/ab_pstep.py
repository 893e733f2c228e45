"""A/B timing of library builds on the steady state of sweep 1 (dev tool):
for each library in JHSVD_LIBS (comma separated; '' = the in-tree build),
in a fresh process, the config-3 input and K p-steps of sweep 1 (engine 1),
timed per p-step with CUDA events, plus the sha256 of G and V afterwards
(every build must give the same bytes).

    JHSVD_LIBS=a.so,b.so python tools/ab_pstep.py [K] [n]
"""

import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import hashlib, json, sys, torch
sys.path.insert(0, '.')
import paper_1401_2720_b200 as J
from paper_1401_2720_b200 import testgen as T, workloads as WL, _lib
from paper_1401_2720_b200.driver import Solver
k, n = int(sys.argv[1]), int(sys.argv[2])
wl = WL.CONFIG3 if n == WL.CONFIG3.n else WL.scaled(WL.CONFIG3, n)
G0, _, npl = T.workload_input_device(wl)
s = Solver(n, J.SolverConfig(**wl.solver_kwargs()), J.Signature(n, npl))
V0 = torch.eye(n, dtype=torch.float64, device='cuda')
out = {}
for overlap in (1, 0):
    _lib.load_library().jh_set_overlap(overlap)
    G, V = G0.clone(), V0.clone()
    s.engine.sweep(G, V, 0, 4)  # warm
    G, V = G0.clone(), V0.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s.engine.sweep(G, V, 0, k); e1.record(); torch.cuda.synchronize()
    out[f"ms_per_pstep_overlap{overlap}"] = e0.elapsed_time(e1) / k
sha = hashlib.sha256(G.cpu().numpy().tobytes() + V.cpu().numpy().tobytes()).hexdigest()[:16]
out["sha"] = sha
print(json.dumps(out))
"""


def main():
    k = sys.argv[1] if len(sys.argv) > 1 else "64"
    n = sys.argv[2] if len(sys.argv) > 2 else "16384"
    libs = os.environ.get("JHSVD_LIBS", "").split(",")
    for lib in libs:
        env = dict(os.environ)
        env.pop("JHSVD_LIBS", None)
        if lib:
            env["JHSVD_LIB"] = str(Path(lib).resolve())
        r = subprocess.run([sys.executable, "-c", CHILD, k, n], cwd=ROOT, env=env,
                           capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
        print(json.dumps({"lib": lib or "in-tree", "result": line}), flush=True)


if __name__ == "__main__":
    main()
