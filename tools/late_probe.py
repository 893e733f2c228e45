"""Fixed cost of the update launches when no task rotates (dev tool): sweeps
over G = diag(d) (orthogonal columns), kernels kept apart.
    python tools/late_probe.py [n] [steps]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_2720_b200 import _lib  # noqa: E402
from paper_1401_2720_b200.driver import SolverConfig, SweepEngine  # noqa: E402
from paper_1401_2720_b200.strategy import make_strategy  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    w = 32
    cfg = SolverConfig(block_width=w)
    eng = SweepEngine(n, n, n, cfg, make_strategy("rrow", n // (w // 2)), make_strategy("rrow", w), n)
    G = torch.diag(torch.linspace(1.0, 2.0, n, dtype=torch.float64, device="cuda"))
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    lib = _lib.load_library()
    lib.jh_set_overlap(0)
    eng.sweep(G, V, 0, 4)
    for _ in range(2):
        lib.jh_profile_begin(4 * steps + 16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = eng.sweep(G, V, 0, steps)
        e1.record()
        torch.cuda.synchronize()
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        lib.jh_profile_end(ms, cnt)
        print(f"n={n}: {e0.elapsed_time(e1) / steps:.3f} ms/p-step, rotations {c.cpu().tolist()[0]}; "
              f"per launch: gram {ms[0] / max(cnt[0], 1) * 1e3:.1f} us, inner "
              f"{ms[1] / max(cnt[1], 1) * 1e3:.1f} us, update "
              f"{(ms[2] + ms[3]) / max(cnt[2], 1) * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
