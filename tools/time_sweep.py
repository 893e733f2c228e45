"""Time block sweeps of the single-GPU engine on random input (dev tool).

    python tools/time_sweep.py N [W] [SWEEPS] [STEPS]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1401_2720_b200.driver import SolverConfig, SweepEngine  # noqa: E402
from paper_1401_2720_b200.strategy import make_strategy  # noqa: E402


def main():
    n = int(sys.argv[1])
    w = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else None
    cfg = SolverConfig(block_width=w)
    t0 = time.time()
    outer = make_strategy("rrow", n // (w // 2))
    inner = make_strategy("rrow", w)
    print(f"strategy {time.time() - t0:.2f}s", flush=True)
    eng = SweepEngine(n, n, n, cfg, outer, inner, n)
    g = torch.Generator(device="cuda").manual_seed(0)
    G = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    # warm-up on a copy
    Gw, Vw = G.clone(), V.clone()
    eng.sweep(Gw, Vw, 0, min(4, eng.nsteps))
    torch.cuda.synchronize()
    import ctypes

    from paper_1401_2720_b200 import _lib

    lib = _lib.load_library()
    for s in range(sweeps):
        lib.jh_profile_begin(4 * eng.nsteps + 16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = eng.sweep(G, V, 0, steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ns = steps or eng.nsteps
        rot, proper, key, nrot = c.cpu().tolist()
        pms = (ctypes.c_double * 4)()
        pcnt = (ctypes.c_int64 * 4)()
        lib.jh_profile_end(pms, pcnt)
        print(f"n={n} w={w} sweep {s}: {ms:.1f} ms for {ns} p-steps "
              f"({ms / ns:.3f} ms/p-step) rot={rot} proper={proper} key={key} "
              f"rotated_tasks={nrot}", flush=True)
        names = ("gram", "factor_inner", "update", "dataflow")
        ntask = n // w
        for k in range(4):
            if pcnt[k] == 0:
                continue
            per = pms[k] / max(pcnt[k], 1)
            extra = ""
            if k == 0:
                gbs = ntask * 8.0 * w * n / (per / 1e3) / 1e9
                extra = f" {gbs:.0f} GB/s"
            if k == 2:
                gbs = nrot * 16.0 * w * 2 * n / (pms[k] / 1e3) / 1e9
                extra = f" {gbs:.0f} GB/s"
            if k == 3:
                nst = steps or eng.nsteps
                byts = nst * ntask * 8.0 * w * n + nrot * 16.0 * w * 2 * n
                extra = f" {byts / (pms[k] / 1e3) / 1e9:.0f} GB/s (Gram + update bytes)"
            print(f"   {names[k]:13s} {pms[k]:9.2f} ms total, {per * 1e3:9.1f} us/launch{extra}")


if __name__ == "__main__" and "--inner" not in sys.argv:
    main()


def inner_profile(n=4096, w=32, steps=8):
    """Phase timing of the inner Jacobi (cycles per inner p-step)."""
    import ctypes

    from paper_1401_2720_b200 import _lib

    lib = _lib.load_library()
    cfg = SolverConfig(block_width=w)
    eng = SweepEngine(n, n, n, cfg, make_strategy("rrow", n // (w // 2)), make_strategy("rrow", w), n)
    g = torch.Generator(device="cuda").manual_seed(0)
    G = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    out = (ctypes.c_ulonglong * 8)()
    lib.jh_inner_profile(1, None)
    eng.sweep(G, V, 0, steps)
    lib.jh_inner_profile(0, out)
    v = list(out)
    nst = max(v[5], 1)
    names = ["dots", "rotation", "publish", "apply+exch", "(v3 bar2)"]
    print(f"inner profile n={n} w={w}: {v[7]} tasks, {v[6] / max(v[7], 1):.2f} inner sweeps/task, "
          f"{v[5] / max(v[7], 1):.1f} inner p-steps/task")
    tot = sum(v[:5]) / nst
    for k in range(5):
        print(f"   {names[k]:9s} {v[k] / nst:8.1f} cycles/step")
    print(f"   total     {tot:8.1f} cycles/step")


if __name__ == "__main__" and "--inner" in sys.argv:
    args = [a for a in sys.argv[1:] if a != "--inner"]
    inner_profile(*(int(a) for a in args))
