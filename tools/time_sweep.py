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
    import os

    m = int(os.environ.get("M", n))  # rows (default square)
    cfg = SolverConfig(block_width=w)
    t0 = time.time()
    outer = make_strategy(os.environ.get("OUTER", "rrow"), n // (w // 2))
    inner = make_strategy("rrow", w)
    print(f"strategy {time.time() - t0:.2f}s", flush=True)
    eng = SweepEngine(m, n, n, cfg, outer, inner, n)
    g = torch.Generator(device="cuda").manual_seed(0)
    G = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g)
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    # warm-up on a copy
    Gw, Vw = G.clone(), V.clone()
    eng.sweep(Gw, Vw, 0, min(4, eng.nsteps))
    torch.cuda.synchronize()
    import ctypes

    from paper_1401_2720_b200 import _lib

    lib = _lib.load_library()
    import os

    trace = None
    if os.environ.get("TRACE"):
        cap = 4_000_000
        trace = torch.zeros(4 + 4 * cap, dtype=torch.int64, device="cuda")
        lib.jh_cycle_trace(trace.data_ptr(), cap)
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
        names = ("gram", "factor_inner", "update", "cycle")
        ntask = n // w
        for k in range(4):
            if pcnt[k] == 0:
                continue
            per = pms[k] / max(pcnt[k], 1)
            extra = ""
            if k == 0:
                gbs = ntask * 8.0 * w * m / (per / 1e3) / 1e9
                extra = f" {gbs:.0f} GB/s"
            if k == 2:
                gbs = nrot * 16.0 * w * 2 * n / (pms[k] / 1e3) / 1e9
                extra = f" {gbs:.0f} GB/s"
            if k == 3:
                nst = steps or eng.nsteps
                byts = nst * ntask * 8.0 * w * n + nrot * 16.0 * w * 2 * n
                extra = f" {byts / (pms[k] / 1e3) / 1e9:.0f} GB/s (Gram + update bytes)"
            print(f"   {names[k]:13s} {pms[k]:9.2f} ms total, {per * 1e3:9.1f} us/launch{extra}")
        if trace is not None:
            report_trace(trace, steps or eng.nsteps)
            lib.jh_cycle_trace(None, 0)
            trace = None


def report_trace(trace, nsteps):
    """Per item type: count, mean / max duration, busy share; and the
    critical-path chain B -> I -> B per p-step."""
    import numpy as np

    cnt = int(trace[0].item())
    rec = trace[4: 4 + 4 * cnt].view(cnt, 4).cpu().numpy()
    rec = rec[((rec[:, 1] >> 16) & 0xFFFF) == 0]  # one record per cluster (rank 0)
    item, smid, t0, t1 = rec[:, 0], rec[:, 1] & 0xFFFF, rec[:, 2], rec[:, 3]
    stream_us = rec[:, 1] >> 32
    cnt = len(rec)
    typ = (item >> 60) & 0xF
    a = (item >> 40) & 0xFFFFF
    dur = (t1 - t0) / 1e3
    tmin, tmax = t0.min(), t1.max()
    span = (tmax - tmin) / 1e3
    print(f"   trace: {cnt} items over {span:.0f} us on {len(np.unique(smid))} SMs (rank-0 CTAs)")
    for k, name in enumerate(("B", "I", "V")):
        m = typ == k
        if m.any():
            print(f"     {name}: n={m.sum():7d} mean {dur[m].mean():8.1f} us  p50 {np.median(dur[m]):8.1f}"
                  f"  max {dur[m].max():8.1f}  busy {dur[m].sum() / span:6.1f} clusters avg"
                  + (f"  (stream part mean {stream_us[m].mean():.1f} us)" if k == 0 else ""))
    # per-boundary: first start and last end of B items, I items per step
    for k, name in ((0, "B"),):
        m = typ == k
        st = a[m]
        if k == 1:
            st = st - st.min()
        first = np.full(nsteps + 2, np.inf)
        last = np.zeros(nsteps + 2)
        np.minimum.at(first, st, (t0[m] - tmin) / 1e3)
        np.maximum.at(last, st, (t1[m] - tmin) / 1e3)
        sel = [0, 1, 2, nsteps // 2, nsteps - 1]
        print(f"     {name} per step (first start / last end, us): " +
              " ".join(f"[{i}] {first[i]:.0f}/{last[i]:.0f}" for i in sel if i <= nsteps))


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
