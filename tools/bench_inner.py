"""A/B timing of the inner-Jacobi kernel variants on real Gram matrices
(p-step 0 of an n x n random factor); checks the variants agree bitwise."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_2720_b200 import _lib  # noqa: E402
from paper_1401_2720_b200.driver import SolverConfig, SweepEngine  # noqa: E402
from paper_1401_2720_b200.strategy import make_strategy  # noqa: E402


def main(n=16384, w=32, variants=(3, 4, 5), reps=5):
    lib = _lib.require_cuda()
    cfg = SolverConfig(block_width=w)
    eng = SweepEngine(n, n, n, cfg, make_strategy("rrow", n // (w // 2)),
                      make_strategy("rrow", w), n)
    g = torch.Generator(device="cuda").manual_seed(0)
    G = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    eng.sweep(G, V, 0, 1)  # leaves the Gram matrices of p-step 0 in the workspace
    torch.cuda.synchronize()
    ntask = n // w
    ws = eng.ws
    H = ws.data_ptr()
    Vb = H + ntask * w * w * 8
    trot = Vb + ntask * w * w * 8
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    ref = None
    for var in variants:
        times = []
        for r in range(reps):
            cnt.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = lib.jh_bench_inner(var, H, Vb, trot, eng.outer_dev.data_ptr(), ntask, w, n,
                                    eng.inner_dev.data_ptr(), cfg.inner_sweep_limit, eng.tol_c,
                                    cnt.data_ptr(), _lib.stream_handle())
            e1.record()
            torch.cuda.synchronize()
            assert rc == 0, rc
            times.append(e0.elapsed_time(e1))
        vout = ws[ntask * w * w * 8: 2 * ntask * w * w * 8].clone()
        same = None if ref is None else bool(torch.equal(vout, ref))
        ref = vout if ref is None else ref
        print(f"variant {var}: {min(times) * 1e3:8.1f} us (min of {reps}), counters "
              f"{cnt.cpu().tolist()}, V' identical to first: {same}", flush=True)


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]]
    main(*args[:2]) if args else main()
