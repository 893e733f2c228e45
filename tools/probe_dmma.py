"""Characterise the rounding of FP64 DMMA (mma.sync m8n8k4 f64) on this GPU.

For each output entry d = c + sum_k a_k b_k (k = 0..3) compare the hardware
result with (i) the in-order fma chain fma(a3,b3,fma(a2,b2,fma(a1,b1,fma(a0,b0,c)))),
(ii) the exact value rounded once.  Writes a JSON summary to
gpurun_out/dmma_probe.json (or the path given).
"""
import json
import sys
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1401_2720_b200 import _lib  # noqa: E402
from tools.dev import devlib  # noqa: E402


def main(out="gpurun_out/dmma_probe.json"):
    _lib.require_cuda()
    lib = devlib.load()
    nt = 8192
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(nt, 32, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(nt, 32, dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(nt, 64, dtype=torch.float64, device="cuda", generator=g)
    scale = torch.tensor([1e8, 1.0, 1e8, 1.0], dtype=torch.float64, device="cuda").repeat(8)
    A[1::3] *= scale
    C[2::3] *= 1e-12
    Dm = torch.empty_like(C)
    Df = torch.empty_like(C)
    _lib.check(lib.jh_probe_dmma(A.data_ptr(), B.data_ptr(), C.data_ptr(), Dm.data_ptr(),
                                 Df.data_ptr(), nt, _lib.stream_handle()), "probe")
    torch.cuda.synchronize()
    a, b, c = A.cpu().numpy(), B.cpu().numpy(), C.cpu().numpy()
    dm, df = Dm.cpu().numpy(), Df.cpu().numpy()
    mism = dm != df
    res = {"entries": int(dm.size), "mismatch_vs_inorder_fma": int(mism.sum())}
    # exact-rounded comparison on a sample of entries
    idx = np.argwhere(mism.reshape(nt, 8, 8))[:200] if mism.any() else np.argwhere(
        np.ones((nt, 8, 8), bool))[:200]
    exact_eq = fma_eq = 0
    for t, r, col in idx:
        at = a[t].reshape(8, 4)
        bt = b[t].reshape(4, 8)
        ex = Fraction(float(c[t].reshape(8, 8)[r, col]))
        for k in range(4):
            ex += Fraction(float(at[r, k])) * Fraction(float(bt[k, col]))
        rounded = float(ex)  # correctly rounded (Fraction -> float rounds to nearest)
        exact_eq += rounded == dm[t].reshape(8, 8)[r, col]
        fma_eq += df[t].reshape(8, 8)[r, col] == dm[t].reshape(8, 8)[r, col]
    res.update({"sampled": int(len(idx)), "sample_equal_exact_single_rounding": int(exact_eq),
                "sample_equal_inorder_fma": int(fma_eq)})
    print(json.dumps(res))
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
