"""The reference-side ctypes binding printed in INTEGRATION.md runs as
written (only the library path is substituted) and matches the package's
own sweep loop bitwise: the snippet a maintainer would paste is tested."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _snippet():
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n(# jhsvd/_b200\.py.*?)```", text, re.S).group(1)
    lib = ROOT / "paper_1401_2720_b200" / "_lib" / "libjhsvd_b200.so"
    return code.replace('ctypes.CDLL("libjhsvd_b200.so")', f'ctypes.CDLL("{lib}")')


def test_snippet_declares_argtypes_for_every_call():
    code = _snippet()
    for fn in re.findall(r"_lib\.(jh_\w+)\(", code):
        assert f"_lib.{fn}.argtypes" in code, fn


@pytest.mark.gpu
@pytest.mark.parametrize("n,nplus", [(256, 256), (256, 100)])
def test_snippet_runs_and_matches(n, nplus):
    import paper_1401_2720_b200 as J

    ns = {}
    exec(compile(_snippet(), "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(n + nplus)
    g = np.asfortranarray(rng.standard_normal((n, n)))
    v = np.asfortranarray(np.eye(n))
    cfg = J.SolverConfig()
    sig = J.Signature(n, nplus)
    outer, inner = J.make_strategy("rrow", n // 16), J.make_strategy("rrow", 32)
    g1, v1 = g.copy(order="F"), v.copy(order="F")
    stats, conv = ns["run_block_jacobi_inplace_gpu"](g1, v1, sig, cfg, outer, inner)
    g2, v2 = g.copy(order="F"), v.copy(order="F")
    ref_stats, ref_conv = J.run_block_jacobi_inplace(g2, v2, sig, cfg)
    assert stats == ref_stats and conv == ref_conv
    assert np.array_equal(g1, g2) and np.array_equal(v1, v2)
