"""The dense contractions of the outer (multi-GPU) level and the kernel-level
API on the DMMA pipe (csrc/jh_outer.cu): Gram (SYRK), post-multiplication
(GEMM) and the blocked Cholesky, bitwise against the C oracle's restatement
of blockkernel.py:76-127, 407-417 at outer-level sizes and ragged shapes."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(np.asfortranarray(a).T)).cuda()


@pytest.mark.parametrize("m,c", [(4096, 1024), (1000, 130), (33, 7), (2, 2), (16384, 256)])
def test_gram_dmma_bitwise(m, c, oracle):
    import paper_1401_2720_b200 as J

    rng = np.random.default_rng(m + c)
    a = np.asfortranarray(rng.standard_normal((m, c)) * np.logspace(0, -6, c))
    h = J.gram(a)
    assert np.array_equal(h, oracle.gram(a))


@pytest.mark.parametrize("m,c", [(4096, 1024), (1001, 67), (5, 4), (16384, 128)])
def test_postmultiply_dmma_bitwise(m, c, oracle):
    import paper_1401_2720_b200 as J

    rng = np.random.default_rng(7 * m + c)
    a = np.asfortranarray(rng.standard_normal((m, c)))
    v = np.asfortranarray(rng.standard_normal((c, c)))
    assert np.array_equal(J.postmultiply(a, v), oracle.postmultiply(a, v))


@pytest.mark.parametrize("c", [1024, 700, 64, 65, 129, 2])
def test_blocked_cholesky_bitwise(c, oracle):
    import paper_1401_2720_b200 as J

    rng = np.random.default_rng(c)
    b = rng.standard_normal((c + 8, c)) * np.logspace(0, -3, c)
    h = oracle.gram(np.asfortranarray(b))
    assert np.array_equal(J.cholesky_in_place(h), oracle.cholesky_in_place(h))


@pytest.mark.parametrize("bad", [151, 1, 64, 65, 200])
def test_blocked_cholesky_reports_first_bad_pivot(bad, oracle):
    import paper_1401_2720_b200 as J

    c = 200
    rng = np.random.default_rng(3)
    b = rng.standard_normal((c + 4, c))
    h = np.asfortranarray(b.T @ b)
    h[bad - 1, bad - 1] = -1.0  # this pivot (and no earlier one) is nonpositive
    if bad < c:
        h[c - 1, c - 1] = -5.0  # a later bad pivot must not be reported
    with pytest.raises(oracle.OracleError) as eo:
        oracle.cholesky_in_place(h)
    with pytest.raises(J.RankDeficiencyError) as ei:
        J.cholesky_in_place(h)
    assert ei.value.index == eo.value.index == bad


def test_outer_step_contractions_at_g8_size(oracle):
    """One outer step's worth at n = 16384, g = 8 in miniature rows: the
    m x 2048 Gram, its Cholesky and the tall update, against the oracle."""
    import torch

    from paper_1401_2720_b200 import _lib

    lib = _lib.require_cuda()
    m, c = 2048, 2048
    rng = np.random.default_rng(11)
    a = np.asfortranarray(rng.standard_normal((m + 64, c)))
    A = _dev(a)
    H = torch.empty((c, c), dtype=torch.float64, device="cuda")
    _lib.check(lib.jh_gram(A.data_ptr(), m + 64, m + 64, c, H.data_ptr(),
                           _lib.stream_handle()), "gram")
    R = torch.empty_like(H)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.jh_cholesky(H.data_ptr(), c, R.data_ptr(), info.data_ptr(),
                               _lib.stream_handle()), "cholesky")
    assert int(info.item()) == 0
    h_or = oracle.gram(a)
    r_or = oracle.cholesky_in_place(h_or)
    assert np.array_equal(R.cpu().numpy().T, r_or)
