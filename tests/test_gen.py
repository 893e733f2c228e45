"""The butterfly input generator: the GPU kernel (jh_gen_butterfly) is
bitwise its host twin (oracle/gen_butterfly.c), whose output has the
prescribed (hyperbolic) singular values.  This equality is what lets the
offline whole-solve oracle goldens (tests/golden/offline) stand for the
matrices the bench solves."""

import numpy as np
import pytest

from paper_1401_2720_b200 import workloads as WL


def _hsv(g, n_plus):
    """Hyperbolic singular values: sqrt|eig(G J G^T)| per class."""
    n = g.shape[1]
    j = np.concatenate((np.ones(n_plus), -np.ones(n - n_plus)))
    lam = np.linalg.eigvals((g * j) @ g.T).real if g.shape[0] == n else None
    return lam


def test_host_generator_spectrum(oracle):
    wl = WL.scaled(WL.CONFIG3, 256)
    sigma, n_plus = wl.sigma_nplus()
    g = oracle.gen_butterfly(sigma, n_plus=n_plus, seed=wl.gen_seed)
    s = np.linalg.svd(g, compute_uv=False)
    assert np.max(np.abs(s - np.sort(sigma)[::-1]) / np.sort(sigma)[::-1]) < 1e-13
    assert np.count_nonzero(g) == g.size  # dense mixing


def test_host_generator_tall_and_hyperbolic(oracle):
    wl = WL.scaled(WL.CONFIG5, 64, 512)
    sigma, _ = wl.sigma_nplus()
    g = oracle.gen_butterfly(sigma, m=512, seed=wl.gen_seed)
    s = np.linalg.svd(g, compute_uv=False)
    ref = np.sort(sigma)[::-1]
    assert np.max(np.abs(s - ref) / ref) < 1e-13
    wl4 = WL.scaled(WL.CONFIG4, 128)
    sigma, n_plus = wl4.sigma_nplus()
    assert n_plus == 64
    g = oracle.gen_butterfly(sigma, n_plus=n_plus, seed=wl4.gen_seed)
    lam = np.sort(_hsv(g, n_plus))
    want = np.sort(np.concatenate((sigma[:n_plus] ** 2, -sigma[n_plus:] ** 2)))
    assert np.max(np.abs(lam - want) / np.abs(want)) < 1e-8


def test_host_generator_rejects_bad_shapes(oracle):
    with pytest.raises(ValueError):
        oracle.gen_butterfly(np.ones(12))
    with pytest.raises(ValueError):
        oracle.gen_butterfly(np.ones(16), n_plus=5)


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,m", [("config3", 1024, 1024), ("config4", 512, 512),
                                      ("config5", 256, 4096), ("config3", 16384, 16384)])
def test_gpu_generator_bitwise_host(oracle, name, n, m):
    from paper_1401_2720_b200 import testgen as T

    wl = WL.WORKLOADS[name]
    if n != wl.n:
        wl = WL.scaled(wl, n, m)
    gt, sigma, n_plus = T.workload_input_device(wl)
    host = oracle.gen_butterfly(sigma, m=wl.m, n_plus=n_plus, seed=wl.gen_seed,
                                passes=wl.passes, tanh_max=wl.tanh_max)
    assert np.array_equal(gt.cpu().numpy(), np.ascontiguousarray(host.T))
