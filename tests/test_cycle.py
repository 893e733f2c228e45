"""Cycle engine (csrc/jh_cycle.cu): plan structure on the host (CPU tests)
and bitwise equality with the per-p-step kernels and the C oracle on the
GPU, for whole sweeps, partial p-step ranges, tall factors, HSVD signatures
and solves without V."""

import ctypes

import numpy as np
import pytest

from paper_1401_2720_b200 import _lib
from paper_1401_2720_b200.strategy import as_table, make_strategy


def _plan(kind, b):
    lib = _lib.load_library()
    table = np.ascontiguousarray(np.array(as_table(make_strategy(kind, b)), dtype=np.int32))
    nints = int(lib.jh_cycle_plan_ints(b))
    if nints <= 0:
        return table, None
    plan = np.full(nints, -7, dtype=np.int32)
    rc = lib.jh_cycle_plan(table.ctypes.data_as(ctypes.c_void_p), b, plan.ctypes.data_as(ctypes.c_void_p))
    return table, (plan if rc == 0 else None)


@pytest.mark.parametrize("kind,b", [("rrow", 4), ("rrow", 8), ("rrow", 16), ("rrow", 64),
                                    ("rrow", 1024), ("rcol", 16), ("rcol", 64)])
def test_plan_covers_every_boundary(kind, b):
    table, plan = _plan(kind, b)
    if kind == "rcol" and plan is None:
        pytest.skip("rcol has no 4-cycle structure at this order")
    assert plan is not None, f"{kind}({b}) should have the 4-cycle structure"
    S, T = b - 1, b // 2
    nc = T // 2
    cyc = plan[: S * nc * 8].reshape(S, nc, 8)
    tpos = plan[S * nc * 8: S * nc * 8 + S * T].reshape(S, T)
    upos = plan[S * nc * 8 + S * T:].reshape(S, T)
    for s in range(S):
        sp = (s - 1) % S
        ts = sorted(np.concatenate([cyc[s, :, 0], cyc[s, :, 1]]).tolist())
        us = sorted(np.concatenate([cyc[s, :, 2], cyc[s, :, 3]]).tolist())
        assert ts == list(range(T)) and us == list(range(T))
        for c in range(nc):
            t1, t2, u1, u2, i1, j1, i2, j2 = cyc[s, c]
            blocks = [*table[sp, t1], *table[sp, t2]]
            assert sorted(blocks) == sorted([*table[s, u1], *table[s, u2]])
            assert (blocks[i1], blocks[j1]) == tuple(table[s, u1])
            assert (blocks[i2], blocks[j2]) == tuple(table[s, u2])
            assert tpos[sp, t1] == 2 * c and tpos[sp, t2] == 2 * c + 1
            assert upos[s, u1] == 2 * c and upos[s, u2] == 2 * c + 1


def test_plan_rejects_tables_without_cycles():
    # modified modulus pairs block-columns in long cycles across p-steps
    _, plan = _plan("mm", 32)
    assert plan is None


# ---------------------------------------------------------------------------
# GPU: the cycle engine against the per-p-step kernels (same device code per
# entry, bitwise) and the C oracle


def _engines(m, n, nv, w, kind, n_plus, variant="full-block", engine=2):
    from paper_1401_2720_b200.driver import SolverConfig, SweepEngine

    cfg = SolverConfig(block_width=w, variant=variant, outer_strategy=kind)
    outer = make_strategy(kind, n // (w // 2))
    inner = make_strategy("rrow", w)
    eng = SweepEngine(m, n, nv, cfg, outer, inner, n_plus, engine=engine)
    ref = SweepEngine(m, n, nv, cfg, outer, inner, n_plus, engine=0)  # per-p-step kernels
    return eng, ref


def _graded(m, n, seed, kappa=1e6):
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((m, n))
    b /= np.linalg.norm(b, axis=0)
    return b * np.logspace(0, -np.log10(kappa), n)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [1, 2])
@pytest.mark.parametrize("m,n,first,count,with_v,n_plus", [
    (256, 256, 0, None, True, 256),     # whole sweep (15 p-steps, odd)
    (512, 512, 0, None, True, 512),     # 31 p-steps
    (1024, 1024, 0, None, True, 1024),
    (512, 512, 3, 6, True, 512),        # partial range, even count
    (512, 512, 10, 7, True, 512),       # partial range, odd count
    (512, 512, 30, 1, True, 512),       # last p-step only
    (768, 512, 0, None, True, 512),     # tall factor
    (512, 512, 0, None, False, 512),    # no V
    (512, 512, 0, None, True, 256),     # hyperbolic (J signature)
    (4096, 256, 0, None, True, 256),    # long rows: many chunks per item
    (2050, 512, 0, None, True, 512),    # m not a multiple of the chunk
    (1024, 1024, 0, None, True, 1024),  # V in two row slabs, odd p-step count
    (4096, 4096, 0, 9, True, 4096),     # many V slabs, odd count
])
def test_engine_sweep_bitwise_vs_pstep_kernels(m, n, first, count, with_v, n_plus, engine):
    import torch

    torch.cuda.set_device(0)
    nv = n if with_v else 0
    eng, ref = _engines(m, n, nv, 32, "rrow", n_plus, engine=engine)
    assert eng.plan_dev is not None and ref.engine == 0
    g = torch.from_numpy(_graded(m, n, 11 + m + n)).cuda()
    G1 = g.t().contiguous()
    G2 = G1.clone()
    V1 = torch.eye(n, dtype=torch.float64, device="cuda") if with_v else None
    V2 = V1.clone() if with_v else None
    for _ in range(2):  # two sweeps: the second starts from rotated data
        c1 = eng.sweep(G1, V1, first, count).clone()
        c2 = ref.sweep(G2, V2, first, count).clone()
        torch.cuda.synchronize()
        assert c1.tolist() == c2.tolist()
        assert torch.equal(G1, G2)
        if with_v:
            assert torch.equal(V1, V2)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["1", "2"])
@pytest.mark.parametrize("variant", ["full-block", "block-oriented"])
def test_engine_solve_bitwise_vs_oracle(variant, engine, oracle, monkeypatch):
    import torch

    import paper_1401_2720_b200 as J

    torch.cuda.set_device(0)
    monkeypatch.setenv("JHSVD_ENGINE", engine)
    n = 512
    g = np.asfortranarray(_graded(n, n, 5, 1e10))
    cfg = J.SolverConfig(block_width=32, variant=variant)
    res = J.block_jacobi(g, None, cfg)
    outer = J.as_table(J.make_strategy("rrow", n // 16))
    inner = J.as_table(J.make_strategy("rrow", 32))
    ref = oracle.block_jacobi(g, n, cfg, outer, inner)
    assert res.stats == ref.stats
    assert np.array_equal(res.sigma, ref.sigma)
    assert np.array_equal(res.u, ref.u) and np.array_equal(res.v, ref.v)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [1, 2])
def test_engine_reports_first_failure_like_pstep_path(engine):
    """A rank-deficient pair fails in the same (p-step, task, status, index)
    on both paths (the error key is the minimum in the reference order)."""
    import torch

    torch.cuda.set_device(0)
    n = 256
    a = _graded(n, n, 3)
    a[:, 37] = 0.0  # a zero column: the Cholesky of its first pair breaks down
    eng, ref = _engines(n, n, n, 32, "rrow", n, engine=engine)
    G1 = torch.from_numpy(a).cuda().t().contiguous()
    G2 = G1.clone()
    V1 = torch.eye(n, dtype=torch.float64, device="cuda")
    V2 = V1.clone()
    k1 = eng.sweep(G1, V1).clone().tolist()
    k2 = ref.sweep(G2, V2).clone().tolist()
    assert k1[2] == k2[2] and k1[2] != -1


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8192, 12288, 16384])
def test_large_prefix_bitwise_vs_oracle(n, oracle):
    """The first p-steps at sizes whose Gram ring shape (3 or 4 CTAs per SM),
    row slabs (4096 / 1536 rows) and mixed launch differ from the small
    cases: G and V bitwise equal to the C oracle."""
    import torch

    from paper_1401_2720_b200.driver import SolverConfig, SweepEngine

    torch.cuda.set_device(0)
    w, steps = 32, 3
    cfg = SolverConfig(block_width=w)
    outer = make_strategy("rrow", n // (w // 2))
    inner = make_strategy("rrow", w)
    gen = torch.Generator(device="cuda").manual_seed(n)
    G = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)  # rows = columns
    host = G.cpu().numpy()
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    eng = SweepEngine(n, n, n, cfg, outer, inner, n)
    eng.sweep(G, V, 0, steps)
    torch.cuda.synchronize()
    g = np.array(host, copy=True).T  # F-order m x n
    v = np.asfortranarray(np.eye(n))
    oracle.block_sweep(g, v, n, dict(block_width=w, variant="full-block"),
                       as_table(outer)[:steps], as_table(inner), threads=oracle.max_threads())
    assert np.array_equal(G.cpu().numpy(), np.ascontiguousarray(g.T))
    assert np.array_equal(V.cpu().numpy(), np.ascontiguousarray(v.T))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,steps", [(1000, 512, 5), (2050, 1024, 4)])
def test_ragged_rows_prefix_bitwise_vs_oracle(m, n, steps, oracle):
    """Row counts that are not multiples of the 104/128-row chunks or of the
    row slabs: the first p-steps of the default engine against the C oracle."""
    import torch

    from paper_1401_2720_b200.driver import SolverConfig, SweepEngine

    torch.cuda.set_device(0)
    w = 32
    cfg = SolverConfig(block_width=w)
    outer = make_strategy("rrow", n // (w // 2))
    inner = make_strategy("rrow", w)
    gen = torch.Generator(device="cuda").manual_seed(m + n)
    G = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=gen)  # rows = columns
    host = G.cpu().numpy()
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    eng = SweepEngine(m, n, n, cfg, outer, inner, n)
    eng.sweep(G, V, 0, steps)
    torch.cuda.synchronize()
    g = np.array(host, copy=True).T  # F-order m x n
    v = np.asfortranarray(np.eye(n))
    oracle.block_sweep(g, v, n, dict(block_width=w, variant="full-block"),
                       as_table(outer)[:steps], as_table(inner), threads=oracle.max_threads())
    assert np.array_equal(G.cpu().numpy(), np.ascontiguousarray(g.T))
    assert np.array_equal(V.cpu().numpy(), np.ascontiguousarray(v.T))


@pytest.mark.gpu
def test_full_solve_4096_bitwise_vs_oracle(oracle):
    """A whole solve at n = 4096 (128 tasks per p-step: the 2-per-SM Gram
    ring, short slabs, the Grams of the next p-step inside the update
    launch) bitwise equal to the C oracle: stats, sigma, U and V."""
    import torch

    import paper_1401_2720_b200 as J

    torch.cuda.set_device(0)
    n = 4096
    rng = np.random.default_rng(11)
    g = np.asfortranarray(rng.standard_normal((n, n)))
    cfg = J.SolverConfig(block_width=32)
    res = J.block_jacobi(g, None, cfg)
    outer = J.as_table(J.make_strategy("rrow", n // 16))
    inner = J.as_table(J.make_strategy("rrow", 32))
    ref = oracle.block_jacobi(g, n, cfg, outer, inner, threads=oracle.max_threads())
    assert res.stats == ref.stats
    assert np.array_equal(res.sigma, ref.sigma)
    assert np.array_equal(res.u, ref.u) and np.array_equal(res.v, ref.v)
