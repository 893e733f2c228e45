"""Engine 1 (csrc/jh_vpair.cu, V updated once per two p-steps over the
4-cycles of the pivot table): the cycle plan on the host (CPU tests) and
bitwise equality with the per-p-step kernels (engine 0) and the C oracle on
the GPU, for whole sweeps, partial p-step ranges, tall factors, HSVD
signatures and solves without V."""

import ctypes

import numpy as np
import pytest

from paper_1401_2720_b200 import _lib
from paper_1401_2720_b200.strategy import as_table, make_strategy


def _plan(kind, b, table=None):
    lib = _lib.load_library()
    if table is None:
        table = np.ascontiguousarray(np.array(as_table(make_strategy(kind, b)), dtype=np.int32))
    steps = table.shape[0]
    nints = int(lib.jh_cycle_plan_ints(b, steps))
    if nints <= 0:
        return table, None
    plan = np.full(nints, -7, dtype=np.int32)
    rc = lib.jh_cycle_plan(table.ctypes.data_as(ctypes.c_void_p), b, steps,
                           plan.ctypes.data_as(ctypes.c_void_p))
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
    for s in range(S):  # boundary s joins p-steps s-1 and s (0: the wrap)
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


def test_plan_of_a_table_segment():
    """Sub-tables (consecutive p-steps of a sweep, as the sharded solve runs
    them) keep the structure; boundary 0 is not needed."""
    table = np.ascontiguousarray(np.array(as_table(make_strategy("rrow", 64)), dtype=np.int32))
    for lo, hi in ((0, 7), (31, 63), (5, 6)):
        seg = np.ascontiguousarray(table[lo:hi])
        _, plan = _plan("rrow", 64, seg)
        assert plan is not None, (lo, hi)
        # boundary 0 groups the last p-step's tasks into disjoint pairs
        t = plan[: 16 * 8].reshape(16, 8)[:, :2]
        assert sorted(t.ravel().tolist()) == list(range(32))


# ---------------------------------------------------------------------------
# GPU: the cycle engine against the per-p-step kernels (same device code per
# entry, bitwise) and the C oracle


def _engines(m, n, nv, w, kind, n_plus, variant="full-block", engine=1):
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
@pytest.mark.parametrize("engine", [1])
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
    assert ref.engine == 0
    assert (eng.engine == 1) == with_v
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
@pytest.mark.parametrize("variant", ["full-block", "block-oriented"])
def test_engine_solve_bitwise_vs_oracle(variant, oracle):
    import torch

    import paper_1401_2720_b200 as J

    torch.cuda.set_device(0)
    n = 512
    g = np.asfortranarray(_graded(n, n, 5, 1e10))
    cfg = J.SolverConfig(block_width=32, variant=variant)
    solver = J.Solver(n, cfg)
    assert solver.engine.engine == 1
    res = J.block_jacobi(g, None, cfg)
    outer = J.as_table(J.make_strategy("rrow", n // 16))
    inner = J.as_table(J.make_strategy("rrow", 32))
    ref = oracle.block_jacobi(g, n, cfg, outer, inner)
    assert res.stats == ref.stats
    assert np.array_equal(res.sigma, ref.sigma)
    assert np.array_equal(res.u, ref.u) and np.array_equal(res.v, ref.v)
