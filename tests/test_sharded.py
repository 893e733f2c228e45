"""Block-column sharding (sharded.py): the segment plan of the pivot table,
and the sharded solve bitwise equal to the single-GPU solve -- on the CPU
with the C oracle as each worker's arithmetic (simulated workers and two
real gloo ranks), on the GPU with the product kernels (simulated workers:
the exchanges are the only difference between 1 and g GPUs)."""

import os
import socket
import tempfile
from types import SimpleNamespace

import numpy as np
import pytest
import torch

import paper_1401_2720_b200 as J
from paper_1401_2720_b200 import sharded as SH
from paper_1401_2720_b200 import strategy as S


class OracleShardEngine:
    """A worker's sweeps from the C oracle on column-major CPU tensors."""

    def __init__(self, cfg, n_plus):
        from oracle import oracle as O

        self.O = O
        self.cfg = cfg
        self.n_plus = n_plus
        self.inner = S.as_table(S.make_strategy(cfg.inner_strategy, cfg.block_width))
        self.dev = torch.device("cpu")

    def zeros_counters(self):
        return [0, 0, -1, 0]

    def sweep(self, loc, key, table, gblock, counters):
        errs = []
        v = None if loc.V is None else loc.V.numpy().T
        rot, proper = self.O.block_sweep(loc.G.numpy().T, v, self.n_plus, self.cfg, table,
                                         self.inner, gblock=gblock, err_out=errs)
        counters[0] += rot
        counters[1] += proper
        if errs:
            st, idx, ps, task = errs[0]
            counters[2] = (ps << 38) | (task << 16) | (st << 13) | idx

    def read(self, counters):
        return list(counters)

    def finish(self, G, V, signature, stats, converged):
        g = G.numpy().T
        sigma = self.O.extract_sigma(g)
        u = g / sigma
        order = self.O.class_sort_order(sigma, signature.n_plus)
        return SimpleNamespace(sigma=sigma[order], u=u[:, order],
                               v=None if V is None else V.numpy().T[:, order],
                               stats=tuple(stats), block_sweeps=len(stats), converged=converged)


def _problem(n, seed, kappa=1e4):
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((n, n))
    b /= np.linalg.norm(b, axis=0)
    return np.asfortranarray(b * np.logspace(0, -np.log10(kappa), n))


def _oracle_solve(g, n_plus, cfg):
    from oracle import oracle as O

    n = g.shape[1]
    outer = S.as_table(S.make_strategy(cfg.outer_strategy, n // (cfg.block_width // 2)))
    inner = S.as_table(S.make_strategy(cfg.inner_strategy, cfg.block_width))
    return O.block_jacobi(g, n_plus, cfg, outer, inner)


@pytest.mark.parametrize("b,g", [(64, 2), (64, 4), (64, 8), (1024, 8), (512, 2), (16, 1)])
def test_plan_segments_cover_the_sweep(b, g):
    plan = SH.shard_plan(S.make_strategy("rrow", b), g)
    seen = 0
    for seg in plan.segments:
        assert seg.first == seen
        seen += seg.nsteps
        for i in range(g):
            slots = list(plan.held(seg.config, i))
            loc, gidx = SH._local_table(plan, seg, slots)
            assert loc.shape == (seg.nsteps, b // (2 * g), 2)
            # local pairs map back to the global pairs of their steps
            gb = SH._gblock(plan, slots)
            for s in range(seg.nsteps):
                glob = plan.table[seg.first + s][gidx[s]]
                assert np.array_equal(gb[loc[s]], glob)
    assert seen == b - 1
    if g > 1:
        assert sum(seg.cross for seg in plan.segments) == 2 * g - 1
        # every exchange keeps one super-column per worker
        assert plan.mapping.fast_exchanges == 2 * g - 1


def test_tables_without_the_structure_are_rejected():
    with pytest.raises(SH.ShardingError):
        SH.shard_plan(S.make_strategy("mm", 64), 2)
    with pytest.raises(SH.ShardingError):
        SH.shard_plan(S.make_strategy("rrow", 12), 4)


@pytest.mark.parametrize("g,n,w,nplus", [(2, 128, 8, 128), (4, 128, 8, 128), (4, 128, 8, 61),
                                         (8, 128, 8, 64)])
def test_sim_workers_bitwise_vs_single_solve_cpu(g, n, w, nplus):
    cfg = J.SolverConfig(block_width=w)
    a = _problem(n, g * n + nplus)
    ref = _oracle_solve(a, nplus, cfg)
    res = SH.block_jacobi_sharded(a, J.Signature(n, nplus), g, cfg, backend="sim",
                                  engine=OracleShardEngine(cfg, nplus))
    assert res.stats == ref.stats
    assert np.array_equal(res.sigma, ref.sigma)
    assert np.array_equal(res.v, ref.v)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, nplus = 128, 70
        cfg = J.SolverConfig(block_width=8)
        a = _problem(n, 5)
        res = SH.block_jacobi_sharded(a, J.Signature(n, nplus), world, cfg,
                                      engine=OracleShardEngine(cfg, nplus))
        if rank == 0:
            np.savez(out_path, sigma=res.sigma, v=res.v, stats=np.array(res.stats))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_bitwise_vs_single_solve():
    import torch.multiprocessing as mp

    cfg = J.SolverConfig(block_width=8)
    ref = _oracle_solve(_problem(128, 5), 70, cfg)
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "r0.npz")
        mp.spawn(_gloo_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        r = np.load(out)
        assert [tuple(s) for s in r["stats"]] == list(ref.stats)
        assert np.array_equal(r["sigma"], ref.sigma)
        assert np.array_equal(r["v"], ref.v)


# ---------------------------------------------------------------------------
# GPU


@pytest.mark.gpu
@pytest.mark.parametrize("g,n,m,nplus,variant", [
    (2, 1024, 1024, 1024, "full-block"), (4, 1024, 1024, 1024, "full-block"),
    (8, 1024, 1024, 1024, "full-block"), (8, 1024, 1024, 512, "full-block"),
    (4, 512, 512, 301, "block-oriented"), (2, 512, 2048, 512, "full-block")])
def test_gpu_sim_workers_bitwise_vs_block_jacobi(g, n, m, nplus, variant):
    cfg = J.SolverConfig(block_width=32, variant=variant)
    rng = np.random.default_rng(n + g)
    a = rng.standard_normal((m, n))
    a /= np.linalg.norm(a, axis=0)
    a = np.asfortranarray(a * np.logspace(0, -5, n))
    ref = J.block_jacobi(a, J.Signature(n, nplus), cfg, allow_tall=m > n)
    res = SH.block_jacobi_sharded(a, J.Signature(n, nplus), g, cfg, backend="sim",
                                  allow_tall=m > n)
    assert res.stats == ref.stats
    assert np.array_equal(res.sigma, ref.sigma)
    assert np.array_equal(res.u, ref.u)
    assert np.array_equal(res.v, ref.v)


# ---------------------------------------------------------------------------
# the non-simulated (per-rank) path with ranks as threads (tests/comm_threads.py)


@pytest.mark.parametrize("g,nplus", [(2, 128), (4, 61)])
def test_thread_ranks_bitwise_vs_single_solve_cpu(g, nplus):
    from tests.comm_threads import run_ranks

    n, cfg = 128, J.SolverConfig(block_width=8)
    a = _problem(n, 7 * g + nplus)
    ref = _oracle_solve(a, nplus, cfg)
    res = run_ranks(g, lambda i, pg: SH.block_jacobi_sharded(
        a, J.Signature(n, nplus), g, cfg, engine=OracleShardEngine(cfg, nplus),
        process_group=pg), backend="gloo")
    for r in res:
        assert r.stats == ref.stats
        assert np.array_equal(r.sigma, ref.sigma)
        assert np.array_equal(r.v, ref.v)


@pytest.mark.gpu
@pytest.mark.parametrize("g,n,nplus", [(2, 1024, 1024), (4, 1024, 600), (8, 2048, 2048)])
def test_gpu_thread_ranks_device_exchange_bitwise(g, n, nplus):
    """The per-rank path of an NCCL job (send/receive of CUDA super-columns
    into the staging buffers, counter all-reduces, the final all-gather)
    with g ranks as threads on cuda:0: bitwise block_jacobi."""
    from tests.comm_threads import run_ranks

    cfg = J.SolverConfig(block_width=32)
    rng = np.random.default_rng(n + g)
    a = rng.standard_normal((n, n))
    a /= np.linalg.norm(a, axis=0)
    a = np.asfortranarray(a * np.logspace(0, -5, n))
    ref = J.block_jacobi(a, J.Signature(n, nplus), cfg)
    A = torch.from_numpy(a).cuda()

    def rank(i, pg):
        r = SH.block_jacobi_sharded(A, J.Signature(n, nplus), g, cfg, process_group=pg)
        torch.cuda.synchronize()
        return r

    def np_(x):
        return x.cpu().numpy() if isinstance(x, torch.Tensor) else x

    res = run_ranks(g, rank, backend="nccl")
    for r in res:
        assert r.stats == ref.stats
        assert np.array_equal(np_(r.sigma), ref.sigma)
        assert np.array_equal(np_(r.u), ref.u)
        assert np.array_equal(np_(r.v), ref.v)
