"""Outer (multi-worker) level: legal mappings, the exchange protocol over a
real torch.distributed group (gloo, world size 2, CPU) and the
single-process simulation, checked bitwise against run_distributed goldens
from the reference (tests/golden/dist.*).  On the CPU the worker arithmetic
comes from the C oracle (an injected engine); on the GPU from the product
kernels."""

import hashlib
import os
import socket
import tempfile
from dataclasses import replace
from types import SimpleNamespace

import numpy as np
import pytest
import torch

import paper_1401_2720_b200 as J
from paper_1401_2720_b200 import distsim as D
from paper_1401_2720_b200 import strategy as S


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class OracleEngine:
    """Worker arithmetic from the C oracle, on column-major CPU tensors."""

    def __init__(self, m, n, local_n, cfg):
        from oracle import oracle as O

        self.O = O
        w = cfg.block_width
        self.local_cfg = replace(
            cfg, accumulate_v=not cfg.solve_v, solve_v=False,
            max_block_sweeps=1 if cfg.variant == "block-oriented" else cfg.max_block_sweeps)
        self.outer = S.as_table(S.make_strategy(cfg.outer_strategy, local_n // (w // 2)))
        self.inner = S.as_table(S.make_strategy(cfg.inner_strategy, w))

    def device(self):
        return torch.device("cpu")

    def gram_cholesky(self, gx):
        h = self.O.gram(gx.numpy().T)
        r = self.O.cholesky_in_place(h)
        return torch.from_numpy(np.ascontiguousarray(r.T))

    def nested(self, work, vhat, n_plus):
        return self.O.run_block_jacobi_inplace(
            work.numpy().T, None if vhat is None else vhat.numpy().T, n_plus, self.local_cfg,
            self.outer, self.inner)

    def nested_sweep(self, work, vhat, n_plus):
        return self.O.block_sweep(work.numpy().T, None if vhat is None else vhat.numpy().T,
                                  n_plus, self.local_cfg, self.outer, self.inner)

    def postmultiply(self, x, vhat):
        out = self.O.postmultiply(x.numpy().T, vhat.numpy().T)
        return torch.from_numpy(np.ascontiguousarray(out.T))

    def solve_for_v(self, r, work):
        out = self.O.solve_for_v(r.numpy().T, work.numpy().T)
        return torch.from_numpy(np.ascontiguousarray(out.T))

    def eye(self, k):
        return torch.eye(k, dtype=torch.float64)

    def finish(self, G, V, signature, stats, converged):
        g = G.numpy().T
        sigma = self.O.extract_sigma(g)
        u = g / sigma
        order = self.O.class_sort_order(sigma, signature.n_plus)
        return SimpleNamespace(sigma=sigma[order], u=u[:, order],
                               v=None if V is None else V.numpy().T[:, order],
                               stats=tuple(stats), block_sweeps=len(stats), converged=converged)


def _cfg(meta):
    return J.SolverConfig(block_width=meta["block_width"], variant=meta["variant"],
                          accumulate_v=meta["accumulate_v"])


@pytest.mark.parametrize("g", [2, 4, 8])
def test_legal_mapping_is_exchange_compatible(g):
    strat = S.make_strategy("rrow", 2 * g)
    m = D.legal_mapping(strat)
    ns = len(m.assignments)
    assert ns == 2 * g - 1
    for s in range(ns):
        assert sorted(m.assignments[s]) == sorted(tuple(sorted(p)) for p in strat.steps[s])
        assert D._moves(m.assignments[s], m.assignments[(s + 1) % ns]) is not None
        # one message in, one out per worker per step
        assert sorted(src for src, _ in m.moves[s]) == list(range(g))


def test_local_signature_pair():
    sig = J.Signature(16, 5)
    assert D.local_signature_pair(sig, 1, 3, 4).n_plus == 4
    assert D.local_signature_pair(sig, 2, 3, 4).n_plus == 1
    assert D.local_signature_pair(sig, 3, 4, 4).n_plus == 0


@pytest.mark.parametrize("name", ["g2_bo", "g4_bo", "g2_fb", "g4_fb", "g2_bo_nov"])
def test_simulated_workers_bitwise_vs_reference(name, dist_golden):
    meta, arrs = dist_golden
    m = meta[name]
    g = arrs["dist_in"]
    nplus = int((arrs["dist_lambda"] > 0).sum())
    n = g.shape[0]
    cfg = _cfg(m)
    eng = OracleEngine(n, n, n // m["g"], cfg)
    res, _ = D.run_distributed(g, J.Signature(n, nplus), m["g"], cfg, engine=eng,
                               backend="sim")
    assert [list(s) for s in res.stats] == m["stats"]
    assert _sha(res.sigma) == m["sigma_sha256"]
    if m["accumulate_v"]:
        assert np.array_equal(res.v, arrs[f"{name}_v"])


def test_hybrid_early_stop_close(dist_golden):
    meta, arrs = dist_golden
    g = arrs["dist_in"]
    lam = arrs["dist_lambda"]
    n = g.shape[0]
    nplus = int((lam > 0).sum())
    cfg = J.SolverConfig(block_width=16)
    eng = OracleEngine(n, n, n // 4, cfg)
    res, trace = D.run_distributed(g, J.Signature(n, nplus), 4, cfg, hybrid_early_stop=True,
                                   collect_trace=True, engine=eng, backend="sim")
    full = meta["g4_fb"]
    ref_sigma = arrs["g4_fb_sigma"]
    assert np.max(np.abs(res.sigma / ref_sigma - 1)) <= 1e-9
    assert res.converged
    assert len(trace) == 4 * 7 * res.block_sweeps
    assert full["converged"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, name, out_path):
    import torch.distributed as dist

    from tests.conftest import GOLDEN

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import json

        meta = json.loads((GOLDEN / "dist.json").read_text())[name]
        arrs = np.load(GOLDEN / "dist.npz")
        g = arrs["dist_in"]
        n = g.shape[0]
        nplus = int((arrs["dist_lambda"] > 0).sum())
        cfg = _cfg(meta)
        res, _ = D.run_distributed(g, J.Signature(n, nplus), world, cfg,
                                   engine=OracleEngine(n, n, n // world, cfg))
        if rank == 0:
            np.savez(out_path, sigma=res.sigma, v=res.v if res.v is not None else np.zeros(0),
                     stats=np.array(res.stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["g2_bo", "g2_fb"])
def test_gloo_two_ranks_bitwise_vs_reference(name, dist_golden):
    import torch.multiprocessing as mp

    meta, arrs = dist_golden
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "r0.npz")
        mp.spawn(_gloo_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
        r = np.load(out)
        assert [list(s) for s in r["stats"]] == meta[name]["stats"]
        assert _sha(r["sigma"]) == meta[name]["sigma_sha256"]
        assert np.array_equal(r["v"], arrs[f"{name}_v"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g2_bo", "g4_bo", "g2_fb", "g4_fb", "g2_bo_nov"])
def test_gpu_simulated_workers_bitwise_vs_reference(name, dist_golden):
    meta, arrs = dist_golden
    m = meta[name]
    g = arrs["dist_in"]
    nplus = int((arrs["dist_lambda"] > 0).sum())
    n = g.shape[0]
    res, _ = D.run_distributed(g, J.Signature(n, nplus), m["g"], _cfg(m), backend="sim")
    assert [list(s) for s in res.stats] == m["stats"]
    assert _sha(res.sigma) == m["sigma_sha256"]
    if m["accumulate_v"]:
        assert np.array_equal(res.v, arrs[f"{name}_v"])


# ---------------------------------------------------------------------------
# the per-rank (non-simulated) path with ranks as threads (tests/comm_threads.py)


@pytest.mark.parametrize("name", ["g2_bo", "g2_fb"])
def test_thread_ranks_bitwise_vs_reference_cpu(name, dist_golden):
    from tests.comm_threads import run_ranks

    meta, arrs = dist_golden
    m = meta[name]
    g = arrs["dist_in"]
    n = g.shape[0]
    nplus = int((arrs["dist_lambda"] > 0).sum())
    cfg = _cfg(m)
    res = run_ranks(m["g"], lambda i, pg: D.run_distributed(
        g, J.Signature(n, nplus), m["g"], cfg, engine=OracleEngine(n, n, n // m["g"], cfg),
        process_group=pg)[0], backend="gloo")
    for r in res:
        assert [list(s) for s in r.stats] == m["stats"]
        assert _sha(r.sigma) == m["sigma_sha256"]
        assert np.array_equal(r.v, arrs[f"{name}_v"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g2_bo", "g4_fb", "g2_bo_nov"])
def test_gpu_thread_ranks_device_exchange_vs_reference(name, dist_golden):
    """run_distributed's per-rank path (device send/receive of the block
    pairs, all-reduces, all-gather) with CUDA tensors, g ranks as threads on
    cuda:0, bitwise against the reference goldens."""
    from tests.comm_threads import run_ranks

    meta, arrs = dist_golden
    m = meta[name]
    g = arrs["dist_in"]
    n = g.shape[0]
    nplus = int((arrs["dist_lambda"] > 0).sum())
    cfg = _cfg(m)

    def rank(i, pg):
        r, _ = D.run_distributed(g, J.Signature(n, nplus), m["g"], cfg, process_group=pg)
        torch.cuda.synchronize()
        return r

    for r in run_ranks(m["g"], rank, backend="nccl"):
        assert [list(s) for s in r.stats] == m["stats"]
        assert _sha(r.sigma) == m["sigma_sha256"]
        if m["accumulate_v"]:
            assert np.array_equal(r.v, arrs[f"{name}_v"])
