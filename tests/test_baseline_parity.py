"""Whole-solve parity on the BASELINE.json workloads at their full sizes.

* config 3 (16384^2, full-block, rrow, w = 32): the GPU solve of the bench's
  input is bitwise the C oracle's offline whole solve of the same bytes
  (tests/golden/offline/config3.json, tools/oracle_offline.py): input sha256,
  per-sweep statistics, sigma, U, V.
* config 4 (8192^2 HSVD, n/2 negative): the same against
  tests/golden/offline/config4.json.
* config 2 (4096^2 column-graded, kappa = 1e12, block-oriented): the whole
  solve against the C oracle run here on the host cores.
* config 5 (131072 x 8192): the same against tests/golden/offline/config5.json,
  and the first p-steps of sweep 1, G and V bitwise against the oracle run
  in the test.
* hybrid early stop of the three-level outer level with the product kernels
  against the same rule on oracle workers.
The C oracle (oracle/) is the checker; the product path never calls it.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1401_2720_b200 as J
from paper_1401_2720_b200 import workloads as WL

OFFLINE = Path(__file__).resolve().parent / "golden" / "offline"

pytestmark = pytest.mark.gpu


def _sha(t):
    a = t.cpu().numpy() if hasattr(t, "cpu") else t
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _offline(name):
    p = OFFLINE / f"{name}.json"
    if not p.exists():
        pytest.fail(f"missing offline oracle golden {p} (tools/oracle_offline.py {name})")
    return json.loads(p.read_text())


@pytest.mark.parametrize("name", ["config3", "config4", "config5"])
def test_whole_solve_bitwise_vs_offline_oracle(name):
    import torch

    from paper_1401_2720_b200 import testgen as T

    gold = _offline(name)
    wl = WL.WORKLOADS[name]
    G0, _, n_plus = T.workload_input_device(wl)
    assert _sha(G0) == gold["input_sha256"]
    solver = J.Solver(wl.n, J.SolverConfig(**wl.solver_kwargs()), J.Signature(wl.n, n_plus),
                      m=wl.m)
    sigma, U, V, stats, conv = solver.solve_device(G0)
    torch.cuda.synchronize()
    assert [list(s) for s in stats] == gold["stats"]
    assert conv == gold["converged"]
    assert _sha(sigma) == gold["sigma_sha256"]
    assert _sha(U) == gold["u_sha256"]
    assert _sha(V) == gold["v_sha256"]


def test_config2_whole_solve_bitwise_vs_oracle(oracle):
    n = 4096
    rng = np.random.default_rng(2)
    b = rng.standard_normal((n, n))
    b /= np.linalg.norm(b, axis=0)
    g = np.asfortranarray(b * np.logspace(0, -12, n))  # column-graded, kappa 1e12
    cfg = J.SolverConfig(block_width=32, variant="block-oriented")
    res = J.block_jacobi(g, None, cfg)
    outer = J.as_table(J.make_strategy("rrow", n // 16))
    inner = J.as_table(J.make_strategy("rrow", 32))
    ref = oracle.block_jacobi(g, n, cfg, outer, inner)
    assert res.stats == ref.stats
    assert np.array_equal(res.sigma, ref.sigma)
    assert np.array_equal(res.u, ref.u) and np.array_equal(res.v, ref.v)
    assert res.sigma.max() / res.sigma.min() > 1e11


def test_config5_prefix_bitwise_vs_oracle(oracle):
    import torch

    from paper_1401_2720_b200 import testgen as T
    from paper_1401_2720_b200.driver import SweepEngine

    wl = WL.CONFIG5
    m, n, w = wl.m, wl.n, wl.block_width
    G0, _, n_plus = T.workload_input_device(wl)
    cfg = J.SolverConfig(**wl.solver_kwargs())
    outer = J.make_strategy(wl.strategy, n // (w // 2))
    inner = J.make_strategy(wl.strategy, w)
    k = 3
    eng = SweepEngine(m, n, n, cfg, outer, inner, n_plus)
    V = torch.eye(n, dtype=torch.float64, device="cuda")
    G = G0.clone()
    c = eng.sweep(G, V, 0, k).cpu().tolist()
    g_or = np.array(G0.cpu().numpy().T, order="F")
    del G0
    v_or = np.asfortranarray(np.eye(n))
    rot, proper = oracle.block_sweep(g_or, v_or, n_plus, cfg, J.as_table(outer), J.as_table(inner),
                                     nsteps=k)
    assert (c[0], c[1]) == (rot, proper)
    assert np.array_equal(G.cpu().numpy(), np.ascontiguousarray(g_or.T))
    assert np.array_equal(V.cpu().numpy(), np.ascontiguousarray(v_or.T))


@pytest.mark.parametrize("g", [2, 4])
def test_hybrid_early_stop_gpu_vs_oracle_workers(g, dist_golden):
    from paper_1401_2720_b200 import distsim as D
    from tests.test_distributed import OracleEngine

    _, arrs = dist_golden
    a = arrs["dist_in"]
    n = a.shape[0]
    nplus = int((arrs["dist_lambda"] > 0).sum())
    cfg = J.SolverConfig(block_width=16)
    ref, rtrace = D.run_distributed(a, J.Signature(n, nplus), g, cfg, hybrid_early_stop=True,
                                    collect_trace=True, engine=OracleEngine(n, n, n // g, cfg),
                                    backend="sim")
    res, trace = D.run_distributed(a, J.Signature(n, nplus), g, cfg, hybrid_early_stop=True,
                                   collect_trace=True, backend="sim")
    assert res.stats == ref.stats
    assert np.array_equal(res.sigma, ref.sigma)
    assert np.array_equal(res.v, ref.v)
    assert trace == rtrace
