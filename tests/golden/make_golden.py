"""Generate golden fixtures by running the REFERENCE `jhsvd` package.

This script is test infrastructure.  It imports the reference Python package
(pure Python + numba) from a writable copy of `/root/reference/pkg` and dumps
its outputs on seeded inputs into `tests/golden/`:

* ``strategies.json`` -- sha256 of ``dump_strategy(make_strategy(kind, n))``
  for every kind and many orders, plus the full text for small orders
  (reference: strategy.py:477-548).
* ``kernels.npz`` -- per-kernel input/output vectors for ``gram``,
  ``cholesky_in_place``, ``inner_jacobi``, ``postmultiply``, ``qr_peeloff``,
  ``solve_for_v`` and ``norm2`` (reference: blockkernel.py, driver.py,
  robustnorm.py).
* ``solves.npz`` + ``solves.json`` -- end-to-end ``block_jacobi`` runs
  (input matrix, sigma, U, V, stats) for small configurations, including
  the BASELINE config 1 (512x512 random, w=32, mm/mm, full-block).
* ``dist.npz`` + ``dist.json`` -- ``run_distributed`` runs for g = 2 and 4.

Run (in the build container, where /root/reference exists):

    python tests/golden/make_golden.py

The generated files are committed; nothing on the GPU box reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path(os.environ.get("JHSVD_REF", "/root/reference/pkg"))
COPY = Path("/tmp/jhsvd_ref_copy")


def _import_reference():
    # numba cache=True writes __pycache__ next to the sources: use a copy
    if not (COPY / "src" / "jhsvd").exists():
        if COPY.exists():
            shutil.rmtree(COPY)
        shutil.copytree(REF_SRC, COPY)
    sys.path.insert(0, str(COPY / "src"))
    import jhsvd  # noqa: F401

    return jhsvd


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def gen_strategies(j):
    out = {"hash": {}, "text": {}}
    kinds = ["row", "col", "rrow", "rcol", "bl", "mm"]
    orders = [2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26, 28, 30, 32, 36,
              40, 48, 56, 64, 96, 128, 256, 512, 1024]
    for kind in kinds:
        for n in orders:
            try:
                s = j.make_strategy(kind, n)
            except j.StrategyError as exc:
                out["hash"][f"{kind}:{n}"] = "error:" + type(exc).__name__
                continue
            txt = j.dump_strategy(s)
            out["hash"][f"{kind}:{n}"] = sha(txt.encode())
            if n <= 32:
                out["text"][f"{kind}:{n}"] = txt
            out.setdefault("kindtag", {})[f"{kind}:{n}"] = s.kind
    # doubled / reversed routes used directly by the tests
    for n in (4, 6, 8):
        for kind in ("row", "col"):
            e = j.expand_pstrategy(j.closest_pstrategy(kind, n), kind)
            out["hash"][f"expand:{kind}:{n}"] = sha(j.dump_strategy(e).encode())
    return out


def gen_kernels(j):
    rng = np.random.default_rng(20240101)
    d = {}
    # gram / cholesky / postmultiply cases (m, c)
    cases = [(64, 8), (100, 6), (512, 32), (96, 16), (33, 2), (256, 64)]
    for k, (m, c) in enumerate(cases):
        g = np.asfortranarray(rng.standard_normal((m, c)))
        h = j.gram(g)
        r = j.cholesky_in_place(h)
        v = np.asfortranarray(rng.standard_normal((c, c)))
        d[f"gram{k}_in"] = g
        d[f"gram{k}_out"] = h
        d[f"chol{k}_out"] = r
        d[f"post{k}_v"] = v
        d[f"post{k}_out"] = j.postmultiply(g, v)
    # inner Jacobi on shortened factors: trig and hyperbolic
    icases = [
        (32, 32, "rrow", 30), (32, 32, "mm", 30), (32, 16, "rrow", 30),
        (16, 16, "row", 30), (32, 32, "rrow", 1), (16, 8, "bl", 30),
        (8, 8, "col", 30), (64, 64, "rrow", 30), (32, 0, "rcol", 30),
    ]
    for k, (c, nplus, kind, ms) in enumerate(icases):
        a = rng.standard_normal((4 * c, c)) + 3.0 * np.vstack([np.eye(c)] * 4)
        r = j.cholesky_in_place(j.gram(np.asfortranarray(a)))
        colmap = np.arange(1, c + 1)
        sig = j.Signature(c, nplus)
        strat = j.make_strategy(kind, c)
        res = j.inner_jacobi(r, colmap, sig, strat, ms)
        d[f"inner{k}_r"] = r
        d[f"inner{k}_meta"] = np.array([c, nplus, ms, res.rotations,
                                        res.proper_rotations, res.inner_sweeps])
        d[f"inner{k}_kind"] = np.array(kind)
        d[f"inner{k}_rout"] = res.r_out
        d[f"inner{k}_vacc"] = res.v_acc
    # qr peel-off
    for k, (m, c) in enumerate([(128, 16), (96, 32), (64, 8)]):
        g = np.asfortranarray(rng.standard_normal((m, c)))
        d[f"qr{k}_in"] = g
        d[f"qr{k}_out"] = j.qr_peeloff(g)
    # solve_for_v
    r = np.asfortranarray(np.triu(rng.standard_normal((32, 32))) + 8 * np.eye(32))
    w = np.asfortranarray(rng.standard_normal((32, 32)))
    d["solve_r"], d["solve_w"], d["solve_out"] = r, w, j.solve_for_v(r, w)
    # robust norms: ordinary, huge, tiny, mixed, long vectors
    vecs = [
        rng.standard_normal(1000),
        rng.standard_normal(16384) * 2.0 ** 600,
        rng.standard_normal(300) * 2.0 ** -600,
        np.concatenate([rng.standard_normal(50) * 2.0 ** 700,
                        rng.standard_normal(70),
                        rng.standard_normal(40) * 2.0 ** -700]),
        rng.standard_normal(131072),
        np.concatenate([np.zeros(10), rng.standard_normal(777)]),
        rng.standard_normal(257),
    ]
    for k, x in enumerate(vecs):
        js, s = j.norm2(x)
        d[f"norm{k}_in"] = x
        d[f"norm{k}_out"] = np.array([float(js), s])
    for n in (1, 2, 3, 255, 256, 257, 512, 4096, 16384, 131072, 1 << 20):
        mu, nu = j.safe_bounds(n)
        d[f"safe_{n}"] = np.array([mu, nu])
    return d


def gen_solves(j):
    arrays = {}
    meta = {}
    rng = np.random.default_rng(7)

    def record(name, g, sig, cfg, keep_full=True):
        res = j.block_jacobi(g, sig, cfg)
        meta[name] = {
            "n": int(g.shape[0]),
            "n_plus": int(res.signature.n_plus),
            "cfg": {
                "block_width": cfg.block_width, "variant": cfg.variant,
                "max_block_sweeps": cfg.max_block_sweeps,
                "max_inner_sweeps": cfg.max_inner_sweeps,
                "outer_strategy": cfg.outer_strategy,
                "inner_strategy": cfg.inner_strategy,
                "accumulate_v": cfg.accumulate_v, "solve_v": cfg.solve_v,
                "shortening": cfg.shortening, "eps_factor": cfg.eps_factor,
            },
            "stats": [list(s) for s in res.stats],
            "block_sweeps": res.block_sweeps,
            "converged": res.converged,
            "sigma_sha256": sha(res.sigma.tobytes()),
            "u_sha256": sha(np.asfortranarray(res.u).tobytes(order="F")),
            "v_sha256": (sha(np.asfortranarray(res.v).tobytes(order="F"))
                         if res.v is not None else None),
        }
        arrays[f"{name}_in"] = np.asfortranarray(g)
        arrays[f"{name}_sigma"] = res.sigma
        if keep_full:
            arrays[f"{name}_u"] = res.u
            if res.v is not None:
                arrays[f"{name}_v"] = res.v
        print(name, res.block_sweeps, res.stats[:2], flush=True)

    SC = j.SolverConfig
    # BASELINE config 1: 512x512 random, w=32, mm/mm, full-block
    g1 = np.random.default_rng(0).standard_normal((512, 512))
    record("config1", np.asfortranarray(g1), None,
           SC(block_width=32, outer_strategy="mm", inner_strategy="mm"),
           keep_full=False)
    # spectra types 1-4 at n=128, both variants, default w=32 rrow
    for t in (1, 2, 3, 4):
        lam = j.gen_spectrum(j.SpectrumSpec(t, 128, seed=100 + t))
        g, sig = j.gen_factor(lam, seed=200 + t)
        arrays[f"type{t}_lambda"] = lam
        record(f"type{t}_fb", g, sig, SC())
        record(f"type{t}_bo", g, sig, SC(variant="block-oriented"), keep_full=False)
    # other widths / strategies
    lam = j.gen_spectrum(j.SpectrumSpec(2, 64, seed=11))
    g, sig = j.gen_factor(lam, seed=12)
    for w, k in ((16, "rrow"), (8, "mm"), (16, "bl"), (16, "row"), (16, "col"),
                 (16, "rcol"), (4, "rrow"), (2, "rrow"), (64, "rrow")):
        record(f"n64_w{w}_{k}", g, sig, SC(block_width=w, outer_strategy=k,
                                            inner_strategy=k))
    # accumulate_v=False, capped sweeps, eps_factor
    record("n64_nov", g, sig, SC(block_width=16, accumulate_v=False))
    record("n64_cap1", g, sig, SC(block_width=16, max_block_sweeps=1))
    record("n64_inner2", g, sig, SC(block_width=16, max_inner_sweeps=2))
    record("n64_eps4", g, sig, SC(block_width=16, eps_factor=4.0))
    # hyperbolic n=96 with signature in the middle of a block
    lam = j.gen_spectrum(j.SpectrumSpec(3, 96, seed=13))
    g, sig = j.gen_factor(lam, seed=14)
    arrays["hsvd96_lambda"] = lam
    record("hsvd96", g, sig, SC(block_width=16))
    # column-graded kappa=1e12 (config 2 analog), block-oriented
    n = 256
    b = rng.standard_normal((n, n))
    b /= np.linalg.norm(b, axis=0)
    dgr = np.logspace(0, -12, n)
    record("graded256_bo", np.asfortranarray(b * dgr), None,
           SC(variant="block-oriented"), keep_full=False)
    # tall-ish rectangular is rejected by the reference: not recorded
    # qr shortening and solve_v
    lam = j.gen_spectrum(j.SpectrumSpec(2, 64, seed=15))
    g, sig = j.gen_factor(lam, seed=16)
    record("n64_qr", g, sig, SC(block_width=16, shortening="qr"))
    tri = np.asfortranarray(np.triu(rng.standard_normal((64, 64))) + 8 * np.eye(64))
    record("n64_solvev", tri, None, SC(block_width=16, accumulate_v=False,
                                        solve_v=True))
    # diagonal input (converges with zero rotations)
    record("diag4", np.asfortranarray(np.diag([3.0, 1.0, 2.0, 5.0])), None,
           SC(block_width=2))
    return arrays, meta


def gen_dist(j):
    from jhsvd import distsim

    arrays = {}
    meta = {}
    lam = j.gen_spectrum(j.SpectrumSpec(3, 128, seed=42))
    g, sig = j.gen_factor(lam, seed=43)
    arrays["dist_in"] = g
    arrays["dist_lambda"] = lam
    SC = j.SolverConfig
    for gw, cfg_name, cfg in (
        (2, "bo", SC(variant="block-oriented")),
        (4, "bo", SC(variant="block-oriented")),
        (2, "fb", SC()),
        (4, "fb", SC(block_width=16)),
        (2, "bo_nov", SC(variant="block-oriented", accumulate_v=False)),
    ):
        res, trace = distsim.run_distributed(g, sig, gw, cfg)
        name = f"g{gw}_{cfg_name}"
        mapping = distsim.optimize_mapping(j.make_strategy(cfg.outer_strategy, 2 * gw),
                                           distsim.Topology(gw))
        meta[name] = {
            "g": gw, "block_width": cfg.block_width, "variant": cfg.variant,
            "accumulate_v": cfg.accumulate_v,
            "stats": [list(s) for s in res.stats],
            "block_sweeps": res.block_sweeps, "converged": res.converged,
            "sigma_sha256": sha(res.sigma.tobytes()),
            "assignments": [[list(pq) for pq in step] for step in mapping.assignments],
        }
        arrays[f"{name}_sigma"] = res.sigma
        if res.v is not None:
            arrays[f"{name}_v"] = res.v
        print(name, res.block_sweeps, flush=True)
    return arrays, meta


def main():
    j = _import_reference()
    HERE.mkdir(parents=True, exist_ok=True)
    strat = gen_strategies(j)
    (HERE / "strategies.json").write_text(json.dumps(strat, indent=1, sort_keys=True))
    np.savez_compressed(HERE / "kernels.npz", **gen_kernels(j))
    arrays, meta = gen_solves(j)
    np.savez_compressed(HERE / "solves.npz", **arrays)
    (HERE / "solves.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    arrays, meta = gen_dist(j)
    np.savez_compressed(HERE / "dist.npz", **arrays)
    (HERE / "dist.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    import numba

    (HERE / "PROVENANCE.txt").write_text(
        f"generated by tests/golden/make_golden.py from {REF_SRC}\n"
        f"numpy {np.__version__}, numba {numba.__version__}\n"
    )


if __name__ == "__main__":
    main()
