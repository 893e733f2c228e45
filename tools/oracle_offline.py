"""Whole-solve oracle goldens for the BASELINE workloads (CPU only, offline).

    python tools/oracle_offline.py config3 [--threads T] [--n N]

Builds the workload's input with the host twin of the GPU generator
(oracle/gen_butterfly.c), records its sha256, runs the C oracle (the C
restatement of the reference solver, oracle/jhsvd_oracle.c) to convergence
sweep by sweep (checkpointing G and V under /tmp so an interrupted run
resumes), and writes

    tests/golden/offline/<name>.json        stats, sweeps, sha256 of the
                                            input, sigma, U and V bytes
    tests/golden/offline/<name>_sigma.npy   sorted sigma (for tolerance checks)

The GPU bench (bench.py) and tests/test_offline_golden.py compare against
these.  Test infrastructure: nothing in the product imports it.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1401_2720_b200 import workloads as WL  # noqa: E402
from paper_1401_2720_b200.strategy import as_table, make_strategy  # noqa: E402


def sha(a: np.ndarray) -> str:
    """sha256 of the column-major bytes (== the GPU's (n, m) storage)."""
    return hashlib.sha256(np.asfortranarray(a).T.tobytes() if a.ndim == 2
                          else np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", choices=sorted(WL.WORKLOADS))
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--n", type=int, default=0, help="scaled-down run (testing the tool)")
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "offline"))
    ap.add_argument("--ckpt", default="/tmp/oracle_ckpt")
    args = ap.parse_args()
    wl = WL.WORKLOADS[args.name]
    if args.n:
        wl = WL.scaled(wl, args.n, args.n * wl.m // wl.n)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    ck = Path(args.ckpt) / wl.name
    ck.mkdir(parents=True, exist_ok=True)
    log = open(out / f"{wl.name}.progress.jsonl", "a")

    sigma_p, n_plus = wl.sigma_nplus()
    m, n, w = wl.m, wl.n, wl.block_width
    t0 = time.time()
    g = O.gen_butterfly(sigma_p, m=m, n_plus=n_plus, seed=wl.gen_seed, passes=wl.passes,
                        tanh_max=wl.tanh_max)
    in_sha = sha(g)
    print(f"input {m}x{n} sha256 {in_sha} ({time.time() - t0:.1f} s)", flush=True)
    cfg = dict(block_width=w, variant=wl.variant)
    outer = as_table(make_strategy(wl.strategy, n // (w // 2)))
    inner = as_table(make_strategy(wl.strategy, w))
    v = np.asfortranarray(np.eye(n))
    stats = []
    state = ck / "state.json"
    if state.exists():
        st = json.loads(state.read_text())
        if st["input_sha256"] == in_sha:
            g = np.asfortranarray(np.load(ck / "g.npy"))
            v = np.asfortranarray(np.load(ck / "v.npy"))
            stats = [tuple(s) for s in st["stats"]]
            print(f"resumed after {len(stats)} sweeps", flush=True)
    c = O._cfg(cfg)
    converged = bool(stats) and stats[-1][1] == 0
    t_solve = time.time()
    while not converged and len(stats) < c.max_block_sweeps:
        ts = time.time()
        rot, proper = O.block_sweep(g, v, n_plus, cfg, outer, inner, threads=args.threads)
        stats.append((rot, proper))
        converged = proper == 0
        rec = {"sweep": len(stats), "rotations": rot, "proper": proper,
               "seconds": time.time() - ts}
        print(json.dumps(rec), flush=True)
        log.write(json.dumps(rec) + "\n")
        log.flush()
        np.save(ck / "g.npy", g)
        np.save(ck / "v.npy", v)
        state.write_text(json.dumps({"input_sha256": in_sha, "stats": stats}))
    sigma = O.extract_sigma(g)
    u = g / sigma
    order = O.class_sort_order(sigma, n_plus)
    sigma, u, v = sigma[order], u[:, order], v[:, order]
    ref = np.sort(sigma_p[:n_plus])[::-1]
    ref = np.concatenate((ref, np.sort(sigma_p[n_plus:])[::-1]))
    gold = {
        "workload": wl.describe(), "name": wl.name, "m": m, "n": n, "n_plus": n_plus,
        "block_width": w, "variant": wl.variant, "strategy": wl.strategy,
        "gen": {"seed": wl.gen_seed, "passes": wl.passes, "tanh_max": wl.tanh_max,
                "spectrum": wl.spectrum, "spectrum_seed": wl.spectrum_seed},
        "input_sha256": in_sha,
        "stats": [list(s) for s in stats], "block_sweeps": len(stats), "converged": converged,
        "sigma_sha256": sha(sigma), "u_sha256": sha(u), "v_sha256": sha(v),
        "sigma_max_rel_err_vs_prescribed": float(np.max(np.abs(sigma - ref) / ref)),
        "oracle": "oracle/jhsvd_oracle.c (C restatement of the reference solver)",
        "threads": O.max_threads() if args.threads <= 0 else args.threads,
        "solve_wall_s": time.time() - t_solve,
    }
    (out / f"{wl.name}.json").write_text(json.dumps(gold, indent=1) + "\n")
    np.save(out / f"{wl.name}_sigma.npy", sigma)
    print(json.dumps(gold), flush=True)


if __name__ == "__main__":
    main()
