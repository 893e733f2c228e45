"""Benchmark: FP64 SVD seconds to convergence (BASELINE.json config 3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One *step* is one complete solve to convergence -- input factor resident in
HBM -> sigma, U, V -- of the BASELINE.json config 3 workload: a 16384 x 16384
FP64 factor, full-block variant, rrow (Mantharam-Eberlein-equivalent)
strategy, block width 32 (block-columns of 16), V accumulated.  The factor is
synthetic and reproducible: G = Q diag(sqrt(lambda)) W^T with the
reference's type-2 spectrum (testgen.gen_spectrum, seed 3) and random Givens
butterfly Q, W generated on the GPU (jh_gen_butterfly; its host twin
oracle/gen_butterfly.c writes the same bytes, so the C oracle's offline
whole solve of this exact matrix, tests/golden/offline/config3.json, is the
parity reference).  The 2 GiB factor is larger than L2, so no flush is
needed between steps.

N > 1 GPUs: one rank per GPU (torchrun; ``--gpus N`` without torchrun
relaunches itself under torchrun, and refuses when the box has fewer GPUs).
The ranks run ``block_jacobi_sharded``: block-columns sharded over the GPUs,
one NCCL exchange per table segment, bitwise the same solve as N = 1.

Prints ONE JSON line (rank 0).  Besides the contract keys it carries
 - e2e: the same metric through the public API with host (pinned) buffers,
   host<->device copies inside the timed region;
 - roofline: the dominant kernel's algorithmic HBM bytes / CUDA-event time;
 - fp64_roofline: the whole solve's DMMA flops against the measured DMMA rate;
 - energy_roofline: the solve runs at the board power limit, so joules bound
   its speed: NVML energy over the timed region against the floor DMMA
   flops x pJ/flop + HBM bytes x pJ/byte + idle power x time
   (profiles/r02/energy_probe.json); clocks carries power draw and limit;
 - cpu_baseline: the C oracle (a port of the reference CPU solver) timed on
   a bounded prefix of the same solve on this host, extrapolated with the
   per-sweep cost profile of the oracle's own offline whole solve;
 - parity: input / sigma / U / V / stats against the offline oracle golden,
   plus the sampled p-steps bitwise against the oracle;
 - accuracy: sigma vs the prescribed spectrum, orthogonality of U and V.
``--impl reference`` times only the CPU oracle on the same workload.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FP64 SVD sec to convergence (n=16384) at 1/2/4/8 B200; σ rel err; sweeps"
PAPER_K20C_16384_S = 2625.642659  # Table 6.2 (Kepler K20c)
GOLDEN = ROOT / "tests" / "golden" / "offline"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", type=int, default=16384, help="order (config 3 at 16384)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU-oracle sample length")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def the_workload(args):
    from paper_1401_2720_b200 import workloads as WL

    return WL.CONFIG3 if args.n == WL.CONFIG3.n else WL.scaled(WL.CONFIG3, args.n)


def workload_config(wl, in_sha=None) -> dict:
    d = {
        "workload": f"config3: {wl.describe()}, V accumulated",
        "n": wl.n, "m": wl.m, "block_width": wl.block_width, "variant": wl.variant,
        "outer_strategy": wl.strategy, "inner_strategy": wl.strategy,
        "l2": (f"inputs larger than L2 (factor {8 * wl.m * wl.n / 2**30:.2f} GiB per step)"
               if 8 * wl.m * wl.n > 126e6 else "factor fits in L2 (no flush)"),
    }
    if in_sha:
        d["input_sha256"] = in_sha
    return d


def load_golden(wl):
    p = GOLDEN / f"{wl.name}.json"
    if not p.exists():
        return None
    gold = json.loads(p.read_text())
    prog = GOLDEN / f"{wl.name}.progress.jsonl"
    if prog.exists():
        secs = [json.loads(x)["seconds"] for x in prog.read_text().splitlines() if x.strip()]
        if len(secs) >= gold["block_sweeps"]:
            gold["sweep_seconds"] = secs[-gold["block_sweeps"]:]
    return gold


def sha_rows(t) -> str:
    """sha256 of a (cols, rows) column-major storage tensor (or numpy)."""
    a = t.cpu().numpy() if hasattr(t, "cpu") else t
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,power.draw,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        rows = []
        for line in Path(self.file.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                pw = float(parts[3]) if parts[3] not in ("", "[N/A]") else None
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[4:8], pw))
            except ValueError:
                continue
        os.unlink(self.file.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        loaded = [r for r in rows if r[2] >= 50.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3])
                          if v.lower() == "active"})
        pws = [r[4] for r in loaded if r[4] is not None]
        return {"sm_mhz": statistics.median(r[0] for r in loaded),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(loaded),
                # the solve runs at the board power limit: energy, not the
                # clock-peak rooflines, sets its speed (profiles/r02/energy_probe.json)
                "power_w": statistics.median(pws) if pws else None,
                "power_limit_w": _power_limit(self.index)}


def _power_limit(index: int):
    try:
        out = subprocess.run(["nvidia-smi", "-i", str(index), "--query-gpu=enforced.power.limit",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=10).stdout.strip()
        return float(out)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU baseline (oracle = C port of the reference solver)


def cpu_sample(g_host_t, wl, target_s: float, nsteps_max=None):
    """Time p-steps of sweep 1 with the C oracle on all host cores, from the
    input factor (storage (n, m)).  Returns (seconds per p-step, timed
    p-steps, threads, oracle G and V after p-steps 0..k)."""
    from oracle import oracle as O
    from paper_1401_2720_b200.strategy import as_table, make_strategy

    n, w = wl.n, wl.block_width
    cfg = dict(block_width=w, variant=wl.variant)
    outer = as_table(make_strategy(wl.strategy, n // (w // 2)))
    inner = as_table(make_strategy(wl.strategy, w))
    g = np.array(g_host_t, copy=True).T  # F-order m x n
    v = np.asfortranarray(np.eye(n))
    threads = O.max_threads()
    t0 = time.perf_counter()
    O.block_sweep(g, v, n, cfg, outer[:1], inner, threads=threads)  # warm, p-step 0
    t1 = time.perf_counter() - t0
    k = int(max(1, min(outer.shape[0] - 1, math.ceil(target_s / max(t1, 1e-3)))))
    if nsteps_max:
        k = min(k, nsteps_max)
    t0 = time.perf_counter()
    O.block_sweep(g, v, n, cfg, outer[1:1 + k], inner, threads=threads)
    tk = time.perf_counter() - t0
    return tk / k, k, threads, g, v


def extrapolate(t_p: float, b: int, gold, sweeps_here=None, rotated_frac=None):
    """Whole-solve CPU seconds from the sweep-1 p-step rate: (b - 1) p-steps
    per sweep, weighted per sweep by the oracle's own offline whole-solve
    profile (its measured per-sweep seconds relative to sweep 1) when the
    golden has it; otherwise by the fraction of tasks that rotated."""
    if gold and gold.get("sweep_seconds"):
        w = [s / gold["sweep_seconds"][0] for s in gold["sweep_seconds"]]
        how = (f"per-sweep weights from the oracle's offline whole solve "
               f"({gold['threads']} threads, {len(w)} sweeps)")
    elif rotated_frac:
        # gram + cholesky + inner ~ 0.3 of a rotated p-step on the oracle
        w = [0.3 + 0.7 * f for f in rotated_frac]
        how = f"per-sweep weights 0.3 + 0.7 x (fraction of tasks rotated), {len(w)} sweeps"
    else:
        w = [1.0] * (sweeps_here or 9)
        how = f"{len(w)} sweeps at the sweep-1 rate"
    return t_p * (b - 1) * sum(w), how


# ---------------------------------------------------------------------------
# reference arm


def run_reference(args, rank: int):
    if rank != 0:
        return
    from oracle import oracle as O

    wl = the_workload(args)
    sigma_p, n_plus = wl.sigma_nplus()
    g = O.gen_butterfly(sigma_p, m=wl.m, n_plus=n_plus, seed=wl.gen_seed, passes=wl.passes,
                        tanh_max=wl.tanh_max)  # input synthesis (not timed)
    host_t = np.ascontiguousarray(g.T)
    del g
    gold = load_golden(wl)
    b = wl.n // (wl.block_width // 2)
    per = []
    k = threads = 0
    for i in range(args.warmup + args.steps):
        t_p, k, threads, _, _ = cpu_sample(host_t, wl, args.cpu_seconds if i >= args.warmup
                                           else 1.0)
        if i >= args.warmup:
            per.append(t_p)
    t_p = statistics.mean(per)
    value, how = extrapolate(t_p, b, gold)
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": workload_config(wl, sha_rows(host_t)),
        "impl": "reference",
        "cpu_baseline": {
            "value": value, "unit": "s", "cores": threads, "kind": "port",
            "sample": (f"C oracle (port of the reference numba solver) on p-steps 1..{k} of "
                       f"sweep 1 (of {b - 1}) from the input, {t_p:.3f} s/p-step, extrapolated "
                       f"x{b - 1} p-steps, {how}")},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# multi-GPU plumbing


def _init_dist(world: int):
    """One process per GPU (torchrun): NCCL group, device = LOCAL_RANK."""
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def _reduce(x: float, world: int, op: str = "max") -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM,
                           "min": dist.ReduceOp.MIN}[op])
    return float(t.item())


def _barrier(world: int):
    import torch

    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        torch.cuda.synchronize()


def _relaunch_under_torchrun(n: int):
    import torch

    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < n:
        raise SystemExit(f"bench.py --gpus {n}: this box has {have} GPU(s); refusing to label a "
                         f"smaller run as {n} GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------
# our arm


def _nvml_handle(index: int):
    try:
        import pynvml

        pynvml.nvmlInit()
        return pynvml.nvmlDeviceGetHandleByIndex(index)
    except Exception:
        return None


def _energy_j(h):
    """Total energy the GPU drew since driver load (NVML), joules."""
    if h is None:
        return None
    try:
        import pynvml

        return pynvml.nvmlDeviceGetTotalEnergyConsumption(h) / 1e3
    except Exception:
        return None


def fp64_peak():
    p = ROOT / "profiles" / "r02" / "dmma_rate.json"
    if p.exists():
        d = json.loads(p.read_text())
        return (float(d["dmma_tflops"]),
                f"builder-measured DMMA rate (profiles/r02/dmma_rate.json, "
                f"SM clock {d.get('sm_mhz')} MHz)")
    return 37.0, "builder-measured DMMA rate (profiles/r01/dmma_chains_probe.jsonl, clock not recorded)"


def traffic_of(kernel: str):
    for p in (ROOT / "profiles" / "r02" / "ncu_traffic.json", ROOT / "profiles" / "ncu_traffic.json"):
        if p.exists():
            d = json.loads(p.read_text())
            if kernel in d:
                return d[kernel], d.get(kernel + "_algorithmic"), str(p.relative_to(ROOT))
    return None, None, None


def run_ours(args, rank: int, world: int):
    import ctypes

    import torch

    import paper_1401_2720_b200 as J
    from paper_1401_2720_b200 import _lib, testgen as T
    from paper_1401_2720_b200.driver import Solver
    from paper_1401_2720_b200.sharded import CudaShardEngine, block_jacobi_sharded, shard_plan

    _init_dist(world)
    lib = _lib.require_cuda()
    wl = the_workload(args)
    cfg = J.SolverConfig(**wl.solver_kwargs())
    G0, sigma_true, n_plus = T.workload_input_device(wl)
    torch.cuda.synchronize()
    n, m, w = wl.n, wl.m, wl.block_width
    b = n // (w // 2)
    sig = J.Signature(n, n_plus)
    in_sha = sha_rows(G0) if rank == 0 else None
    solver = Solver(n, cfg, sig, m=m) if world == 1 else None
    eng1 = solver.engine if solver else None
    plan = shard_plan(J.make_strategy(wl.strategy, b), world) if world > 1 else None
    sh_eng = CudaShardEngine(m, n, plan, cfg, n_plus, True) if world > 1 else None

    def solve(g_dev=G0):
        """One step: a full solve from the resident factor."""
        if world == 1:
            return solver.solve_device(g_dev)
        res = block_jacobi_sharded(g_dev.t(), sig, world, cfg, engine=sh_eng)
        return (res.sigma, res.u.t(), res.v.t(), [list(s) for s in res.stats], res.converged)

    for _ in range(args.warmup):
        out = solve()
        del out
    _barrier(world)

    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
    launches0 = lib.jh_launch_count()
    nvml = _nvml_handle(torch.cuda.current_device())
    energy0 = _energy_j(nvml)
    times = []
    res = None
    for _ in range(args.steps):
        _barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = solve()
        e1.record()
        _barrier(world)
        times.append(_reduce(e0.elapsed_time(e1) / 1e3, world, "max"))
    launches = int(_reduce(float(lib.jh_launch_count() - launches0), world, "sum"))
    energy1 = _energy_j(nvml)
    clocks = sampler.stop() if sampler else None
    value = statistics.mean(times)
    sigma, U, V, stats, converged = res
    del res

    # per-kernel timing: one more (untimed) solve with the kernels kept apart
    # (engine 1 otherwise overlaps the update with the inner Jacobi), CUDA
    # events around each launch on the launching stream
    lib.jh_set_overlap(0)
    lib.jh_profile_begin(4 * (b + 8) * cfg.max_block_sweeps * 4)
    if sh_eng is not None:
        sh_eng.tasks_rotated = []
    prof = solve()
    ms = (ctypes.c_double * 4)()
    cnt = (ctypes.c_int64 * 4)()
    lib.jh_profile_end(ms, cnt)
    lib.jh_set_overlap(1)
    del prof
    rotated_tasks = sum(eng1.tasks_rotated) if eng1 is not None else sum(sh_eng.tasks_rotated)
    rotated_per_sweep = (list(eng1.tasks_rotated) if eng1 is not None
                         else list(sh_eng.tasks_rotated_sweeps))

    # ---- roofline of the dominant streaming kernel (this rank) ----
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    ntask = n // w // world
    bytes_gram_launch = ntask * 8.0 * w * m
    # update launches: read + write of the pair columns of G per rotated task;
    # V once per two p-steps (engine 1 pairs the p-steps over 4-cycles)
    v_factor = 0.5
    bytes_update_total = rotated_tasks * 16.0 * w * (m + v_factor * n)
    classes = {
        "gram": {"ms": ms[0], "launches": cnt[0], "bytes_total": bytes_gram_launch * cnt[0],
                 "flops_total": ntask * m * w * (w + 1.0) * cnt[0]},
        "factor_inner": {"ms": ms[1], "launches": cnt[1], "bytes_total": 0.0},
        "update": {"ms": ms[2] + ms[3], "launches": cnt[2], "bytes_total": bytes_update_total,
                   "flops_total": rotated_tasks * 2.0 * w * w * (m + n)},
    }
    tot_ms = sum(c["ms"] for c in classes.values()) or 1.0
    dom = max(("gram", "update"), key=lambda k: classes[k]["ms"])
    d = classes[dom]
    achieved = d["bytes_total"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else 0.0
    traffic, traffic_alg, traffic_src = traffic_of(dom)
    chol_flops = ntask * w ** 3 / 3.0 * cnt[0]
    solve_flops = classes["gram"]["flops_total"] + classes["update"]["flops_total"] + chol_flops
    solve_flops_all = _reduce(solve_flops, world, "sum")
    peak_tf, peak_src = fp64_peak()
    fp64 = {
        "achieved_tflops": solve_flops_all / value / 1e12 if value else 0.0,
        "peak_tflops": peak_tf * world, "frac": solve_flops_all / value / 1e12 / (peak_tf * world),
        "solve_flops": solve_flops_all,
        "gram_tflops": (classes["gram"]["flops_total"] / (classes["gram"]["ms"] / 1e3) / 1e12
                        if classes["gram"]["ms"] > 0 else None),
        "update_tflops": (classes["update"]["flops_total"] / (classes["update"]["ms"] / 1e3)
                          / 1e12 if classes["update"]["ms"] > 0 else None),
        "peak_source": peak_src,
    }
    roofline = {
        "kernel": dom, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
        "frac": achieved / hbm_peak, "traffic": traffic,
        "traffic_launch_algorithmic_bytes": traffic_alg, "traffic_source": traffic_src,
        "bytes_per_launch": d["bytes_total"] / max(d["launches"], 1),
        "avg_launch_ms": d["ms"] / max(d["launches"], 1),
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
        "kernel_share": {k: c["ms"] / tot_ms for k, c in classes.items()},
        "solve_hbm_frac": ((classes["gram"]["bytes_total"] + bytes_update_total) * world
                           / value / 1e9 / (hbm_peak * world)),
        "timing_note": ("per-kernel times from one extra solve with the kernels kept apart "
                        "(jh_set_overlap(0)); the timed solves overlap the update with the "
                        "inner Jacobi" + ("; rank 0's kernels" if world > 1 else "")),
    }

    # ---- energy roofline: the solve runs at the board power limit, so its
    # speed is set by joules, not by the clock-peak rooflines.  Per solve:
    # the measured energy (NVML counter over the timed region) against the
    # model's floor from this pool's measured unit costs
    # (profiles/r02/energy_probe.json): DMMA flops x J/flop + algorithmic
    # HBM bytes x J/byte + idle power x the measured time.
    energy = None
    probe = ROOT / "profiles" / "r02" / "energy_probe.json"
    if energy0 is not None and energy1 is not None and probe.exists():
        ep = json.loads(probe.read_text())
        e_meas = (energy1 - energy0) / args.steps
        solve_bytes = classes["gram"]["bytes_total"] + bytes_update_total
        e_dmma = solve_flops * ep["dmma"]["pj_per_flop_above_idle"] * 1e-12
        e_hbm = solve_bytes * ep["hbm"]["pj_per_byte_above_idle"] * 1e-12
        e_idle = ep["idle_w"] * value
        floor = e_dmma + e_hbm + e_idle
        limit = (clocks or {}).get("power_limit_w") or 1000.0
        energy = {
            "joules_per_solve": e_meas, "avg_power_w": e_meas / value if value else None,
            "model_floor_j": floor, "frac": floor / e_meas if e_meas else None,
            "model_j": {"dmma": e_dmma, "hbm": e_hbm, "idle": e_idle},
            # the time at which the floor's dynamic energy would run at the limit
            "time_at_power_limit_s": (e_dmma + e_hbm) / (limit - ep["idle_w"]),
            "unit_costs": {"pj_per_dmma_flop": ep["dmma"]["pj_per_flop_above_idle"],
                           "pj_per_hbm_byte": ep["hbm"]["pj_per_byte_above_idle"],
                           "idle_w": ep["idle_w"], "source": "profiles/r02/energy_probe.json"},
            "note": "rank-local GPU" if world > 1 else "one GPU",
        }

    def run_e2e():
        """The same solve through the public API from pinned host memory
        (host->device copy of the factor and device->host copy of sigma, U,
        V inside the timed region)."""
        host_in = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        host_in.copy_(G0)
        g_host = host_in.t()  # m x n, column-major, pinned
        torch.cuda.empty_cache()
        et = []
        # one untimed warm-up call: steady state of a process that solves
        # repeatedly (pinned output buffers come from torch's caching host
        # allocator; a first-ever call also pays ~0.9 s per 2 GB of page pinning)
        for k in range((1 if args.warmup > 0 else 0) + args.steps):
            _barrier(world)
            t0 = time.perf_counter()
            if world == 1:
                r = J.block_jacobi(g_host, sig, cfg, allow_tall=m > n)
            else:
                r = block_jacobi_sharded(g_host, sig, world, cfg, engine=sh_eng,
                                         allow_tall=m > n)
            dt = _reduce(time.perf_counter() - t0, world, "max")
            if k >= (1 if args.warmup > 0 else 0):
                et.append(dt)
            del r
        return {"value": statistics.mean(et), "unit": "s",
                "h2d_bytes_per_step": 8 * m * n * world,
                "d2h_bytes_per_step": 8 * (n + m * n + n * n) * world,
                "note": ("public API " + ("block_jacobi" if world == 1 else
                                          f"block_jacobi_sharded (each of {world} ranks passes "
                                          "the full host factor and receives the full result)")
                         + " on a pinned host factor: H2D of G, solve, sigma/U/V back to host, "
                           "after one untimed warm-up call")}

    gold = load_golden(wl)
    if rank != 0:
        del U, V, sigma
        if not args.no_e2e:
            run_e2e()
        _rank_info(world)
        return

    # ---- accuracy and whole-solve parity (outside the timed region) ----
    sig_h = sigma.cpu().numpy()
    ref = np.concatenate((np.sort(sigma_true[:n_plus])[::-1], np.sort(sigma_true[n_plus:])[::-1]))
    rel = float(np.max(np.abs(sig_h - ref) / ref))
    eye = torch.eye(n, dtype=torch.float64, device=U.device)
    ortho_u = float((U @ U.t() - eye).abs().max()) if m == n else None
    ortho_v = float((V @ V.t() - eye).abs().max())
    del eye
    accuracy = {"sigma_max_rel_err_vs_prescribed": rel, "u_orth_max": ortho_u,
                "v_orth_max": ortho_v, "n_eps": n * 2.0 ** -53}
    parity = {"golden": None}
    if gold is not None:
        gs = np.load(GOLDEN / f"{wl.name}_sigma.npy")
        parity = {
            "golden": f"tests/golden/offline/{wl.name}.json (C oracle whole solve, "
                      f"{gold['threads']} threads, {gold.get('solve_wall_s', 0):.0f} s)",
            "input_sha256_equal": in_sha == gold["input_sha256"],
            "stats_equal_oracle": [list(s) for s in stats] == gold["stats"],
            "sigma_bitwise_vs_oracle": sha_rows(sigma) == gold["sigma_sha256"],
            "u_bitwise_vs_oracle": sha_rows(U) == gold["u_sha256"],
            "v_bitwise_vs_oracle": sha_rows(V) == gold["v_sha256"],
            "sigma_max_rel_vs_oracle": float(np.max(np.abs(sig_h - gs) / gs)),
        }
    del U, V

    # ---- CPU baseline (bounded oracle sample) + bitwise prefix parity ----
    cpu = None
    if not args.no_cpu:
        host = G0.cpu().numpy()
        t_p, k, threads, g_or, v_or = cpu_sample(host, wl, args.cpu_seconds)
        nt_all = n // w
        frac = [r / nt_all / (b - 1) for r in rotated_per_sweep] if rotated_per_sweep else None
        est, how = extrapolate(t_p, b, gold, len(stats), frac)
        cpu = {"value": est, "unit": "s", "cores": threads, "kind": "port",
               "sample": (f"C oracle (port of the reference numba solver): p-steps 1..{k} of "
                          f"sweep 1 ({t_p:.3f} s/p-step), extrapolated x{b - 1} p-steps, {how}")}
        if not args.no_parity and world == 1:
            Gp = G0.clone()
            Vp = torch.eye(n, dtype=torch.float64, device=G0.device)
            eng1.sweep(Gp, Vp, 0, 1 + k)
            torch.cuda.synchronize()
            parity["prefix_psteps"] = 1 + k
            parity["prefix_G_bitwise"] = bool(np.array_equal(Gp.cpu().numpy(),
                                                             np.ascontiguousarray(g_or.T)))
            parity["prefix_V_bitwise"] = bool(np.array_equal(Vp.cpu().numpy(),
                                                             np.ascontiguousarray(v_or.T)))
            del Gp, Vp
        del host, g_or, v_or

    e2e = run_e2e() if not args.no_e2e else None
    del G0

    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
        "higher_is_better": False, "scaling": "strong",
        "vs_baseline": value / PAPER_K20C_16384_S,
        "dtype": "f64", "data": "synthetic", "config": workload_config(wl, in_sha),
        "parallelism": ("1 GPU" if world == 1 else
                        f"block-columns sharded over {world} GPUs (block_jacobi_sharded, "
                        f"{2 * world - 1} NCCL exchanges per sweep, bitwise = 1 GPU)"),
        "sweeps": len(stats), "converged": converged, "stats": [list(s) for s in stats],
        "tasks_rotated_per_sweep": rotated_per_sweep,
        "accuracy": accuracy, "parity": parity,
        "e2e": e2e, "roofline": roofline, "fp64_roofline": fp64, "energy_roofline": energy,
        "cpu_baseline": cpu,
        "clocks": clocks, "gpu_launches": launches,
        "per_step_s": times,
        "ranks": _rank_info(world),
    }
    print(json.dumps(line), flush=True)


def _rank_info(world: int) -> dict:
    """Process-group evidence: world size, backend, NCCL version, the GPUs
    the ranks ran on (all-gathered)."""
    import torch

    info = {"world": world, "device": torch.cuda.get_device_name()}
    if world > 1:
        import torch.distributed as dist

        names = [None] * world
        dist.all_gather_object(names, (dist.get_rank(), torch.cuda.current_device(),
                                       torch.cuda.get_device_name()))
        info.update(backend=dist.get_backend(), ranks=names,
                    nccl=".".join(map(str, torch.cuda.nccl.version())))
    return info


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus > 1 and world == 1 and args.impl == "ours":
        _relaunch_under_torchrun(args.gpus)
    if world > 1 and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_ours(args, rank, world)


if __name__ == "__main__":
    main()
