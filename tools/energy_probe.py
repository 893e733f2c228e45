"""Energy model of the config-3 p-step on this B200 (dev tool).

The long solve runs at the board power limit (sw_power_cap, ~1000 W,
SM clock 1750-1850 MHz instead of 1965), so joules per p-step, not the
clock-peak rooflines, bound its speed.  This probe measures, with the NVML
total-energy counter and CUDA events:

  idle        power with the GPU idle (static + clock tree)
  dmma        the DMMA rate probe (tools/dev, 2 CTAs x 4 warps per SM,
              8 chains per warp): J per DMMA flop above idle, TF/s, clock
  hbm         device copies of 4 GiB buffers: J per HBM byte above idle,
              GB/s, clock
  pstep       K all-rotating p-steps of sweep 1 of config 3 (engine 1):
              J per p-step, ms per p-step, clock

and writes profiles/r02/energy_probe.json with the decomposition of one
p-step's energy into DMMA flops (45.1 GF) x J/flop + HBM bytes (8.59 GB) x
J/byte + idle power x time, the modelled power at the measured p-step time
and the p-step time the model predicts at the 1000 W limit.

    python tools/energy_probe.py [K]
"""

import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import pynvml
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1401_2720_b200 as J  # noqa: E402
from paper_1401_2720_b200 import _lib, testgen as T, workloads as WL  # noqa: E402
from paper_1401_2720_b200.driver import Solver  # noqa: E402
from tools.dev import devlib  # noqa: E402

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)


def energy_mj():
    return pynvml.nvmlDeviceGetTotalEnergyConsumption(H)


def measured(fn, seconds):
    """Run fn() back to back for ~seconds: (ms per call, J per call, median
    SM MHz, median W)."""
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    fn()
    torch.cuda.synchronize()
    one = max(time.time() - t0, 1e-4)
    reps = max(3, int(seconds / one))
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                            "--format=csv,noheader,nounits", "-lms", "100"], stdout=f,
                           stderr=subprocess.DEVNULL)
    time.sleep(0.5)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    j0 = energy_mj()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    j1 = energy_mj()
    smi.terminate()
    smi.wait()
    ms = e0.elapsed_time(e1)
    clk, pw = [], []
    for line in Path(f.name).read_text().splitlines():
        try:
            a, b = line.split(",")
            clk.append(float(a))
            pw.append(float(b))
        except ValueError:
            pass
    med = lambda v: sorted(v)[len(v) // 2] if v else None  # noqa: E731
    return ms / reps, (j1 - j0) / 1e3 / reps, med(clk), med(pw), ms / 1e3


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    _lib.require_cuda()
    dev = devlib.load()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = {}
    # idle
    torch.cuda.synchronize()
    time.sleep(1.0)
    j0, t0 = energy_mj(), time.time()
    time.sleep(3.0)
    res["idle_w"] = (energy_mj() - j0) / 1e3 / (time.time() - t0)
    # DMMA
    ctas, threads, iters = sms * 2, 128, 20000
    flops = 2.0 * ctas * threads / 32 * iters * 8 * 256
    ms, jc, clk, pw, secs = measured(
        lambda: _lib.check(dev.jh_probe_rate(0, ctas, threads, iters, out.data_ptr(),
                                             _lib.stream_handle()), "rate"), 6.0)
    res["dmma"] = {"tflops": flops / ms / 1e9, "j_per_call": jc, "sm_mhz": clk, "power_w": pw,
                   "pj_per_flop_above_idle": (jc - res["idle_w"] * ms / 1e3) / flops * 1e12}
    # HBM copy
    a = torch.empty(1 << 29, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    nbytes = 2 * a.numel() * 8
    ms, jc, clk, pw, secs = measured(lambda: b.copy_(a), 6.0)
    res["hbm"] = {"gbs": nbytes / ms / 1e6, "j_per_call": jc, "sm_mhz": clk, "power_w": pw,
                  "pj_per_byte_above_idle": (jc - res["idle_w"] * ms / 1e3) / nbytes * 1e12}
    del a, b
    torch.cuda.empty_cache()
    # p-steps of sweep 1 (all rotating)
    wl = WL.CONFIG3
    n = wl.n
    G0, _, npl = T.workload_input_device(wl)
    s = Solver(n, J.SolverConfig(**wl.solver_kwargs()), J.Signature(n, npl))
    V0 = torch.eye(n, dtype=torch.float64, device="cuda")
    G, V = G0.clone(), V0.clone()

    def steps():
        G.copy_(G0)
        V.copy_(V0)
        s.engine.sweep(G, V, 0, k)

    ms, jc, clk, pw, secs = measured(steps, 12.0)
    # subtract the two 2 GiB re-initialisation copies (8.6 GB of HBM traffic)
    init_ms, init_j, *_ = measured(lambda: (G.copy_(G0), V.copy_(V0)), 2.0)
    ms_p = (ms - init_ms) / k
    j_p = (jc - init_j) / k
    dmma_flops = 45.1e9
    hbm_bytes = 8.59e9
    e_dmma = dmma_flops * res["dmma"]["pj_per_flop_above_idle"] * 1e-12
    e_hbm = hbm_bytes * res["hbm"]["pj_per_byte_above_idle"] * 1e-12
    e_idle = res["idle_w"] * ms_p / 1e3
    res["pstep"] = {
        "k": k, "ms": ms_p, "j": j_p, "sm_mhz": clk, "power_w": pw,
        "model_j": {"dmma": e_dmma, "hbm": e_hbm, "idle": e_idle,
                    "sum": e_dmma + e_hbm + e_idle,
                    "other (instruction overhead, K2, L2/smem traffic)":
                        j_p - e_dmma - e_hbm - e_idle},
        "p_step_ms_at_1000w_if_only_dmma_hbm_idle":
            (e_dmma + e_hbm) / (1000.0 - res["idle_w"]) * 1e3,
    }
    res["how"] = ("NVML total energy over back-to-back runs, CUDA-event time; per-unit "
                  "energies above idle power; p-step count excludes the re-initialisation "
                  "copies (measured separately)")
    res["device"] = torch.cuda.get_device_name(0)
    p = ROOT / "profiles" / "r02" / "energy_probe.json"
    p.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
