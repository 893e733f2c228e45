"""Measure sustained FP64 DMMA and DFMA rates on this GPU (dev tool)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_2720_b200 import _lib  # noqa: E402
from tools.dev import devlib  # noqa: E402


def main():
    _lib.require_cuda()
    lib = devlib.load()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = []
    for kind, name, per in ((0, "dmma", 256), (1, "dfma", 32)):
        for wps in (1, 2, 4, 8, 16, 32):
            iters = 20000 if kind == 0 else 100000
            ctas = sms * max(1, wps // 4)
            threads = 32 * min(wps, 4)
            for rep in range(2):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.check(lib.jh_probe_rate(kind, ctas, threads, iters, out.data_ptr(),
                                             _lib.stream_handle()), "rate")
                e1.record()
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            fma = ctas * threads / 32 * iters * 8 * per
            r = {"kind": name, "warps_per_sm": wps, "tflops": 2 * fma / ms / 1e9}
            print(json.dumps(r), flush=True)
            res.append(r)
    return res


def timed(lib, kind, ctas, threads, iters, out):
    for rep in range(2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.jh_probe_rate(kind, ctas, threads, iters, out.data_ptr(),
                                     _lib.stream_handle()), "rate")
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def chains_and_mixed():
    """DMMA rate vs independent chains per warp (1 warp per SMSP, i.e. 4 per
    SM, and 1 per SM), and DMMA + DFMA warps side by side."""
    _lib.require_cuda()
    lib = devlib.load()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk = torch.cuda.clock_rate() if hasattr(torch.cuda, "clock_rate") else None
    iters = 20000
    for wps in (1, 4, 8):
        for c in (1, 2, 4, 8, 16):
            kind = {1: 11, 2: 12, 4: 14, 8: 18, 16: 26}[c]
            ctas, threads = sms * max(1, wps // 4), 32 * min(wps, 4)
            ms = timed(lib, kind, ctas, threads, iters, out)
            fma = ctas * threads / 32 * iters * 8 * 256
            tf = 2 * fma / ms / 1e9
            # cycles per dependent DMMA of one chain at the observed rate
            ns_per = ms * 1e6 / (iters * 8 / c)
            print(json.dumps({"probe": "dmma_chains", "warps_per_sm": wps, "chains": c,
                              "tflops": tf, "ns_per_chain_step": ns_per}), flush=True)
    for wps in (8, 16):
        ctas, threads = sms * (wps // 8), 256
        ms = timed(lib, 2, ctas, threads, iters, out)
        fma = ctas * threads / 32 * iters * 8 * 256  # same per warp for both halves
        print(json.dumps({"probe": "dmma+dfma", "warps_per_sm": wps,
                          "tflops_combined": 2 * fma / ms / 1e9}), flush=True)




def latency():
    _lib.require_cuda()
    lib = devlib.load()
    out = torch.zeros(9, dtype=torch.float64, device="cuda")
    for _ in range(2):
        _lib.check(lib.jh_probe_latency(out.data_ptr(), _lib.stream_handle()), "lat")
        torch.cuda.synchronize()
    names = ["dfma", "dmul", "ddiv", "dsqrt", "rotation_core", "lds", "div_fp", "sqrt_fp",
             "rotation_core_fast"]
    r = dict(zip(names, out.cpu().tolist()))
    print(json.dumps({"latency_cycles": r}))
    return r




def peak_with_clock(out_path="profiles/r02/dmma_rate.json", seconds=6.0):
    """Sustained DMMA rate (8 warps per SM, 8 independent chains each) for
    ~`seconds`, with nvidia-smi sampling the SM clock meanwhile: the FP64
    tensor roofline denominator bench.py reports."""
    import subprocess
    import tempfile
    import time
    from pathlib import Path

    _lib.require_cuda()
    lib = devlib.load()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ctas, threads, iters = sms * 2, 128, 20000
    per = 256
    ms = timed(lib, 0, ctas, threads, iters, out)
    reps = max(1, int(seconds * 1e3 / max(ms, 1e-3)))
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,"
                            "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=f, stderr=subprocess.DEVNULL)
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _lib.check(lib.jh_probe_rate(0, ctas, threads, iters, out.data_ptr(),
                                     _lib.stream_handle()), "rate")
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    smi.wait()
    tot = e0.elapsed_time(e1)
    fma = ctas * threads / 32 * iters * 8 * per * reps
    clocks = []
    for line in Path(f.name).read_text().splitlines():
        try:
            clocks.append(float(line.split(",")[0]))
        except ValueError:
            pass
    clocks = sorted(clocks)
    r = {"dmma_tflops": 2 * fma / tot / 1e9, "seconds": tot / 1e3,
         "sm_mhz": clocks[len(clocks) // 2] if clocks else None,
         "how": ("mma.sync.m8n8k4.f64 (SASS DMMA), 2 CTAs x 4 warps per SM, 8 independent "
                 "accumulator chains per warp, back to back for ~6 s (tools/dev/csrc/jh_probe.cu)"),
         "device": torch.cuda.get_device_name(0)}
    Path(out_path).parent.mkdir(parents=True, exist_ok=True)
    Path(out_path).write_text(json.dumps(r, indent=1) + "\n")
    print(json.dumps(r), flush=True)
    return r


if __name__ == "__main__":
    if "--chains" in sys.argv:
        chains_and_mixed()
    elif "--latency" in sys.argv:
        latency()
    elif "--peak" in sys.argv:
        peak_with_clock()
    else:
        main()
