#!/usr/bin/env python3
"""fp64 pipe peaks of this B200 with the SM clock recorded beside them (the roofline denominator
of bench.py for the fp64-bound configs).

Runs tools/fp64_peaks (DFMA, DMMA m8n8k4 f64, both interleaved) twice: a burst pass (5 timed
launches per test, ~1-13 ms) and a sustained pass (REPS launches per test, seconds each), while an
NVML thread samples the SM clock, power and clock-event reasons every 5 ms.  The samples taken
between two result lines belong to the test of the second line.  Output:
profiles/fp64_peaks_<tag>.json.

    python tools/fp64_peaks.py [tag] [reps]
"""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}


def run_pass(binary, reps):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            try:
                samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    t = threading.Thread(target=sampler, daemon=True)
    t.start()
    p = subprocess.Popen([binary, str(reps)], stdout=subprocess.PIPE, text=True)
    header, tests, t_prev = None, [], time.time()
    for ln in p.stdout:
        now = time.time()
        d = json.loads(ln)
        if "test" not in d:
            header, t_prev = d, now
            continue
        win = [s for s in samples if t_prev <= s[0] <= now]
        bits = 0
        for s in win:
            bits |= s[3]
        d["clocks"] = {"sm_mhz_median": statistics.median([s[1] for s in win]) if win else None,
                       "sm_mhz_min": min((s[1] for s in win), default=None),
                       "power_w_median": statistics.median([s[2] for s in win]) if win else None,
                       "reasons": [n for b, n in REASONS.items() if bits & b], "samples": len(win)}
        tests.append(d)
        t_prev = now
    p.wait()
    stop.set()
    t.join()
    return {"header": header, "max_sm_mhz": pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM),
            "tests": tests}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    binary = os.path.join(HERE, "fp64_peaks")
    if not os.path.exists(binary):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", binary,
                        os.path.join(HERE, "fp64_peaks.cu")], check=True)
    burst = run_pass(binary, 5)
    sustained = run_pass(binary, reps)
    best = lambda res, name: max((t for t in res["tests"] if t["test"] == name), key=lambda t: t["tflops"])  # noqa: E731
    out = {"what": "fp64 pipe peaks (tools/fp64_peaks.cu) with NVML SM clock / power / reasons sampled per test",
           "burst": burst, "sustained": sustained,
           "dmma_burst_tflops": best(burst, "dmma")["tflops"], "dfma_burst_tflops": best(burst, "dfma")["tflops"],
           "dmma_sustained_tflops": best(sustained, "dmma")["tflops"],
           "dfma_sustained_tflops": best(sustained, "dfma")["tflops"],
           "dmma_sustained_clocks": best(sustained, "dmma")["clocks"],
           "dfma_sustained_clocks": best(sustained, "dfma")["clocks"]}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", f"fp64_peaks_{tag}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("burst", "sustained")}))


if __name__ == "__main__":
    main()
