#!/usr/bin/env python
"""Build and run the FP64 pipe microbenchmark (fp64_peak.cu) while NVML samples the SM clock and
the clock-event (throttle) reasons every 20 ms; prints the benchmark's lines and a clocks record.

    python tools/microbench/run_fp64_peak.py > profiles/r02_fp64_peak_microbench.txt
"""
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent


def main():
    exe = HERE / "fp64_peak"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe),
                           str(HERE / "fp64_peak.cu")])
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
    samples, on = [], [True]

    def loop():
        while on[0]:
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.02)

    t = threading.Thread(target=loop, daemon=True)
    t.start()
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    on[0] = False
    t.join()
    print(out.stdout, end="")
    busy = [s for s in samples if s[2] > 300.0] or samples  # under load (power above idle)
    names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
    reasons = sorted({n for _, r, _ in busy for b, n in names.items() if r & b})
    print(f"clocks: sm_mhz median {statistics.median(s[0] for s in busy):.0f} (min {min(s[0] for s in busy)}, "
          f"max {max(s[0] for s in busy)}), sm_max_mhz {smax}, reasons {reasons}, "
          f"samples {len(busy)} under load of {len(samples)}, power max {max(s[2] for s in samples):.0f} W "
          f"(NVML, 20 ms)")
    return out.returncode


if __name__ == "__main__":
    sys.exit(main())
