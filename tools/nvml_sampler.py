"""Out-of-process NVML clock sampler for bench.py: prints "ready" after its
first sample, samples every PERIOD seconds until stdin closes or says
"stop", then prints one JSON list of [sm_mhz, max_mhz, reasons] samples.
A separate process keeps the sampling off the benchmark's interpreter (no
GIL hand-offs inside the timed region)."""
import json
import sys
import threading

import pynvml as N


def main():
    idx, period = int(sys.argv[1]), float(sys.argv[2])
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(idx)
    mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
    reasons_fn = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
        getattr(N, "nvmlDeviceGetCurrentClocksThrottleReasons")
    stop = threading.Event()
    threading.Thread(target=lambda: (sys.stdin.readline(), stop.set()), daemon=True).start()
    samples = []

    def sample():
        samples.append([float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)), mx,
                        int(reasons_fn(h))])

    sample()
    print("ready", flush=True)
    while not stop.wait(period):
        sample()
    sample()
    print(json.dumps(samples), flush=True)
    N.nvmlShutdown()


if __name__ == "__main__":
    main()
