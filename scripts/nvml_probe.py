"""Time the NVML calls the bench's clock sampler makes (per-call latency on this box)."""
import time

import pynvml as nv

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
for name, fn in (("clock_info", lambda: nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                 ("clock_current", lambda: nv.nvmlDeviceGetClock(h, nv.NVML_CLOCK_SM, nv.NVML_CLOCK_ID_CURRENT)),
                 ("event_reasons", lambda: nv.nvmlDeviceGetCurrentClocksEventReasons(h))):
    ts = []
    for _ in range(20):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    ts.sort()
    print(f"{name:14s} median {ts[10] * 1e3:.2f} ms, max {ts[-1] * 1e3:.2f} ms")
