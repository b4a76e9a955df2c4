"""Developer tool: latency of the NVML queries the bench's ClockSampler makes."""
import time
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name, fn in (("clock", lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                 ("reasons", lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))):
    ts = []
    for _ in range(50):
        t = time.perf_counter(); fn(); ts.append(time.perf_counter() - t)
    ts.sort()
    print(f"{name}: median {ts[25]*1e3:.3f} ms, max {ts[-1]*1e3:.3f} ms")
