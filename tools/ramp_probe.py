"""Throughput ramp under sustained bench-shaped load: 1000 bench steps (3 x 1 GiB on three
streams), CUDA events every 20 steps, NVML sampled every 2 ms (SM clock, memory clock,
power, throttle reasons). Shows when throughput leaves its fresh-GPU level and why."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ab_step  # noqa: E402  (builds the bench-shaped inputs)
import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def poll():
    t0 = time.perf_counter()
    while not stop.is_set():
        samples.append((time.perf_counter() - t0, pynvml.nvmlDeviceGetClockInfo(h, 1), pynvml.nvmlDeviceGetClockInfo(h, 2),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1e3, pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.002)


th = threading.Thread(target=poll, daemon=True)
torch.cuda.synchronize()
th.start()
time.sleep(0.05)
t_start = time.perf_counter()
marks = []
for blk in range(50):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    ms, gbs = ab_step.run("three", steps=20, warm=0)
    marks.append((time.perf_counter() - t_start, gbs))
stop.set()
th.join()
off = samples[0][0]
print("t_host_s  GB/s   | nearest NVML sample: sm_mhz mem_mhz power_W reasons")
for t, g in marks:
    near = min(samples, key=lambda s: abs(s[0] - 0.05 - t))
    print(f"{t:7.3f} {g:7.1f} | {near[1]:5d} {near[2]:5d} {near[3]:6.1f} {hex(near[4])}")
