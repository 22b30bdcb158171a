"""Sustained-load probe: back-to-back 1 GiB k_lane launches for N seconds while NVML is
sampled every 100 ms (SM/memory clock, power, enforced power limit, throttle reasons,
temperatures). Shows when and why the SM clock leaves its maximum under this kernel.
usage: python tools/power_probe.py [SECONDS]"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402
import pynvml  # noqa: E402

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)
REASONS = {0x1: "gpu_idle", 0x2: "app_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
           0x20: "sw_thermal", 0x40: "hw_thermal", 0x80: "hw_power_brake", 0x100: "display_clocks"}
print("power limit (enforced) W:", pynvml.nvmlDeviceGetEnforcedPowerLimit(H) / 1e3,
      " default:", pynvml.nvmlDeviceGetPowerManagementDefaultLimit(H) / 1e3,
      " max clocks sm/mem:", pynvml.nvmlDeviceGetMaxClockInfo(H, 1), pynvml.nvmlDeviceGetMaxClockInfo(H, 2), flush=True)
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
L = N.lib()
n = 1 << 30
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("normal", n, 3, mean=128.0, sigma=32.0), buf)
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
b0 = np.arange(64, dtype=np.uint64) * (n // 64)
b1 = b0 + n // 64
st = torch.cuda.current_stream().cuda_stream
samples = []
stop = threading.Event()


def sampler():
    t0 = time.time()
    while not stop.is_set():
        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(H)
        samples.append((time.time() - t0, pynvml.nvmlDeviceGetClockInfo(H, 1), pynvml.nvmlDeviceGetClockInfo(H, 2),
                        pynvml.nvmlDeviceGetPowerUsage(H) / 1e3, pynvml.nvmlDeviceGetTemperature(H, 0),
                        [v for k, v in REASONS.items() if r & k]))
        time.sleep(0.1)


th = threading.Thread(target=sampler, daemon=True)
th.start()
t_end = time.time() + secs
launches = 0
evs = []
while time.time() < t_end:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), 64, N.HS_KIND_NAIVE, N.HS_IMPL_LANE,
                                       None, None, 0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(), st), "h")
    b.record()
    b.synchronize()
    launches += 50
    evs.append((time.time(), a.elapsed_time(b) / 50 * 1e3))
stop.set()
th.join()
t0 = evs[0][0]
for i in range(0, len(samples), 5):
    t, sm, mem, pw, tc, rs = samples[i]
    near = [us for (te, us) in evs if abs(te - t0 - t) < 0.2]
    print(f"t={t:5.1f}s sm={sm:4d} mem={mem:4d} MHz power={pw:6.1f} W temp={tc}C reasons={rs} "
          f"us/launch={np.mean(near) if near else float('nan'):.1f}")
