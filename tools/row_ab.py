"""A/B of k_lane builds (library from HS_LIBHIST256): per-launch time of 10 back-to-back
1 GiB launches (64 segments, ticketed) per distribution/kind after a 1 s idle settle,
then a sustained phase (back-to-back launches for SECONDS) with NVML clock and power.
Counts are checked against torch.bincount once per distribution.
usage: HS_LIBHIST256=tools/ablib/X.so python tools/row_ab.py [SECONDS]"""
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
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
tag = os.path.basename(os.environ.get("HS_LIBHIST256", "in-tree"))
L = N.lib()
n = 1 << 30
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
b0 = np.arange(64, dtype=np.uint64) * (n // 64)
b1 = b0 + n // 64
st = torch.cuda.current_stream().cuda_stream


def launch(kind, pat):
    if pat is None:
        off = cnt = None
        ts = cap = 0
    else:
        off, cnt = N.i64p(np.asarray(pat.offset, np.int64)), N.i64p(np.asarray(pat.count, np.int64))
        ts, cap = pat.total_slots, pat.cap
    N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), 64, kind, N.HS_IMPL_LANE,
                                   off, cnt, ts, cap, out.data_ptr(), ws.data_ptr(), ws.numel(), st), "h")


def timed(kind, pat, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        launch(kind, pat)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


cases = [("uniform", {}), ("normal", {"mean": 128.0, "sigma": 32.0}), ("normal", {"mean": 128.0, "sigma": 8.0}),
         ("constant", {"value": 127})]
for dist, kw in cases:
    hs.generate_device(hs.SourceSpec(dist, n, 3, **kw), buf)
    ref = torch.bincount(buf.view(64, -1)[0].to(torch.int64), minlength=256)
    hist = hs.Histogram256(torch.bincount(buf.to(torch.int64), minlength=256).cpu().numpy().astype(np.uint64))
    pat = hs.compute_binning_pattern(hist)
    for kname, kind, p in (("NAIVE", N.HS_KIND_NAIVE, None), ("ADAPTIVE", N.HS_KIND_ADAPTIVE, pat)):
        launch(kind, p)
        torch.cuda.synchronize()
        ok = bool(torch.equal(out[0], ref))
        time.sleep(1.0)
        us = timed(kind, p, 10)
        print(f"{tag:10s} {dist:8s} {kw.get('sigma', ''):>4} {kname:8s} {us:7.1f} us/launch "
              f"{n / us / 1e3:7.1f} GB/s  ok={ok}", flush=True)

# sustained: normal sigma 32, NAIVE
hs.generate_device(hs.SourceSpec("normal", n, 3, mean=128.0, sigma=32.0), buf)
time.sleep(1.0)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(H, 1), pynvml.nvmlDeviceGetPowerUsage(H) / 1e3))
        time.sleep(0.05)


th = threading.Thread(target=sampler, daemon=True)
th.start()
t0 = time.time()
res = []
while time.time() - t0 < secs:
    res.append((time.time() - t0, timed(N.HS_KIND_NAIVE, None, 50)))
stop.set()
th.join()
late = [us for t, us in res if t > secs / 3]
sm = [c for t, c, p in samples if t - t0 > secs / 3]
pw = [p for t, c, p in samples if t - t0 > secs / 3]
print(f"{tag:10s} sustained {secs:.0f}s: {np.mean(late):7.1f} us/launch {n / np.mean(late) / 1e3:7.1f} GB/s "
      f"sm_mhz median {np.median(sm):.0f} power median {np.median(pw):.0f} W", flush=True)
