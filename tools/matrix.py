"""Per-launch cost matrix of the production k_lane path: distribution x segments x kind,
10 back-to-back launches (ticketed + PDL) per cell, 1 GiB each; then the same cell
again after a sustained-load interval, with GPU / HBM temperature from NVML.

usage: python tools/matrix.py [SUSTAIN_SECONDS]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

try:
    import pynvml

    pynvml.nvmlInit()
    H = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:  # pragma: no cover
    H = None


def temps():
    if H is None:
        return {}
    out = {"gpu_c": pynvml.nvmlDeviceGetTemperature(H, 0),
           "sm_mhz": pynvml.nvmlDeviceGetClockInfo(H, 1), "mem_mhz": pynvml.nvmlDeviceGetClockInfo(H, 2)}
    try:
        fv = pynvml.nvmlDeviceGetFieldValues(H, [82])[0]  # NVML_FI_DEV_MEMORY_TEMP
        out["hbm_c"] = fv.value.uiVal if fv.nvmlReturn == 0 else None
    except Exception:
        pass
    return out


L = N.lib()
st = torch.cuda.current_stream()
n = 1 << 30
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
bufs = {}
for name, spec in (("uniform", hs.SourceSpec("uniform", n, 5)),
                   ("sigma8", hs.SourceSpec("normal", n, 5, mean=128.0, sigma=8.0)),
                   ("sigma32", hs.SourceSpec("normal", n, 5, mean=128.0, sigma=32.0)),
                   ("sigma64", hs.SourceSpec("normal", n, 5, mean=128.0, sigma=64.0)),
                   ("const127", hs.SourceSpec("constant", n, 5, value=127))):
    b = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(spec, b)
    bufs[name] = b
torch.cuda.synchronize()


def pattern_of(buf):
    c = torch.bincount(buf[: 1 << 24], minlength=256).cpu().numpy().astype(np.uint64)
    return hs.compute_binning_pattern(hs.Histogram256(c))


def cell(buf, nseg, kind, pat, reps=10, sleep=True):
    b0 = np.arange(nseg, dtype=np.uint64) * (n // nseg)
    b1 = b0 + n // nseg

    def call():
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, kind, N.HS_IMPL_LANE,
                                       N.i64p(pat.offset), N.i64p(pat.count), 960, 8, out.data_ptr(),
                                       ws.data_ptr(), ws.numel(), st.cuda_stream), "hist")

    for _ in range(3):
        call()
    if sleep:
        torch.cuda._sleep(20_000_000)  # queue all launches before the first runs
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        call()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


pats = {k: pattern_of(v) for k, v in bufs.items()}
uni = hs.uniform_pattern(960)
print("temps at start:", temps())
print(f"{'data':10s} {'nseg':>4s} {'kind':9s} {'hot_pattern':>11s} {'us/launch':>9s} {'TB/s':>6s}")
for name, buf in bufs.items():
    for nseg in (1, 64):
        for kind, pat, tag in ((N.HS_KIND_NAIVE, uni, "naive"), (N.HS_KIND_ADAPTIVE, pats[name], "adaptive")):
            us = cell(buf, nseg, kind, pat)
            print(f"{name:10s} {nseg:4d} {tag:9s} {'':>11s} {us:9.1f} {n / us / 1e6:6.3f}")

sustain = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
if sustain > 0:
    buf = bufs["sigma32"]
    t_end = time.time() + sustain
    k = 0
    while time.time() < t_end:
        cell(buf, 64, N.HS_KIND_NAIVE, uni, reps=2000, sleep=False)
        k += 2003
        print(f"after {k} sustained launches: sigma32 nseg64 naive {cell(buf, 64, N.HS_KIND_NAIVE, uni):.1f} us  {temps()}",
              flush=True)
