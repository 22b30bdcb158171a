"""Per-call costs of hs_histogram_batched: host submission time (wall clock per call in
a tight loop) and pure GPU time (events recorded while a sleep kernel keeps the GPU
busy, so host latency is excluded)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
s = torch.cuda.current_stream().cuda_stream
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
pat = hs.uniform_pattern(960)
off, cnt = N.i64p(pat.offset), N.i64p(pat.count)
for n in (1 << 10, 1 << 20, 16 << 20, 256 << 20, 1 << 30):
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("uniform", n, 3), buf)
    b0 = np.zeros(1, np.uint64)
    b1 = np.full(1, n, np.uint64)

    def call(kind=N.HS_KIND_ADAPTIVE):
        return L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), 1, kind, 0, off, cnt, 960, 8,
                                      out.data_ptr(), ws.data_ptr(), ws.numel(), s)

    for _ in range(5):
        call()
    torch.cuda.synchronize()
    reps = 200 if n <= (16 << 20) else 20
    torch.cuda._sleep(int(2e9))  # ~1 s of GPU work: the host loop below never waits
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    host_us = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    # GPU time: sleep keeps the queue busy while a / launches / b are enqueued
    gpu = []
    for _ in range(5):
        torch.cuda._sleep(int(5e7))
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            call()
        b.record()
        b.synchronize()
        gpu.append(a.elapsed_time(b) / 10 * 1e3)
    g = float(np.median(gpu))
    print(f"n={n:>11d}  host {host_us:7.2f} us/call   gpu {g:8.2f} us/launch   {n / g / 1e3:8.1f} GB/s (back-to-back)")
    del buf
