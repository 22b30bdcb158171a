"""Cost of segment boundaries: back-to-back launches over the same 1 GiB split into
1/4/16/64 equal segments (ticketed output, PDL), GPU time per launch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
s = torch.cuda.current_stream().cuda_stream
n = 1 << 30
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("normal", n, 3, mean=128.0, sigma=32.0), buf)
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
pat = hs.uniform_pattern(960)
side = torch.cuda.Stream()
for nseg in (64,):
    b0 = (np.arange(nseg, dtype=np.uint64) * (n // nseg))
    b1 = b0 + n // nseg
    for kind, st, blocked in ((N.HS_KIND_ADAPTIVE, s, True), (N.HS_KIND_ADAPTIVE, side.cuda_stream, True),
                              (N.HS_KIND_ADAPTIVE, side.cuda_stream, False)):
        def call():
            N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, kind, 0, N.i64p(pat.offset),
                                           N.i64p(pat.count), 960, 8, out.data_ptr(), ws.data_ptr(), ws.numel(), st), "x")
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        ts = torch.cuda.ExternalStream(st) if st != s else torch.cuda.current_stream()
        if blocked:
            with torch.cuda.stream(ts):
                torch.cuda._sleep(50_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ts)
        for _ in range(10):
            call()
        b.record(ts)
        b.synchronize()
        us = a.elapsed_time(b) / 10 * 1e3
        print(f"nseg={nseg:3d} kind={kind} stream={'default' if st == s else 'side'} queue_blocked={blocked} {us:8.1f} us/launch  {n / us / 1e3:7.1f} GB/s")
