"""Segment-boundary A/B: per-launch time of 1 GiB as 1 or 64 segments, ticketed
(workspace) or memset + RED, 10 back-to-back launches; library from HS_LIBHIST256."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
st = torch.cuda.current_stream()
n = 1 << 30
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
uni = hs.uniform_pattern(960)
tag = os.path.basename(os.environ.get("HS_LIBHIST256", "in-tree"))
res = []
for name, spec in (("uniform", hs.SourceSpec("uniform", n, 5)),
                   ("sigma32", hs.SourceSpec("normal", n, 5, mean=128.0, sigma=32.0))):
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(spec, buf)
    for nseg in (1, 64):
        b0 = np.arange(nseg, dtype=np.uint64) * (n // nseg)
        b1 = b0 + n // nseg
        for use_ws in (True, False):
            def call():
                N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, N.HS_KIND_NAIVE,
                                               N.HS_IMPL_LANE, None, None, 0, 0, out.data_ptr(),
                                               ws.data_ptr() if use_ws else None, ws.numel() if use_ws else 0,
                                               st.cuda_stream), "hist")
            for _ in range(3):
                call()
            ts = []
            for _ in range(3):
                torch.cuda._sleep(20_000_000)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(10):
                    call()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b) / 10 * 1e3)
            print(f"{tag:18s} {name:8s} nseg={nseg:2d} {'ticket' if use_ws else 'memset':6s} {np.median(ts):7.1f} us", flush=True)
    del buf
