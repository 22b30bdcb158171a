"""Per-launch device time vs input size (one segment, NAIVE, uniform bytes): 10
launches captured in a CUDA graph, median of 5 replays. Fits t = fixed + bytes/rate
to separate the per-launch fixed cost from the streaming rate."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

impl = {"lane": N.HS_IMPL_LANE, "warp": N.HS_IMPL_WARP}[sys.argv[1] if len(sys.argv) > 1 else "lane"]
L = N.lib()
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", big.numel(), 1), big)
ws = D.default_staging().workspace()
out = torch.empty((1, 256), dtype=torch.int64, device="cuda")
rows = []
for mib in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1024):
    n = mib << 20
    b0 = np.zeros(1, np.uint64)
    b1 = np.full(1, n, np.uint64)

    def call(s):
        N.check(L.hs_histogram_batched(big.data_ptr(), N.u64p(b0), N.u64p(b1), 1, N.HS_KIND_NAIVE, impl, None, None,
                                       0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(), s), "h")

    side = torch.cuda.Stream()
    call(side.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(10):
            call(torch.cuda.current_stream().cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 10 * 1e3)
    us = float(np.median(ts))
    rows.append((n, us))
    print(f"{mib:5d} MiB {us:9.2f} us/launch {n / us / 1e3:8.1f} GB/s", flush=True)
x = np.array([r[0] for r in rows], float)
y = np.array([r[1] for r in rows], float)
A = np.vstack([np.ones_like(x), x]).T
fixed, per = np.linalg.lstsq(A[-5:], y[-5:], rcond=None)[0]
print(f"fit over >= 32 MiB: fixed {fixed:.2f} us per launch, streaming {1e-3 / per:.1f} GB/s")
