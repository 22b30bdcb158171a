"""Chained back-to-back single-segment calls at small sizes (the
fixed per-launch cost): per-launch time and GB/s for 1/4/16/48/64 MiB, CUDA events,
best of 3 x 40 launches. Run once per library variant (HS_LIBHIST256)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
tot = 2 << 30
buf = torch.empty(tot, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", tot, 5), buf)
out = torch.empty((1, 256), dtype=torch.int64, device="cuda")
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
torch.cuda.synchronize()
row = []
for mib in (1, 4, 16, 48, 64, 256):
    size = mib << 20
    b0, b1 = np.zeros(1, np.uint64), np.full(1, size, np.uint64)
    best = 1e9
    for rep in range(3):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        a.record()
        reps = 40
        for k in range(reps):
            off = (k * size) % (tot - size)  # distinct bytes each launch (no L2 reuse)
            N.check(L.hs_histogram_batched(buf.data_ptr() + off, N.u64p(b0), N.u64p(b1), 1,
                                           N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, 0, None, None, 0, 0,
                                           out.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream), "x")
        z.record()
        z.synchronize()
        best = min(best, a.elapsed_time(z) / reps * 1e3)
    row.append(f"{mib} MiB {best:.2f} us ({size / best / 1e3:.0f} GB/s)")
assert int(out.sum().item()) == 256 << 20
print(os.environ.get("HS_LIBHIST256", "shipped"), " | ".join(row), flush=True)
