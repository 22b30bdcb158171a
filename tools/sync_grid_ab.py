"""Blocking-call latency (hs_histogram_sync, device data, page-locked result) by input
size, for A/B of the latency grid rule (library from HS_LIBHIST256); mean of 300 calls.
usage: HS_LIBHIST256=tools/ablib/X.so python tools/sync_grid_ab.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
tag = os.path.basename(os.environ.get("HS_LIBHIST256", "in-tree"))
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("normal", 256 << 20, 1, mean=128.0, sigma=32.0), big)
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
d_out = torch.empty((1, 256), dtype=torch.int64, device="cuda")
h = torch.empty(256, dtype=torch.int64).pin_memory()
hp = ctypes.cast(h.data_ptr(), N._U64P)
st = torch.cuda.current_stream().cuda_stream
line = [f"{tag:12s}"]
for mib in (1, 4, 16, 64, 256):
    n = mib << 20
    b0, b1 = np.zeros(1, np.uint64), np.full(1, n, np.uint64)
    args = (big.data_ptr(), N.u64p(b0), N.u64p(b1), 1, 0, 0, None, None, 0, 0, d_out.data_ptr(), hp, ws.data_ptr(),
            ws.numel(), st)
    for _ in range(20):
        L.hs_histogram_sync(*args)
    reps = 300 if mib < 64 else 100
    t0 = time.perf_counter()
    for _ in range(reps):
        L.hs_histogram_sync(*args)
    us = (time.perf_counter() - t0) / reps * 1e6
    assert np.array_equal(h.numpy(), torch.bincount(big[:n], minlength=256).cpu().numpy())
    line.append(f"{mib}MiB {us:7.1f}us {n / us / 1e3:6.0f}GB/s")
print(" | ".join(line), flush=True)
