"""Host cost of one hs_histogram_batched call (ctypes + SegParams + cudaLaunchKernelEx),
measured while the GPU is held busy by a sleep kernel so the launch queue never blocks:
1 and 64 segments, 16 MiB total, NAIVE, chained, one workspace."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
buf = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
ws = torch.zeros(int(L.hs_workspace_bytes(256)), dtype=torch.uint8, device="cuda")
out = torch.zeros((256, 256), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for nseg in (1, 64, 256):
    b0 = (np.arange(nseg, dtype=np.uint64) * np.uint64((16 << 20) // nseg))
    b1 = b0 + np.uint64((16 << 20) // nseg)
    pb, pe = N.u64p(b0), N.u64p(b1)
    for rep in range(2):
        torch.cuda._sleep(200_000_000)  # ~100 ms of GPU time ahead of the calls
        t0 = time.perf_counter()
        for _ in range(100):
            L.hs_histogram_batched(buf.data_ptr(), pb, pe, nseg, N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, 0, None,
                                   None, 0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(), s)
        dt = (time.perf_counter() - t0) / 100 * 1e6
        torch.cuda.synchronize()
    print(f"{nseg:4d} segments: {dt:.1f} us host time per call", flush=True)
