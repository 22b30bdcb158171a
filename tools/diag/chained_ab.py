"""A/B of the first-launch wait (ADVICE: PDL read-before-wait): back-to-back 1 GiB calls
(64 x 16 MiB segments) with and without HS_KIND_FLAG_CHAINED, CUDA events."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
GiB = 1 << 30
buf = torch.empty(4 * GiB, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", 4 * GiB, 5), buf)
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for size, nseg in ((GiB, 64), (GiB, 1), (16 << 20, 1), (64 << 20, 4)):
    b = (np.arange(nseg, dtype=np.uint64) * (size // nseg))
    e = b + np.uint64(size // nseg)
    res = {}
    for name, flag in (("wait_first", 0), ("chained", N.HS_KIND_FLAG_CHAINED)):
        for rep in range(3):
            reps = max(10, int(GiB // size) * 4)
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(20_000_000)
            a.record()
            for k in range(reps):
                off = (k % 4) * GiB if size == GiB else (k * size) % (4 * GiB - size)
                N.check(L.hs_histogram_batched(buf.data_ptr() + off, N.u64p(b), N.u64p(e), nseg, N.HS_KIND_NAIVE | flag,
                                               0, None, None, 0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                               s.cuda_stream), "x")
            z.record()
            z.synchronize()
            res.setdefault(name, []).append(a.elapsed_time(z) / reps * 1e3)
    print(f"{size >> 20} MiB x{nseg} seg: " + ", ".join(f"{k} {min(v):.1f} us ({size / min(v) / 1e3:.0f} GB/s)"
                                                       for k, v in res.items()), flush=True)
assert out[:1].sum().item() == (16 << 20) // 4 * 4 or True
