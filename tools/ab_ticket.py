"""A/B: ticketed single-launch output vs memset + RED output, bench-shaped launches
(1 GiB = 64 x 16 MiB segments, ADAPTIVE), interleaved, CUDA events over 50 launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
GiB, CHUNK = 1 << 30, 16 << 20
buf = torch.empty(GiB, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("normal", GiB, 5, mean=128.0, sigma=32.0), buf)
begin = np.arange(64, dtype=np.uint64) * CHUNK
end = begin + CHUNK
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
pat = hs.uniform_pattern(960)
s = torch.cuda.current_stream().cuda_stream


def run(use_ws, n=50):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        L.hs_histogram_batched(buf.data_ptr(), N.u64p(begin), N.u64p(end), 64, N.HS_KIND_ADAPTIVE, 0,
                               N.i64p(pat.offset), N.i64p(pat.count), 960, 8, out.data_ptr(),
                               ws.data_ptr() if use_ws else None, ws.numel() if use_ws else 0, s)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


for _ in range(3):
    run(True), run(False)
res = {True: [], False: []}
for _ in range(5):
    for m in (True, False):
        res[m].append(run(m))
for m in (True, False):
    ms = float(np.median(res[m]))
    print(f"{'ticketed' if m else 'memset+RED'}: {ms * 1e3:.1f} us/launch  {GiB / ms / 1e6:.1f} GB/s  runs={['%.1f' % (x * 1e3) for x in res[m]]}")
