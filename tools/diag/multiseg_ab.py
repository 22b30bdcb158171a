"""Many-segment launches (CTAs that span several segments take one ticket per segment):
back-to-back chained calls of NSEG segments of SEG bytes each, CUDA events, best of 3 x
20 calls, bins checked against torch.bincount on sampled segments. Library from
HS_LIBHIST256 (tools/ab_build.sh variants) or the shipped one."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
s = torch.cuda.current_stream()
row = []
for nseg, seg in ((256, 1 << 20), (256, 64 << 10), (64, 16 << 20), (200, 4 << 10)):
    buf = torch.empty(nseg * seg, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("uniform", buf.numel(), 3), buf)
    b0 = np.arange(nseg, dtype=np.uint64) * seg
    b1 = b0 + seg
    out = torch.zeros((nseg, 256), dtype=torch.int64, device="cuda")
    ws = torch.zeros(int(L.hs_workspace_bytes(nseg)), dtype=torch.uint8, device="cuda")
    kind = N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED

    def call():
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, kind, 0, None, None, 0, 0,
                                       out.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream), "x")

    for _ in range(3):
        call()
    best = 1e9
    for _ in range(3):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        a.record()
        for _ in range(20):
            call()
        z.record()
        z.synchronize()
        best = min(best, a.elapsed_time(z) / 20 * 1e3)
    for k in (0, nseg // 2, nseg - 1):
        want = torch.bincount(buf[k * seg:(k + 1) * seg], minlength=256)
        assert torch.equal(want, out[k]), (nseg, seg, k)
    row.append(f"{nseg}x{seg >> 10}KiB {best:.2f} us ({nseg * seg / best / 1e3:.0f} GB/s)")
print(os.environ.get("HS_LIBHIST256", "shipped"), " | ".join(row), flush=True)
