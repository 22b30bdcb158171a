"""Small chained calls with rotated workspaces (DESIGN §10 item 2): per-launch time of
back-to-back single-segment calls when each call uses its own workspace slice (K
slices in rotation) and its own output row. Run with HS_LIBHIST256 pointing at a
variant build; CUDA events, best of 3 x 64 launches."""
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
K = int(os.environ.get("HS_AB_SLOTS", "8"))
# AB_WAIT=1: plain calls (each waits for its predecessor before loading) instead of chained ones
KIND = N.HS_KIND_NAIVE | (0 if os.environ.get("AB_WAIT") else N.HS_KIND_FLAG_CHAINED)
wsb = int(L.hs_workspace_bytes(64))
ws = torch.zeros(K * wsb, dtype=torch.uint8, device="cuda")
reps = 64
out = torch.zeros((reps, 256), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
torch.cuda.synchronize()
row = []
SIZES_KIB = [int(x) for x in os.environ.get("AB_KIB", "").split(",") if x] or \
    [m << 10 for m in (1, 4, 8, 16, 24, 32, 48, 64, 256)]
for kib in SIZES_KIB:
    size = kib << 10
    mib = kib / 1024
    b0, b1 = np.zeros(1, np.uint64), np.full(1, size, np.uint64)
    best = 1e9
    for rep in range(3):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        a.record()
        for k in range(reps):
            off = (k * size) % (tot - size)
            N.check(L.hs_histogram_batched(buf.data_ptr() + off, N.u64p(b0), N.u64p(b1), 1,
                                           KIND, 0, None, None, 0, 0,
                                           out[k].data_ptr(), ws.data_ptr() + (k % K) * wsb, wsb,
                                           s.cuda_stream), "x")
        z.record()
        z.synchronize()
        best = min(best, a.elapsed_time(z) / reps * 1e3)
    if os.environ.get("AB_NOCHECK"):
        row.append(f"{mib:g} MiB {best:.2f} us ({size / best / 1e3:.0f} GB/s)")
        continue
    sums = out.sum(dim=1).cpu().numpy()
    assert (sums == size).all(), (mib, sums[:8])
    want = torch.stack([torch.bincount(buf[(k * size) % (tot - size):(k * size) % (tot - size) + size], minlength=256)
                        for k in range(0, reps, 13)])
    assert torch.equal(want, out[0:reps:13]), "bins differ"
    assert all(not ws[k * wsb + 384:(k + 1) * wsb].any().item() for k in range(K)), "workspace slots not left zero"
    row.append(f"{mib:g} MiB {best:.2f} us ({size / best / 1e3:.0f} GB/s)")
print(os.environ.get("HS_LIBHIST256", "shipped"), f"K={K}", " | ".join(row), flush=True)
