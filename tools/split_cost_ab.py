"""A/B of the cost-weighted CTA split (HS_SPLIT_COST builds, library from HS_LIBHIST256):
per-launch time of 1 GiB cut into 1 / 16 / 64 / 256 equal segments and 64 random-size
segments, ticketed, 10 back-to-back launches after a short idle (median of 5), counts
checked against torch.bincount once per layout.
usage: HS_LIBHIST256=tools/ablib/X.so python tools/split_cost_ab.py"""
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
ws = torch.zeros(int(L.hs_workspace_bytes(256)), dtype=torch.uint8, device="cuda")
out = torch.empty((256, 256), dtype=torch.int64, device="cuda")
tag = os.path.basename(os.environ.get("HS_LIBHIST256", "in-tree"))
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("normal", n, 5, mean=128.0, sigma=32.0), buf)
rng = np.random.default_rng(3)
layouts = {}
for k in (1, 16, 64, 256):
    b0 = np.arange(k, dtype=np.uint64) * (n // k)
    layouts[f"{k}x{(n // k) >> 20}MiB"] = (b0, b0 + np.uint64(n // k))
b0 = np.arange(256, dtype=np.uint64) * (1 << 20)
layouts["256x1MiB (256 MiB)"] = (b0, b0 + np.uint64(1 << 20))
b0 = np.arange(64, dtype=np.uint64) * (1 << 20)
layouts["64x1MiB (64 MiB)"] = (b0, b0 + np.uint64(1 << 20))
cuts = np.sort(4 * rng.integers(1, n // 4, 63)).astype(np.uint64)
layouts["64 random"] = (np.concatenate([[0], cuts]).astype(np.uint64), np.concatenate([cuts, [n]]).astype(np.uint64))
line = [tag]
for name, (b0, b1) in layouts.items():
    k = len(b0)

    def call():
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), k, N.HS_KIND_NAIVE,
                                       N.HS_IMPL_LANE, None, None, 0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       st.cuda_stream), "hist")

    call()
    torch.cuda.synchronize()
    got = out[:k].cpu().numpy()
    for s in (0, k // 2, k - 1):
        want = torch.bincount(buf[int(b0[s]):int(b1[s])], minlength=256).cpu().numpy()
        assert np.array_equal(got[s], want), (name, s)
    ts = []
    for _ in range(5):
        torch.cuda._sleep(20_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            call()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 10 * 1e3)
    line.append(f"{name} {np.median(ts):6.1f}")
    if k == 256 and name.startswith("256x1"):
        line[-1] += f" ({np.median(ts) / 256:.3f}/seg)"
print(" | ".join(line), flush=True)
