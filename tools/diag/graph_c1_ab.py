"""C1's graph-replayed single-image calls (bench_extras.c1_image): 100 chained 1 MiB
calls on ONE workspace captured in a CUDA graph, replayed; per-call time, best and
median of 7 replays. Library from HS_LIBHIST256 or the shipped one."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
n = 1 << 20
imgs = torch.empty(n, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", n, 0), imgs)
ws = torch.zeros(int(L.hs_workspace_bytes(256)), dtype=torch.uint8, device="cuda")
one0, one1 = np.zeros(1, np.uint64), np.full(1, n, np.uint64)
out1 = torch.empty((1, 256), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
cs = torch.cuda.Stream()
cs.wait_stream(s)
with torch.cuda.stream(cs):
    N.check(L.hs_histogram_batched(imgs.data_ptr(), N.u64p(one0), N.u64p(one1), 1, N.HS_KIND_NAIVE, 0, None, None,
                                   0, 0, out1.data_ptr(), ws.data_ptr(), ws.numel(), cs.cuda_stream), "warm")
s.wait_stream(cs)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    gs = torch.cuda.current_stream()
    for _ in range(100):
        N.check(L.hs_histogram_batched(imgs.data_ptr(), N.u64p(one0), N.u64p(one1), 1,
                                       N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, 0, None, None, 0, 0,
                                       out1.data_ptr(), ws.data_ptr(), ws.numel(), gs.cuda_stream), "capture")
g.replay()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b) / 100 * 1e3)
assert np.array_equal(out1[0].cpu().numpy(), torch.bincount(imgs, minlength=256).cpu().numpy())
print(os.environ.get("HS_LIBHIST256", "shipped"), f"graph single image: best {min(ts):.3f} us, median {np.median(ts):.3f} us",
      [round(t, 3) for t in ts], flush=True)
