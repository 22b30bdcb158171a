"""One libhist256 configuration, timed with CUDA events (development / ncu target).

usage: python tools/kbench.py DIST KIND IMPL [NBYTES] [REPS]
  DIST uniform|normal8|normal32|normal64|const127   KIND naive|adaptive
  IMPL auto|lane|warp|subbin
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1011_0235_b200 import _native as N  # noqa: E402

dist, kind, impl = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 30
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
L = N.lib()
s = torch.cuda.current_stream().cuda_stream
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
out = torch.empty(256, dtype=torch.int64, device="cuda")
if dist == "uniform":
    N.check(L.hs_generate_device(N.HS_GEN_UNIFORM, 7, 0, 0.0, 1.0, 0, buf.data_ptr(), n, s), "gen")
elif dist.startswith("normal"):
    N.check(L.hs_generate_device(N.HS_GEN_NORMAL, 7, 0, 128.0, float(dist[6:]), 0, buf.data_ptr(), n, s), "gen")
else:
    N.check(L.hs_generate_device(N.HS_GEN_CONSTANT, 7, int(dist[5:]), 0.0, 1.0, 0, buf.data_ptr(), n, s), "gen")
ref = torch.bincount(buf, minlength=256).cpu().numpy().astype(np.uint64)
off = np.zeros(256, np.int64)
cnt = np.zeros(256, np.int64)
N.check(L.hs_binning_pattern(N.u64p(ref), 960, 8, N.i64p(off), N.i64p(cnt)), "pattern")
k = {"naive": N.HS_KIND_NAIVE, "adaptive": N.HS_KIND_ADAPTIVE}[kind]
im = {"auto": 0, "lane": 1, "warp": 2, "subbin": 3}[impl]
ts = []
for r in range(reps):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    N.check(L.hs_histogram(buf.data_ptr(), n, k, im, N.i64p(off), N.i64p(cnt), 960, 8, out.data_ptr(), None, 0, s), "hist")
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
ok = np.array_equal(out.cpu().numpy().astype(np.uint64), ref)
ms = sorted(ts[min(3, reps - 1):])[len(ts[min(3, reps - 1):]) // 2]
print(f"{dist} {kind} {impl} n={n} {ms:.4f} ms {n / ms / 1e6:.1f} GB/s {'exact' if ok else 'MISMATCH'}")
