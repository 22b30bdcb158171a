"""Quick on-GPU check of libhist256: correctness of every impl vs torch.bincount and
CUDA-event throughput. Development tool (not the bench, not a test)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream().cuda_stream
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
buf = torch.empty(n + 64, dtype=torch.uint8, device=dev)
out = torch.empty(256, dtype=torch.int64, device=dev)


def pattern_for(prior):
    off = np.zeros(256, np.int64)
    cnt = np.zeros(256, np.int64)
    N.check(L.hs_binning_pattern(N.u64p(prior), 960, 8, N.i64p(off), N.i64p(cnt)), "pattern")
    return off, cnt


for dist in ("uniform", "normal8", "normal32", "normal64", "const127"):
    if dist == "uniform":
        N.check(L.hs_generate_device(N.HS_GEN_UNIFORM, 7, 0, 0.0, 1.0, 0, buf.data_ptr(), n, stream), "gen")
    elif dist.startswith("normal"):
        N.check(L.hs_generate_device(N.HS_GEN_NORMAL, 7, 0, 128.0, float(dist[6:]), 0, buf.data_ptr(), n, stream), "gen")
    else:
        N.check(L.hs_generate_device(N.HS_GEN_CONSTANT, 7, 127, 0.0, 1.0, 0, buf.data_ptr(), n, stream), "gen")
    ref = torch.bincount(buf[:n], minlength=256).cpu().numpy().astype(np.uint64)
    off, cnt = pattern_for(ref)
    for name, kind, impl in (
        ("naive/auto", N.HS_KIND_NAIVE, N.HS_IMPL_AUTO),
        ("naive/warp", N.HS_KIND_NAIVE, N.HS_IMPL_WARP),
        ("adaptive/auto", N.HS_KIND_ADAPTIVE, N.HS_IMPL_AUTO),
        ("adaptive/subbin", N.HS_KIND_ADAPTIVE, N.HS_IMPL_SUBBIN),
    ):
        # unaligned sub-range exercises head/tail paths
        for lo, hi in ((0, n), (4, n - 12)):
            st = L.hs_histogram(buf.data_ptr() + lo, hi - lo, kind, impl, N.i64p(off), N.i64p(cnt), 960, 8,
                                out.data_ptr(), None, 0, stream)
            N.check(st, name)
            got = out.cpu().numpy().astype(np.uint64)
            want = ref.copy() if (lo, hi) == (0, n) else torch.bincount(buf[lo:hi], minlength=256).cpu().numpy().astype(np.uint64)
            ok = np.array_equal(got, want)
            if not ok:
                print("MISMATCH", dist, name, lo, hi, int(got.sum()), int(want.sum()))
        ts = []
        for r in range(8):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            L.hs_histogram(buf.data_ptr(), n, kind, impl, N.i64p(off), N.i64p(cnt), 960, 8, out.data_ptr(), None, 0, stream)
            b.record()
            b.synchronize()
            if r >= 3:
                ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        print(f"{dist:9s} {name:16s} {ms:8.3f} ms {n / ms / 1e6:8.1f} GB/s  {'exact' if ok else 'MISMATCH'}", flush=True)
