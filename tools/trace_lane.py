"""Per-CTA timeline of k_lane from an instrumented build (tools/ab_build.sh with
-DHS_TRACE, loaded through HS_LIBHIST256): stamps at CTA start, after zeroing, after
each piece's streaming loop and after each flush, and at exit. Runs 10 back-to-back
launches and reports the last one.
usage: HS_LIBHIST256=tools/ablib/trace.so python tools/trace_lane.py NSEG"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
raw = ctypes.CDLL(os.environ["HS_LIBHIST256"])
nseg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = (int(sys.argv[2]) if len(sys.argv) > 2 else 1024) << 20
st = torch.cuda.current_stream()
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
hs.generate_device(hs.SourceSpec("normal", n, 5, mean=128.0, sigma=32.0), buf)
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
b0 = np.arange(nseg, dtype=np.uint64) * (n // nseg)
b1 = b0 + n // nseg


def call():
    N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, N.HS_KIND_NAIVE, N.HS_IMPL_LANE,
                                   None, None, 0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream), "h")


for _ in range(3):
    call()
torch.cuda.synchronize()
raw.hs_trace_clear()
torch.cuda._sleep(20_000_000)
for _ in range(reps):
    call()
torch.cuda.synchronize()
t = np.zeros((1024, 16), np.uint64)
assert raw.hs_trace_read(t.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(t.nbytes)) == 0
g = int((t[:, 0] > 0).sum())  # CTAs of the last launch that stamped
t = t[:g].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print(f"nseg={nseg} grid={g} launch span {rel[:, 15].max():.1f} us (first CTA start -> last CTA exit)")
print(f"  CTA start  min {rel[:, 0].min():.1f} max {rel[:, 0].max():.1f} us")
print(f"  zeroing    mean {np.mean(rel[:, 1] - rel[:, 0]):.2f} us")
np_ = np.array([sum(1 for i in range(7) if t[c, 3 + 2 * i] > 0) for c in range(g)])
print(f"  pieces per CTA: {dict(zip(*np.unique(np_, return_counts=True)))}")
for i in range(3):
    m = t[:, 3 + 2 * i] > 0
    if not m.any():
        break
    start = rel[m, 1] if i == 0 else rel[m, 1 + 2 * i]
    loop = rel[m, 2 + 2 * i] - start
    fl = rel[m, 3 + 2 * i] - rel[m, 2 + 2 * i]
    print(f"  piece {i}: n={m.sum():3d} loop mean {loop.mean():7.2f} us  flush(t0 view) mean {fl.mean():6.2f} max {fl.max():6.2f} us")
last = np.array([max(rel[c, 3 + 2 * i] for i in range(7) if t[c, 3 + 2 * i] > 0) for c in range(g)])
print(f"  tickets    mean {np.mean(rel[:, 15] - last):.2f} us")
print(f"  CTA exit   min {rel[:, 15].min():.1f} max {rel[:, 15].max():.1f} us")
loop0 = rel[:, 2] - rel[:, 1]
print(f"  loop (thread 0) per CTA: min {loop0.min():.2f} median {np.median(loop0):.2f} max {loop0.max():.2f} us")
print(f"  start->loop begin (zero + piece list): median {np.median(rel[:, 1] - rel[:, 0]):.2f} us")
print(f"  last piece end -> exit (flush + tickets): median {np.median(rel[:, 15] - rel[:, 2]):.2f} "
      f"max {np.max(rel[:, 15] - rel[:, 2]):.2f} us")
ex = rel[:, 15]
print(f"  CTA exit spread: p10 {np.percentile(ex, 10):.1f} p50 {np.percentile(ex, 50):.1f} p90 {np.percentile(ex, 90):.1f} max {ex.max():.1f} us")
sm = np.array([0] * g)
hist = np.histogram(rel[:, 0], bins=8)
print("  CTA start histogram (us edges, counts):", [round(e, 1) for e in hist[1]], hist[0].tolist())
if (t[:, 14] > 0).any():  # instrumented with a stamp after the first-launch wait (waiting calls)
    w = rel[:, 14]
    print(f"  wait return: min {w.min():.2f} max {w.max():.2f} us; wait return -> last exit {rel[:, 15].max() - w.min():.2f} us")
    print(f"  wait return -> loop begin median {np.median(rel[:, 1] - w):.2f} us; loop median {np.median(rel[:, 2] - rel[:, 1]):.2f} us")
    per = None
