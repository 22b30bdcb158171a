"""Launch-split A/B: 16 GiB counted as 16 calls of 1 GiB or one 16 GiB call, with 1 or 64
segments, each measured after a 1 s power settle (the board's power cap otherwise
confounds long runs). Library from HS_LIBHIST256 (profiles/r1_launch_split.txt)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N, device as D
L = N.lib()
buf = torch.empty(16 << 30, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", buf.numel(), 3), buf)
ws = D.default_staging().workspace()
out = torch.empty((64, 256), dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def run(total_gib, per_call_gib, nseg):
    n_call = total_gib // per_call_gib
    size = per_call_gib << 30
    edges = np.linspace(0, size // 4, nseg + 1).astype(np.uint64) * np.uint64(4)
    b0, b1 = edges[:-1].copy(), edges[1:].copy()
    def once():
        for k in range(n_call):
            N.check(L.hs_histogram_batched(buf.data_ptr() + k * size, N.u64p(b0), N.u64p(b1), nseg, N.HS_KIND_NAIVE, N.HS_IMPL_LANE,
                                           None, None, 0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(), st), "h")
    torch.cuda.synchronize(); time.sleep(1.0)  # let the power controller settle
    once(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        torch.cuda._sleep(2_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); once(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"{os.path.basename(os.environ.get('HS_LIBHIST256', 'in-tree')):12s} {total_gib:3d} GiB as {n_call:3d} calls x {per_call_gib:2d} GiB, nseg {nseg:2d}: {ms:8.3f} ms  {(total_gib << 30) / ms / 1e6:7.1f} GB/s", flush=True)
for nseg in (1, 64):
    run(16, 1, nseg); run(16, 16, nseg)
