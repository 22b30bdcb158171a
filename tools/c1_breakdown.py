"""Where the per-image time of the synchronous API goes (1024x1024 image, BASELINE
configs[0]): the public call, the same native call with prepared arguments, and each
Python piece of the device path on its own (mean of 2000 calls, wall clock)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N, device as D  # noqa: E402

n = 1 << 20
chunk = hs.generate(hs.SourceSpec("uniform", n, 0))
cfg = hs.WorkerGroupConfig()
dc = hs.DeviceChunk(torch.from_numpy(chunk.words.view(np.uint8).copy()).cuda())
pin = D.pinned_words(chunk.words.size)
pin[:] = chunk.words
pc = hs.PackedChunk(pin)
L = N.lib()
st = D.default_staging()
s = torch.cuda.current_stream()
for _ in range(50):
    hs.naive_histogram(dc, cfg), hs.naive_histogram(chunk, cfg), hs.naive_histogram(pc, cfg)
torch.cuda.synchronize()


def T(name, f, reps=2000):
    for _ in range(20):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    print(f"{name:44s} {(time.perf_counter() - t0) / reps * 1e6:8.2f} us", flush=True)


T("naive_histogram(DeviceChunk)", lambda: hs.naive_histogram(dc, cfg))
T("naive_histogram(pinned PackedChunk)", lambda: hs.naive_histogram(pc, cfg))
T("naive_histogram(pageable PackedChunk)", lambda: hs.naive_histogram(chunk, cfg), 500)
T("D.histograms([dc])", lambda: D.histograms([dc], N.HS_KIND_NAIVE))
b0, b1 = np.zeros(1, np.uint64), np.full(1, n, np.uint64)
out_dev, h_out, ws = st.device_out(1), st.host_out(1), st.workspace()
hp = ctypes.cast(h_out.data_ptr(), N._U64P)
args = (dc.data.data_ptr(), N.u64p(b0), N.u64p(b1), 1, 0, 0, None, None, 0, 0, out_dev.data_ptr(), hp,
        ws.data_ptr(), ws.numel(), s.cuda_stream)
T("hs_histogram_sync, prepared args", lambda: L.hs_histogram_sync(*args))
args0 = args[:-1] + (None,)
T("hs_histogram_sync, legacy stream", lambda: L.hs_histogram_sync(*args0))
bargs = (dc.data.data_ptr(), N.u64p(b0), N.u64p(b1), 1, 0, 0, None, None, 0, 0, out_dev.data_ptr(),
         ws.data_ptr(), ws.numel(), s.cuda_stream)
T("hs_histogram_batched only (async)", lambda: L.hs_histogram_batched(*bargs))


def launch_sync():
    L.hs_histogram_batched(*bargs)
    s.synchronize()


T("hs_histogram_batched + stream sync", launch_sync)
T("torch.cuda.synchronize() idle", torch.cuda.synchronize)
T("require_cuda", D.require_cuda)
T("torch.cuda.current_stream", torch.cuda.current_stream)
T("default_staging", D.default_staging)
T("stage([dc])", lambda: D.stage([dc], st, s))
T("N.u64p x2", lambda: (N.u64p(b0), N.u64p(b1)))
T("ctypes.cast pinned ptr", lambda: ctypes.cast(h_out.data_ptr(), N._U64P))
T("result copy + Histogram256", lambda: hs.Histogram256(h_out.numpy().reshape(1, 256).view(np.uint64).copy()[0]))
ptrs = (ctypes.c_void_p * 1)(chunk.words.ctypes.data)
sizes = np.array([n], np.uint64)
dev = st.device_bytes(n)
hargs = (ptrs, N.u64p(sizes), 1, 0, 0, None, None, 0, 0, dev.data_ptr(), dev.numel(), out_dev.data_ptr(), hp,
         ws.data_ptr(), ws.numel(), s.cuda_stream)
T("hs_histogram_host pageable, prepared", lambda: L.hs_histogram_host(*hargs), 500)
pptrs = (ctypes.c_void_p * 1)(pin.ctypes.data)
hargs_p = (pptrs,) + hargs[1:]
T("hs_histogram_host pinned, prepared", lambda: L.hs_histogram_host(*hargs_p))
# throughput form: 100 single-image launches replayed from a CUDA graph (PDL overlaps them)
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(s)
with torch.cuda.stream(cs):
    L.hs_histogram_batched(*bargs[:-1], cs.cuda_stream)
s.wait_stream(cs)
with torch.cuda.graph(g):
    gs = torch.cuda.current_stream().cuda_stream
    for _ in range(100):
        N.check(L.hs_histogram_batched(*bargs[:-1], gs), "capture")
g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    g.replay()
b.record()
b.synchronize()
print(f"{'graph: single-image launch (throughput)':44s} {a.elapsed_time(b) / 1000 * 1e3:8.2f} us", flush=True)
got = out_dev[0].cpu().numpy().view(np.uint64)
assert np.array_equal(got, np.bincount(chunk.pixels(), minlength=256)), "counts"
assert np.array_equal(hs.naive_histogram(dc, cfg).counts, got) and np.array_equal(hs.naive_histogram(pc, cfg).counts, got)
print("counts ok")
