"""Per-image latency of the synchronous API on a 1024x1024 image (BASELINE configs[0]):
pageable host chunk, pinned host chunk, device chunk, and the stage/launch/readback
pieces of the device path."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import device as D, _native as N
chunk = hs.generate(hs.SourceSpec("uniform", 1 << 20, 0))
cfg = hs.WorkerGroupConfig()
for _ in range(20): hs.naive_histogram(chunk, cfg)
torch.cuda.synchronize()
def T(f, n=200):
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
st = D.default_staging(); s = torch.cuda.current_stream()
print("naive_histogram API      %.1f us" % T(lambda: hs.naive_histogram(chunk, cfg)))
print("stage only (pageable H2D) %.1f us" % T(lambda: D.stage([chunk], st, s)))
staged = D.stage([chunk], st, s)
print("launch only              %.1f us" % T(lambda: D.launch(staged, N.HS_KIND_NAIVE, None, s, staging=st)))
out = D.launch(staged, N.HS_KIND_NAIVE, None, s, staging=st)
print("readback only            %.1f us" % T(lambda: D.readback(out, st, s)))
print("Histogram256 construct   %.1f us" % T(lambda: hs.Histogram256(np.zeros(256, np.uint64))))
pin = D.pinned_words(chunk.words.size); pin[:] = chunk.words
pc = hs.PackedChunk(pin)
print("naive_histogram pinned   %.1f us" % T(lambda: hs.naive_histogram(pc, cfg)))
dev = torch.from_numpy(chunk.words.view(np.uint8).copy()).cuda()
dc = hs.DeviceChunk(dev)
print("naive_histogram device   %.1f us" % T(lambda: hs.naive_histogram(dc, cfg)))
