"""How fast can pageable host chunks reach the device? Host memcpy into page-locked memory
with 1-8 threads (numpy copyto releases the GIL), torch's own pageable H2D copy, and
run_pipeline over 4 GiB of pageable 16 MiB chunks (batches of 16) vs the same bytes pinned."""
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

MiB = 1 << 20
n = 256 * MiB
src = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
dst = D.pinned_bytes(n)


def par_copy(k):
    step = n // k
    ths = [threading.Thread(target=np.copyto, args=(dst[i * step:(i + 1) * step], src[i * step:(i + 1) * step]))
           for i in range(k)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()


for k in (1, 2, 4, 8):
    best = 0.0
    for _ in range(5):
        t0 = time.perf_counter()
        par_copy(k)
        best = max(best, n / (time.perf_counter() - t0) / 1e9)
    print(f"host copy pageable -> pinned, {k} threads: {best:.1f} GB/s", flush=True)

d = torch.empty(n, dtype=torch.uint8, device="cuda")
ts = torch.from_numpy(src)
best = 0.0
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(ts)
    torch.cuda.synchronize()
    best = max(best, n / (time.perf_counter() - t0) / 1e9)
print(f"torch H2D from pageable (driver staging): {best:.1f} GB/s", flush=True)

CH, B, total = 16 * MiB, 16, 4 << 30
page = np.random.default_rng(1).integers(0, 256, total, dtype=np.uint8)
pin = D.pinned_bytes(total)
pin[:] = page
for name, buf in (("pageable", page), ("pinned", pin)):
    words = buf.view(np.uint32)
    chunks = [hs.PackedChunk(words[i * (CH // 4):(i + 1) * (CH // 4)]) for i in range(total // CH)]
    iters = len(chunks) // B
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=CH, batch_size=B, window_size=8)

    def srcf():
        for i in range(iters):
            yield chunks[i * B:(i + 1) * B]

    hs.run_pipeline(srcf(), cfg, hs.SwitchPolicy())
    for _ in range(2):
        t0 = time.perf_counter()
        acc = hs.run_pipeline(srcf(), cfg, hs.SwitchPolicy())[0]
        print(f"run_pipeline {name} 16 MiB x 16: {total / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
    assert acc.running.total() == total

# the synchronous API on one large pageable chunk (routed through the copy pool when >= 2 MiB)
for size in (1 << 20, 4 << 20, 64 << 20, 256 << 20):
    ch = hs.PackedChunk(page[:size].view(np.uint32))
    hs.naive_histogram(ch, hs.WorkerGroupConfig())
    best = 0.0
    for _ in range(5):
        t0 = time.perf_counter()
        hs.naive_histogram(ch, hs.WorkerGroupConfig())
        best = max(best, size / (time.perf_counter() - t0) / 1e9)
    print(f"naive_histogram pageable {size >> 20} MiB: {best:.1f} GB/s ({size / best / 1e3:.0f} us)", flush=True)
