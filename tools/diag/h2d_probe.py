"""H2D copy rate from pinned host memory by copy size and source offset (why run_pipeline's
256 MiB copies run below the 1 GiB link figure). CUDA events, best of 5."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1011_0235_b200 import device as D  # noqa: E402

GiB = 1 << 30
n = 16 * GiB
pinned = D.pinned_bytes(n)
host = torch.from_numpy(pinned)
host.fill_(1)
dst = torch.empty(GiB, dtype=torch.uint8, device="cuda")
tp = torch.empty(GiB, dtype=torch.uint8, pin_memory=True)
s = torch.cuda.Stream()


def rate(src, size, reps=5):
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record()
            dst[:size].copy_(src[:size], non_blocking=True)
            b.record()
        b.synchronize()
        best = max(best, size / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


for size in (16 << 20, 64 << 20, 256 << 20, GiB):
    row = [f"{size >> 20:5d} MiB"]
    for off in (0, 4 * GiB, 8 * GiB, 15 * GiB):
        row.append(f"off {off // GiB:2d} GiB {rate(host[off:], size):6.2f}")
    row.append(f"torch pinned {rate(tp, size):6.2f} GB/s")
    print(" | ".join(row), flush=True)
# back to back 256 MiB copies over 4 GiB (the pipeline's pattern)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    a.record()
    for k in range(16):
        dst[(k % 4) * (256 << 20):(k % 4 + 1) * (256 << 20)].copy_(host[k * (256 << 20):(k + 1) * (256 << 20)],
                                                                   non_blocking=True)
    b.record()
b.synchronize()
print(f"16 x 256 MiB back to back: {4 * GiB / (a.elapsed_time(b) / 1e3) / 1e9:.2f} GB/s")
