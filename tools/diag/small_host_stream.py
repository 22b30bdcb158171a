"""The reference's default pipeline shape (1 MiB chunks, batch 1) streamed from pinned host
memory: run_pipeline (per-iteration host fold) vs run_device_stream (device fold, host
chunks staged per block on a copy stream). 4 GiB = 4096 iterations, identical results."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

px, n = 1 << 20, 4096
pinned = D.pinned_bytes(px * n)
dev = torch.empty(px * n, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", px * n, 5), dev)
torch.from_numpy(pinned).copy_(dev)
del dev
words = pinned.view(np.uint32)
chunks = [hs.PackedChunk(words[i * (px // 4):(i + 1) * (px // 4)]) for i in range(n)]
cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=px, window_size=128)


def src():
    for c in chunks:
        yield [c]


res = {}
for name, fn in (("run_pipeline", lambda: hs.run_pipeline(src(), cfg, hs.SwitchPolicy())),
                 ("run_device_stream", lambda: hs.run_device_stream(src(), cfg, hs.SwitchPolicy()))):
    fn()
    t0 = time.perf_counter()
    out = fn()
    dt = time.perf_counter() - t0
    res[name] = out
    print(f"{name:18s} {px * n / dt / 1e9:7.2f} GB/s ({dt * 1e6 / n:.1f} us per 1 MiB iteration)", flush=True)
a, b = res["run_pipeline"], res["run_device_stream"]
assert a[0] == b[0] and a[1] == b[1] and a[3] == b[3] and a[2].degeneracy_log == b[2].degeneracy_log
print("identical accumulator, window, kernel and degeneracy logs")
