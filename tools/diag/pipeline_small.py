"""run_pipeline at the reference's default PipelineConfig chunk size (1 MiB, batch 1)
from pinned host memory: iterations per second and GB/s, with a per-stage breakdown
(VERDICT r1 item 8)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

px, n = 1 << 20, 1024
pinned = D.pinned_bytes(n * px)
stage = torch.empty(n * px, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", n * px, 1), stage)
torch.from_numpy(pinned).copy_(stage)
words = pinned.view(np.uint32)
chunks = [hs.PackedChunk(words[i * px // 4:(i + 1) * px // 4]) for i in range(n)]
for batch in (1, 4, 16):
    iters = n // batch
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=px, batch_size=batch)
    for rep in range(2):
        t0 = time.perf_counter()
        acc, _, r, _ = hs.run_pipeline((chunks[i * batch:(i + 1) * batch] for i in range(iters)), cfg,
                                       hs.SwitchPolicy())
        dt = time.perf_counter() - t0
    tot = r.stage_totals_ns()
    print(f"batch {batch}: {iters / dt:.0f} it/s, {n * px / dt / 1e9:.2f} GB/s; per-iteration us: "
          + ", ".join(f"{k[:-3]} {v / iters / 1e3:.1f}" for k, v in tot.items()), flush=True)
    assert acc.running.total() == n * px
