"""Copy/compute overlap of the host-streamed pipeline (BASELINE configs[3] shape):
pinned 16 MiB chunks, batches of 16 (256 MiB), run_pipeline on a copy and a compute stream.
Writes profiles/<tag>_stream_timeline.csv and prints the overlap summary."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
CHUNK, BATCH, ITERS = 16 << 20, 16, 16
n = CHUNK * BATCH * ITERS  # 4 GiB, mixed schedule: uniform / normal / constant thirds
pinned = D.pinned_bytes(n)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
third = n // 3 // CHUNK * CHUNK
hs.generate_device(hs.SourceSpec("uniform", third, 1), dev[:third])
hs.generate_device(hs.SourceSpec("normal", third, 2, mean=128.0, sigma=16.0), dev[third:2 * third])
dev[2 * third:].fill_(127)
pinned[:] = dev.cpu().numpy()
words = pinned.view(np.uint32)
chunks = [hs.PackedChunk(words[c * (CHUNK // 4):(c + 1) * (CHUNK // 4)]) for c in range(n // CHUNK)]


def src():
    for i in range(ITERS):
        yield chunks[i * BATCH:(i + 1) * BATCH]


cfg = hs.PipelineConfig(num_iterations=ITERS, chunk_pixels=CHUNK, batch_size=BATCH, window_size=8)
hs.run_pipeline(src(), cfg, hs.SwitchPolicy())  # warm-up
tl = []
acc, _, rep, log = hs.run_pipeline(src(), cfg, hs.SwitchPolicy(), timeline=tl)
assert acc.running.total() == n
out = ROOT / "profiles" / f"{tag}_stream_timeline.csv"
with open(out, "w") as f:
    f.write("iteration,stage,start_us,end_us\n")
    for it, st, a, b in tl:
        f.write(f"{it},{st},{a:.3f},{b:.3f}\n")
h2d = [(a, b) for it, st, a, b in tl if st == "h2d"]
ker = [(a, b) for it, st, a, b in tl if st == "kernel"]
span = max(b for _, _, _, b in tl) - min(a for _, _, a, _ in tl)
busy_h2d = sum(b - a for a, b in h2d)
busy_k = sum(b - a for a, b in ker)
overlap = sum(max(0.0, min(b, d) - max(a, c)) for a, b in ker for c, d in h2d)
print(f"timeline: {len(tl)} events over {span / 1e3:.2f} ms -> {out}")
print(f"h2d busy {busy_h2d / span:.1%} of the span ({n / (busy_h2d / 1e6) / 1e9:.1f} GB/s while copying)")
print(f"kernel busy {busy_k / span:.1%}; kernel time overlapped with H2D: {overlap / max(busy_k, 1e-9):.1%}")
print(f"end-to-end {n / (span / 1e6) / 1e9:.1f} GB/s; kernels {[k.value for k in log[:3]]} ... {[k.value for k in log[-3:]]}")
