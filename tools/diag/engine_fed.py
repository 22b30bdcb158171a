"""The block engine fed (host ahead): 1 MiB device chunks, batch 1, 256-iteration blocks,
16 blocks; for an ncu launch list of the engine's kernels."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402

px, n = 1 << 20, 4096
buf = torch.empty(n * px, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", n * px, 3), buf)
batches = [[hs.DeviceChunk(buf[i * px:(i + 1) * px])] for i in range(n)]
cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=px, window_size=128)
for _ in range(2):
    hs.run_device_stream(iter(batches), cfg, hs.SwitchPolicy(), block_bytes=256 << 20, blocks_ahead=None)
torch.cuda.synchronize()
print("ok")
