"""ncu target: the bench's C5 step shape on a 4 GiB shard -- one merged, chained library
call (four chained 1 GiB k_lane launches) repeated; profile one steady-state launch with
  ncu --set full -k regex:k_lane --launch-skip 6 -c 1 python tools/prof/ncu_c5.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200.distributed import ShardedHistogram  # noqa: E402

n = 4 << 30
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", 64 << 30, 0x10110235 ^ 0xC5), buf)
torch.cuda.synchronize()
sh = ShardedHistogram()
for _ in range(3):
    sh.count(buf, chained=True)
torch.cuda.synchronize()
assert int(sh.result().counts.sum()) == n
print("ok")
