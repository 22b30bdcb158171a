"""Functional dry run of bench.py's N>1 path on a one-GPU box: every rank on GPU 0 and
the collectives over gloo instead of NCCL (NCCL refuses two ranks on one device). It
exercises the sharding, the per-rank merged calls, the allreduces, max-over-ranks
timing, the per-rank e2e and the rank-0-only legs; its throughput numbers mean nothing
(the ranks share one GPU and one PCIe link).
run: python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
       --master-port 29511 tools/diag/bench_world2_one_gpu.py --gpus 2 --steps 3 ..."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ["LOCAL_RANK"] = "0"  # every rank on cuda:0

import paper_1011_0235_b200.distributed as dd  # noqa: E402

_init = dd.init_process_group
dd.init_process_group = lambda backend=None, device=None: _init("gloo")

import bench  # noqa: E402

sys.exit(bench.main(sys.argv[1:]))
