"""bench.py's host-side pieces on the CPU: the reference arm's sample bytes are the C5
stream's bytes (the same splitmix64 positions the device generator writes), both arms
name the same workload, and the reference arm prints one contract line."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402


def test_uniform_stream_at_offset_matches_generator():
    for first in (0, 8, 4096, 1 << 20):
        n = 1 << 16
        buf = np.empty(n, np.uint8)
        bench._fill_uniform_at(O.lib(), buf, bench.C5_SEED, first)
        want = O.generate("uniform", first + n, bench.C5_SEED)[first:]
        assert np.array_equal(buf, want), first


def test_config_names_c5_at_every_world():
    for world in (1, 2, 4, 8):
        c = bench.config_dict(world)
        assert c["total_bytes"] == 64 << 30 and c["bytes_per_gpu"] * world == 64 << 30
        assert "C5" in c["workload"]


def test_reference_arm_line(tmp_path):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=tmp_path)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["config"] == bench.config_dict(1)
    assert line["cpu_baseline"]["cores"] >= 1 and line["e2e"]["h2d_bytes_per_step"] == 0
