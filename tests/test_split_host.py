"""The weighted CTA split of multi-segment k_lane launches, checked on the host (no
GPU): tests/native/split_check.cu includes the library source with HS_CHECK_SPLIT,
runs random segment layouts through split_grid(), compares the one-pass table with
the binary-search definition at every CTA, and recomputes the per-segment ticket
targets by brute force."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_weighted_split_table(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc not available")
    exe = tmp_path / "split_check"
    r = subprocess.run([nvcc, "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-I", str(ROOT / "include"), str(ROOT / "tests" / "native" / "split_check.cu"),
                        "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "split_check ok" in r.stdout, r.stdout + r.stderr
