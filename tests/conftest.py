"""Shared fixtures. `-m gpu` tests need a CUDA device and the built libhist256.so;
everything else runs on the CPU (oracle vs golden vectors, host logic, ABI exports,
gloo multi-process)."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_DIR = ROOT / "tests" / "golden"

# the vendored reference suites run only through their harnesses (subprocess + shim)
collect_ignore = ["refsuites", "refshim"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhist256.so")
    config.addinivalue_line("markers", "slow: long-running (large inputs)")


class Golden:
    """Reference-generated vectors (tests/golden/make_golden.py)."""

    def __init__(self):
        self.meta = json.loads((GOLDEN_DIR / "reference_vectors.json").read_text())
        with np.load(GOLDEN_DIR / "reference_vectors.npz") as z:
            self.arr = {k: z[k] for k in z.files}

    def __getitem__(self, key):
        return self.arr[key]


@pytest.fixture(scope="session")
def golden():
    return Golden()


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()
    return o


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1011_0235_b200 import _native

    _native.lib()
    return torch


WS_HEAD_BYTES = 384  # include/hist256.h HS_WS_HEAD_BYTES: calls u64 @0, drained u32[4] @128, finalized @256
WS_DRAINED = slice(128, 144)
WS_FINALIZED = slice(256, 272)


def ws_clean(ws) -> bool:
    """A ticketed-histogram workspace between calls: every call slot (tickets and
    accumulator rows) zero again and no finalization pending; the header's call
    counter and per-slot drain counts advance and are not checked here."""
    head = ws[:WS_HEAD_BYTES].cpu().numpy()
    finalized = head[WS_FINALIZED]
    return not ws[WS_HEAD_BYTES:].any().item() and not finalized.any()
