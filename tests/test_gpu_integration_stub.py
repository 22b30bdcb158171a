"""The ctypes stub INTEGRATION.md tells a reference maintainer to add (histostream/_b200.py)
is executed as written -- only its relative import and library path are pointed at
this checkout -- and its batch_on_b200 must return the oracle's counts."""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N

pytestmark = pytest.mark.gpu
DOC = Path(__file__).resolve().parents[1] / "INTEGRATION.md"


def load_stub():
    text = DOC.read_text()
    block = re.search(r"A ctypes stub to add as `histostream/_b200.py`.*?```python\n(.*?)```", text, re.S).group(1)
    block = block.replace("from .core import Histogram256", "from paper_1011_0235_b200 import Histogram256")
    block = block.replace('"/path/to/paper_1011_0235_b200/_lib/libhist256.so"', repr(str(N.library_path())))
    ns: dict = {}
    exec(compile(block, str(DOC), "exec"), ns)
    return ns


def test_documented_stub_counts_exactly(cuda, oracle):
    stub = load_stub()
    chunks = [hs.PackedChunk(oracle.pack(oracle.generate(k, n, 3, **kw)))
              for k, n, kw in (("uniform", 1 << 20, {}), ("normal", (1 << 18) + 12, {"mean": 9.0, "sigma": 3.0}),
                               ("constant", 4096, {"value": 200}), ("uniform", 0, {}))]
    want = [oracle.histogram(c.pixels()) if c.byte_size else np.zeros(256, np.uint64) for c in chunks]
    got = stub["batch_on_b200"](chunks, False, None)
    assert [g.counts.tolist() for g in got] == [w.tolist() for w in want]
    pattern = hs.compute_binning_pattern(hs.Histogram256(want[1]))
    got = stub["batch_on_b200"](chunks, True, pattern)
    assert [g.counts.tolist() for g in got] == [w.tolist() for w in want]


def test_plain_c_host_counts_exactly(cuda, tmp_path):
    """examples/c_api_demo.c: the C ABI from a C program with no Python or torch in the
    process (cudaMalloc'd buffers, batched NAIVE and ADAPTIVE, host control plane,
    blocking host entry), each result checked against a host count inside the demo."""
    import subprocess
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_native_abi import _build_c_demo

    exe = _build_c_demo(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "c_api_demo ok" in r.stdout, r.stdout + r.stderr
