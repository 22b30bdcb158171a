"""The reference's own unit tests for the host-side modules -- core (packing, value
types), pattern (binning pattern, validation, text dump), policy (degeneracy, switch,
divergence), datagen (splitmix64 generators, streams) and the CLI's configuration
handling -- run unmodified against the drop-in through an import shim.

The suites are vendored byte-for-byte in tests/refsuites/ (SHA256SUMS there), so they
run anywhere; the kernel, stream and acceptance suites need the GPU and run in
tests/test_reference_gpu_suites.py."""
import hashlib
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITES = ROOT / "tests" / "refsuites"
REF_TESTS = Path("/root/reference/pkg/tests")

# test_cli.py: the configuration, source-grammar and precedence tests; the ones that
# run a mode need the GPU (every mode warms the kernels first, as the reference does)
CLI_HOST_ONLY = "not tiny_run and not non_timing and not profile and not schedule and not dump"


def run_suite(suite: str, select: str | None, tmp_path, timeout: int = 900, extra=()):
    """Run one vendored reference suite in a subprocess with `histostream` aliased to
    the drop-in. Returns the CompletedProcess."""
    env = dict(os.environ, PYTHONPATH=f"{ROOT / 'tests' / 'refshim'}{os.pathsep}{ROOT}",
               NUMBA_CACHE_DIR=str(tmp_path))
    cmd = [sys.executable, "-m", "pytest", suite, "-q", "-rxXs", "-p", "histostream_shim", "-p", "no:cacheprovider",
           "--rootdir", str(SUITES), "-c", str(SUITES / "pytest.ini"), *extra]
    if select:
        cmd += ["-k", select]
    return subprocess.run(cmd, cwd=SUITES, env=env, capture_output=True, text=True, timeout=timeout)


def test_vendored_suites_unmodified():
    """Every vendored file matches SHA256SUMS, and -- where the reference checkout
    exists -- the reference's own bytes."""
    sums = {}
    for line in (SUITES / "SHA256SUMS").read_text().splitlines():
        digest, name = line.split()
        sums[name] = digest
        assert hashlib.sha256((SUITES / name).read_bytes()).hexdigest() == digest, name
    assert {"test_kernels.py", "test_stream.py", "test_acceptance.py", "conftest.py"} <= set(sums)
    if REF_TESTS.is_dir():
        for name, digest in sums.items():
            assert hashlib.sha256((REF_TESTS / name).read_bytes()).hexdigest() == digest, f"{name} drifted"


@pytest.mark.parametrize("suite,select", [("test_core.py", None), ("test_pattern.py", None), ("test_policy.py", None),
                                          ("test_datagen.py", None), ("test_cli.py", CLI_HOST_ONLY)])
def test_reference_suite_passes(suite, select, tmp_path):
    r = run_suite(suite, select, tmp_path)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
