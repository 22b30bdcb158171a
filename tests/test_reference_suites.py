"""The reference's own unit tests for the host-side modules -- core (packing, value
types), pattern (binning pattern, validation, text dump), policy (degeneracy, switch,
divergence), datagen (splitmix64 generators, streams) and the CLI's configuration
handling -- run unmodified against the drop-in through an import shim. Needs the reference checkout (build container
only: /root/reference is not present on the GPU box, where the kernel suites' parity
is covered by tests/test_gpu_*.py against reference-generated vectors)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[1]


# test_cli.py: the configuration, source-grammar and precedence tests; the ones that
# run a mode need the GPU (every mode warms the kernels first, as the reference does)
CLI_HOST_ONLY = "not tiny_run and not non_timing and not profile and not schedule and not dump"


@pytest.mark.skipif(not REF_TESTS.is_dir(), reason="reference checkout not present")
@pytest.mark.parametrize("suite,select", [("test_core.py", None), ("test_pattern.py", None), ("test_policy.py", None),
                                          ("test_datagen.py", None), ("test_cli.py", CLI_HOST_ONLY)])
def test_reference_suite_passes(suite, select, tmp_path):
    env = dict(os.environ, PYTHONPATH=f"{ROOT / 'tests' / 'refshim'}{os.pathsep}{ROOT}",
               NUMBA_CACHE_DIR=str(tmp_path))
    cmd = [sys.executable, "-m", "pytest", suite, "-q", "-p", "histostream_shim", "-p", "no:cacheprovider"]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
