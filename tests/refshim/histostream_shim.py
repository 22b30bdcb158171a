"""pytest plugin for running the reference's own test suites against the drop-in:
`import histostream` (and its submodules) resolve to paper_1011_0235_b200.

Used by tests/test_reference_suites.py in the build container, where the reference
checkout exists; it is never imported by the package."""
import importlib
import sys

import paper_1011_0235_b200 as pkg

sys.modules["histostream"] = pkg
for _name in ("bench", "core", "datagen", "kernels", "pattern", "policy", "stream", "cli"):
    sys.modules[f"histostream.{_name}"] = importlib.import_module(f"paper_1011_0235_b200.{_name}")

try:
    import torch

    _gpu = torch.cuda.is_available()
except Exception:  # pragma: no cover
    _gpu = False
if not _gpu:
    # without a GPU the reference conftest's kernel warm-up cannot run; the host-side
    # suites (core, pattern, policy, datagen) do not use the kernels
    sys.modules["histostream.kernels"].warm_kernels = lambda: None
