"""Import alias used only by the reference-suite runs (tests/test_reference_suites.py,
tests/test_reference_gpu_suites.py): `import histostream` and every
`histostream.<module>` resolve to the drop-in `paper_1011_0235_b200`, also in the
subprocesses the reference's acceptance suite starts (test_acceptance.py:318-345), as
long as tests/refshim is on PYTHONPATH. Test infrastructure; never imported by the
package."""
import importlib
import sys

import paper_1011_0235_b200 as _pkg

for _name in ("bench", "core", "datagen", "kernels", "pattern", "policy", "stream", "cli"):
    sys.modules[f"histostream.{_name}"] = importlib.import_module(f"paper_1011_0235_b200.{_name}")
# the import statement that loaded this module returns sys.modules["histostream"]
sys.modules["histostream"] = _pkg
