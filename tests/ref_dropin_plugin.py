"""pytest plugin: run the REFERENCE's own test files against this package's GPU path.

    python -m pytest -p ref_dropin_plugin baseline/_ref/ncstream_tests/test_attention.py

Loaded before collection (``-p``), so the reference tests' ``from ncstream.attention import ...``
binds the FlashSign functions installed by ``attention.patch_ncstream()`` (INTEGRATION.md
section 1).  Test infrastructure only."""

import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (_ROOT, os.path.join(_ROOT, "baseline", "_ref")):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2505_09326_b200 import attention as _fs_attention  # noqa: E402

PATCHED = _fs_attention.patch_ncstream()
