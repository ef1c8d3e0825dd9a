"""Reference type identity at the drop-in boundary.

When the reference package ``ncstream`` is importable, the exception classes the
drop-in API raises and the ``DenseTensor`` carrier it returns ARE ncstream's own:

    ncstream.normalizers.DegenerateDenominatorError   normalizers.py:29-35
    ncstream.tensor.ShapeMismatchError                tensor.py:32-33
    ncstream.attention.ConfigError                    attention.py:36-37
    ncstream.tensor.DenseTensor                       tensor.py:36-98

so a caller's ``except ncstream...`` clause and the reference's own ``pytest.raises``
(test_attention.py:73-80, 276) match errors raised by the GPU path after the
INTEGRATION.md section 1 switch.  Without ncstream the package defines same-named
``ValueError`` subclasses (``_errors.py``, ``normalizers.py``, ``tensor.py``).

Only types are borrowed; nothing on the compute path calls into ncstream.
``FLASHSIGN_NCSTREAM=0`` forces the local classes.
"""

from __future__ import annotations

import os

REF = None
if os.environ.get("FLASHSIGN_NCSTREAM", "1") != "0":
    try:
        import ncstream.attention as _att
        import ncstream.normalizers as _norm
        import ncstream.tensor as _ten

        REF = {
            "ConfigError": _att.ConfigError,
            "DegenerateDenominatorError": _norm.DegenerateDenominatorError,
            "ShapeMismatchError": _ten.ShapeMismatchError,
            "DenseTensor": _ten.DenseTensor,
        }
    except Exception:  # not installed (or broken): local classes
        REF = None


def ref_type(name: str):
    """ncstream's class ``name`` when the reference is importable, else None."""
    return None if REF is None else REF[name]
