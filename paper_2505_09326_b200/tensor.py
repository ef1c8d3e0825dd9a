"""Boundary types of the hot path, mirroring ``ncstream.tensor`` (tensor.py:32-198):
the read-only ``DenseTensor`` carrier, ``ShapeMismatchError``, RNE binary16
quantisation and the ``allclose`` / ``frac_within`` accuracy report."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._reftypes import ref_type

DTYPES = {"float32": np.float32, "float64": np.float64}
FLOAT16_MAX = 65504.0


class ShapeMismatchError(ValueError):
    """Incompatible operand shapes or dtypes (tensor.py:32-33)."""


if ref_type("ShapeMismatchError") is not None:
    ShapeMismatchError = ref_type("ShapeMismatchError")  # noqa: F811  (ncstream's own class)


class DenseTensor:
    """Immutable row-major float32/float64 array (tensor.py:36-98)."""

    __slots__ = ("_array", "_dtype")

    def __init__(self, values, dtype: str | None = None, allow_nonfinite: bool = False):
        if dtype is None:
            src = np.asarray(values)
            dtype = "float32" if src.dtype == np.float32 else "float64"
        if dtype not in DTYPES:
            raise ValueError(f"unsupported dtype {dtype!r} (expected float32 or float64)")
        arr = np.ascontiguousarray(values, dtype=DTYPES[dtype])
        if any(n < 1 for n in arr.shape):
            raise ValueError(f"axis sizes must be >= 1, got shape {arr.shape}")
        if not allow_nonfinite and not np.isfinite(arr).all():
            raise ValueError("non-finite values in tensor (pass allow_nonfinite=True to permit)")
        arr.setflags(write=False)
        self._array = arr
        self._dtype = dtype

    @property
    def shape(self):
        return self._array.shape

    @property
    def rank(self) -> int:
        return self._array.ndim

    @property
    def dtype(self) -> str:
        return self._dtype

    @property
    def array(self) -> np.ndarray:
        return self._array

    @property
    def size(self) -> int:
        return self._array.size

    def tolist(self):
        return self._array.tolist()

    def __repr__(self) -> str:
        return f"DenseTensor(shape={self.shape}, dtype={self._dtype})"


if ref_type("DenseTensor") is not None:
    DenseTensor = ref_type("DenseTensor")  # noqa: F811  (the wrappers return ncstream's carrier)


def quantize_f16_array(arr: np.ndarray) -> np.ndarray:
    """Round to the nearest binary16 value (RNE), kept float32 (tensor.py:132-139)."""
    with np.errstate(over="ignore"):
        return arr.astype(np.float16).astype(np.float32)


@dataclass(frozen=True)
class CloseReport:
    equal: bool
    max_abs_diff: float
    n_total: int
    abs_threshold: float | None = None
    n_within: int | None = None

    def __bool__(self) -> bool:
        return self.equal

    @property
    def frac_within(self) -> float:
        if self.n_within is None:
            raise ValueError("no abs_threshold was requested")
        return self.n_within / self.n_total


def allclose(a, b, rtol: float = 1e-7, atol: float = 0.0, abs_threshold: float | None = None) -> CloseReport:
    """|a-b| <= atol + rtol |b| everywhere, plus the within-threshold count (tensor.py:175-198)."""
    aa = a.array if isinstance(a, DenseTensor) else np.asarray(a)
    bb = b.array if isinstance(b, DenseTensor) else np.asarray(b)
    if aa.shape != bb.shape:
        raise ShapeMismatchError(f"shape mismatch: {aa.shape} vs {bb.shape}")
    with np.errstate(invalid="ignore"):
        diff = np.abs(aa.astype(np.float64) - bb.astype(np.float64))
    finite = np.isfinite(diff)
    equal = bool(finite.all()) and bool((diff <= atol + rtol * np.abs(bb)).all())
    n_within = None if abs_threshold is None else int(np.count_nonzero(finite & (diff <= abs_threshold)))
    return CloseReport(equal, float(diff.max()) if diff.size else 0.0, aa.size, abs_threshold, n_within)
