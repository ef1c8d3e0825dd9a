"""Normaliser triples and the degenerate-denominator error -- the math contract
of the hot path, mirroring ``ncstream.normalizers`` (normalizers.py:29-126).

SPHERICAL (a1=id, a2=square, b=sqrt; normalizers.py:94-100) and SIGNED_L1
(a1=id, a2=abs, b=id; normalizers.py:111-117) run on the FlashSign kernel (the
epilogue math is a compile-time switch).  SOFTMAX exists so that reference
callers can name it; the GPU streamed path rejects it with ``ConfigError`` (it
is not an exp-free FlashSign triple, and there is no CPU fallback).  The scalar maps are kept so ``NormalizerSpec`` objects behave like
the reference's (e.g. for callers that evaluate ``spec.a2`` themselves).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable

import numpy as np

from ._reftypes import ref_type

PROPERTY_FLAGS = frozenset({"sign_preserving", "shift_invariant", "positive_scale_invariant"})


class DegenerateDenominatorError(ValueError):
    """b(z + eps) was zero or non-finite for some row (normalizers.py:29-35).

    ``z`` is the row's sum of a2(scores); the message carries the reference's
    context string, e.g. ``"row 1"``.
    """

    def __init__(self, z, context: str = ""):
        self.z = z
        text = f"degenerate denominator: b applied to z={z!r} is zero or non-finite"
        super().__init__(text + (f" ({context})" if context else ""))


if ref_type("DegenerateDenominatorError") is not None:
    # the reference's own class (normalizers.py:29-35): `except ncstream...` matches the GPU path
    DegenerateDenominatorError = ref_type("DegenerateDenominatorError")  # noqa: F811


def _identity(u):
    return u


def _square(u):
    return u * u


def _exp(u):
    return np.exp(u)


def _sqrt(z):
    return np.sqrt(z)


@dataclass(frozen=True)
class NormalizerSpec:
    """(a1, a2, b) plus ``denom_epsilon`` and property flags (normalizers.py:54-91)."""

    name: str
    a1: Callable
    a2: Callable
    b: Callable
    denom_epsilon: float = 0.0
    properties: frozenset = field(default_factory=frozenset)
    sfu_evals: int = 0

    def __post_init__(self):
        unknown = set(self.properties) - PROPERTY_FLAGS
        if unknown:
            raise ValueError(f"unknown property flags: {sorted(unknown)}")
        if self.denom_epsilon < 0:
            raise ValueError("denom_epsilon must be nonnegative")

    def with_epsilon(self, eps: float) -> "NormalizerSpec":
        return replace(self, denom_epsilon=eps)

    def denominator(self, z, context: str = ""):
        """b(z + denom_epsilon), raising DegenerateDenominatorError when it is unusable
        (normalizers.py:83-91: a scalar must be finite and nonzero; an array must not
        compare equal to 0 -- the reference's own truth test, so a multi-element array
        raises numpy's ambiguity ValueError exactly as there)."""
        den = self.b(z + self.denom_epsilon) if self.denom_epsilon else self.b(z)
        if isinstance(den, (int, float, np.floating)):
            if not math.isfinite(den) or den == 0:
                raise DegenerateDenominatorError(z, context)
        elif den == 0:
            raise DegenerateDenominatorError(z, context)
        return den


SPHERICAL = NormalizerSpec("spherical", _identity, _square, _sqrt,
                           properties=frozenset({"sign_preserving", "positive_scale_invariant"}))
SOFTMAX = NormalizerSpec("softmax", _exp, _exp, _identity,
                         properties=frozenset({"shift_invariant"}), sfu_evals=2)
SIGNED_L1 = NormalizerSpec("signed_l1", _identity, abs, _identity,
                           properties=frozenset({"sign_preserving", "positive_scale_invariant"}))

BUILTIN_SPECS = {s.name: s for s in (SPHERICAL, SOFTMAX, SIGNED_L1)}


def get_spec(name: str) -> NormalizerSpec:
    if name not in BUILTIN_SPECS:
        raise ValueError(f"unknown normalizer {name!r} (expected one of {sorted(BUILTIN_SPECS)})")
    return BUILTIN_SPECS[name]
