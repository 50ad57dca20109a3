"""Calibration profile: the *input* type of overhead correction.

Mirrors ``CalibrationProfile`` and its ``xstrace-profile v1`` text format from
``pkg/src/xstrace/calibration.py:28-233`` (the estimators that *build* a
profile -- delta / difference-of-average calibration -- are off the hot path
and out of scope).  ``scaled()`` turns the exact
rational means into integers over one common denominator, which is how the
device carries ``fractions.Fraction`` arithmetic exactly (K6).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from fractions import Fraction
from pathlib import Path
from typing import Sequence, Union

import numpy as np

PROFILE_HEADER = "xstrace-profile v1"

HOOK_ANNOTATION = "annotation"
HOOK_TRANSITION = "transition"
HOOK_API_INTERCEPTION = "api_interception"
HOOK_API_INTERNAL = "api_internal"
HOOK_KINDS = (HOOK_ANNOTATION, HOOK_TRANSITION, HOOK_API_INTERCEPTION, HOOK_API_INTERNAL)


@dataclass(frozen=True)
class CalibrationProfile:
    """Mean book-keeping overhead per hook kind (calibration.py:142-220)."""

    annotation_ns: Fraction
    transition_ns: Fraction
    api_interception_ns: Fraction
    api_internal_ns: dict
    provenance: tuple = ()

    def is_zero(self) -> bool:
        return (
            self.annotation_ns == 0
            and self.transition_ns == 0
            and self.api_interception_ns == 0
            and all(v == 0 for v in self.api_internal_ns.values())
        )

    def to_text(self) -> str:
        lines = [PROFILE_HEADER]
        lines.append(f"annotation = {_format_ns(self.annotation_ns)}")
        lines.append(f"transition = {_format_ns(self.transition_ns)}")
        lines.append(f"api_interception = {_format_ns(self.api_interception_ns)}")
        for api in sorted(self.api_internal_ns):
            lines.append(f"api_internal.{api} = {_format_ns(self.api_internal_ns[api])}")
        for note in self.provenance:
            lines.append(f"# {note}")
        return "\n".join(lines) + "\n"

    @classmethod
    def from_text(cls, text: str) -> "CalibrationProfile":
        lines = text.splitlines()
        if not lines or lines[0].strip() != PROFILE_HEADER:
            raise ValueError(f"not a calibration profile: expected header '{PROFILE_HEADER}'")
        values: dict = {}
        internal: dict = {}
        provenance: list = []
        for line in lines[1:]:
            line = line.strip()
            if not line:
                continue
            if line.startswith("#"):
                provenance.append(line.lstrip("# "))
                continue
            if "=" not in line:
                raise ValueError(f"bad profile line: {line!r}")
            key, _, raw = line.partition("=")
            key = key.strip()
            value = _parse_ns(raw.strip())
            if value < 0:
                raise ValueError(f"negative overhead for {key!r}")
            if key.startswith("api_internal."):
                internal[key[len("api_internal."):]] = value
            elif key in ("annotation", "transition", "api_interception"):
                values[key] = value
            else:
                raise ValueError(f"unknown profile key {key!r}")
        for required in ("annotation", "transition", "api_interception"):
            if required not in values:
                raise ValueError(f"profile missing key {required!r}")
        return cls(values["annotation"], values["transition"], values["api_interception"],
                   internal, tuple(provenance))

    def write(self, path: Union[str, os.PathLike]) -> None:
        Path(path).write_text(self.to_text(), encoding="utf-8")

    @classmethod
    def read(cls, path: Union[str, os.PathLike]) -> "CalibrationProfile":
        return cls.from_text(Path(path).read_text(encoding="utf-8"))

    @classmethod
    def zero(cls, api_names: Sequence[str] = ()) -> "CalibrationProfile":
        return cls(Fraction(0), Fraction(0), Fraction(0), {n: Fraction(0) for n in api_names},
                   ("zero profile",))

    def scaled(self, names: Sequence[str]) -> "ScaledProfile":
        """Integer form for one name table, memoised per (profile, names): a
        repeated analysis of the same trace re-uses the resident device tables."""
        key = (id(self), tuple(names))
        hit = _SCALED_CACHE.get(key)
        if hit is not None and hit[0] is self:
            return hit[1]
        sp = ScaledProfile.build(self, names)
        if len(_SCALED_CACHE) >= 8:
            _SCALED_CACHE.pop(next(iter(_SCALED_CACHE)))
        _SCALED_CACHE[key] = (self, sp)
        return sp


_SCALED_CACHE: dict = {}


def _format_ns(value: Fraction) -> str:
    value = Fraction(value)
    if value.denominator == 1:
        return str(value.numerator)
    return f"{value.numerator}/{value.denominator}"


def _parse_ns(raw: str) -> Fraction:
    try:
        return Fraction(raw)
    except ValueError as exc:
        raise ValueError(f"bad overhead value {raw!r}") from exc


INT64_MAX = 2**63 - 1


@dataclass(frozen=True)
class ScaledProfile:
    """The profile's per-site amounts in the device's exact form.

    The amounts the reference draws per site (correction.py:90-100):
    ``annotation/2`` at ANN_START, ``annotation - annotation/2`` at ANN_END,
    ``transition``, ``api_interception`` and ``api_internal[name]``.  Each is
    split as ``whole + frac / L`` (``0 <= frac < L``, L the common denominator
    of all of them) and L / frac are held in ``words`` 64-bit words, so
    ``quantize_amounts``' floor of exact Fraction running sums
    (_timeline.py:57-67) is reproduced for any denominator: the device keeps
    the fractional running sum modulo L and adds 1 where it wraps.
    """

    words: int
    L: int
    whole: tuple          # 4 ints: ANN_START, ANN_END, TRANSITION, API_INTERCEPT
    frac: tuple           # 4 ints, same order
    internal: np.ndarray      # int64 [n_names] whole parts of api_internal
    internal_frac: tuple      # ints [n_names]
    has_internal: np.ndarray  # uint8 [n_names]

    @classmethod
    def build(cls, profile: CalibrationProfile, names: Sequence[str]) -> "ScaledProfile":
        ann = Fraction(profile.annotation_ns)
        half = ann / 2
        base = [half, ann - half, Fraction(profile.transition_ns), Fraction(profile.api_interception_ns)]
        internal = {k: Fraction(v) for k, v in profile.api_internal_ns.items()}
        den = 1
        for v in base + [internal[n] for n in names if n in internal]:
            den = den * v.denominator // math.gcd(den, v.denominator)
        words = next((w for w in (1, 2, 4, 8) if den.bit_length() <= 64 * w - 1), None)
        if words is None:
            raise ValueError(f"calibration profile common denominator has {den.bit_length()} bits; "
                             "the device supports up to 511")

        def split(v: Fraction):
            w = math.floor(v)
            _check64(w)
            return w, int((v - w) * den)

        whole, frac = zip(*[split(v) for v in base])
        ints = np.zeros(len(names), dtype=np.int64)
        ifrac = [0] * len(names)
        has = np.zeros(len(names), dtype=np.uint8)
        for i, n in enumerate(names):
            if n in internal:
                ints[i], ifrac[i] = split(internal[n])
                has[i] = 1
        ints.flags.writeable = False  # immutable: engines keep a device copy per profile
        has.flags.writeable = False
        return cls(words, den, tuple(whole), tuple(frac), ints, tuple(ifrac), has)

    def words_of(self, v: int) -> list:
        return [(v >> (64 * k)) & 0xFFFFFFFFFFFFFFFF for k in range(self.words)]

    def frac_table(self) -> np.ndarray:
        """uint64 [(4 + n_names) * words]: the fractional numerators, rows in
        xs_profile_t order."""
        rows = list(self.frac) + list(self.internal_frac)
        return np.array([x for r in rows for x in self.words_of(r)], dtype=np.uint64)


def _check64(v: int) -> None:
    if abs(v) > INT64_MAX:
        raise ValueError("calibration amount exceeds int64 nanoseconds")
