"""Tolerance configuration, precision levels and the scalar scoring helpers.

Host-side mirror of the reference's qdot.scoring interface (scoring.py:15-216):
same names, fields, argument meaning and exceptions, so code written against
the reference runs unchanged.  The per-bin scoring of a qdot call itself runs
on the device (csrc/qdot_kernels.cu, k_score); the scalar helpers here are
the API surface the reference exports (and what the report audit uses).
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


class PrecisionLevel(enum.Enum):
    """Formats a bin may be computed in, plus full perforation (scoring.py:15-41)."""

    PERFORATE = ("perforate", 0)
    HALF = ("half", 10)
    SINGLE = ("single", 23)
    DOUBLE = ("double", 52)

    def __init__(self, label: str, mantissa_bits: int):
        self.label = label
        self.mantissa_bits = mantissa_bits

    @property
    def eps(self) -> float:
        return math.ldexp(1.0, -self.mantissa_bits)

    @property
    def code(self) -> int:
        """Index used by the C ABI (qdot_precision)."""
        return LEVELS_ASC.index(self)

    # Interoperate with the reference's own enum (qdot.scoring.PrecisionLevel):
    # equal by label, same hash as an Enum member of the same name, so
    # report.counts[<reference PrecisionLevel>] and == comparisons work.
    def __eq__(self, other):
        if self is other:
            return True
        lab = getattr(other, "label", None)
        mb = getattr(other, "mantissa_bits", None)
        if lab is None or mb is None:
            return NotImplemented
        return lab == self.label and mb == self.mantissa_bits

    def __hash__(self):
        return hash(self._name_)

    @classmethod
    def from_mu(cls, mu: int) -> "PrecisionLevel":
        for level in cls:
            if level.mantissa_bits == mu:
                return level
        raise ValueError(f"no precision level with {mu} mantissa bits")

    @classmethod
    def from_code(cls, code: int) -> "PrecisionLevel":
        return LEVELS_ASC[code]


LEVELS_ASC = (PrecisionLevel.PERFORATE, PrecisionLevel.HALF, PrecisionLevel.SINGLE, PrecisionLevel.DOUBLE)
_MU_BELOW = {52: 23, 23: 10, 10: 0}
_EPS_MAX = math.ldexp(1.0, 60)


class SplitMode(enum.Enum):
    NONE = "none"
    PER_BIN = "per-bin"

    def __eq__(self, other):   # equal to the reference's SplitMode member of the same value
        if self is other:
            return True
        v = getattr(other, "value", None)
        return NotImplemented if v is None else v == self.value

    def __hash__(self):
        return hash(self._name_)


@dataclass
class ToleranceConfig:
    """Relative tolerance and how it is shared across bins (scoring.py:59-79)."""

    epsilon: float
    split: SplitMode = SplitMode.NONE
    input_mu: int = 52

    def __post_init__(self):
        if not (isinstance(self.epsilon, (int, float)) and math.isfinite(self.epsilon)):
            raise ValueError("epsilon must be finite")
        self.epsilon = float(self.epsilon)
        if not (0.0 < self.epsilon <= _EPS_MAX):
            raise ValueError("epsilon must lie in (0, 2^60]")
        if self.input_mu not in _MU_BELOW:
            raise ValueError("input_mu must be one of 10, 23, 52")


def floor_log2(x: float) -> int:
    """floor(log2 x) for x > 0 (scoring.py:82-86)."""
    if not (x > 0.0 and math.isfinite(x)):
        raise ValueError("floor_log2 needs a positive finite value")
    return math.frexp(x)[1] - 1


def ceil_log2(m: int) -> int:
    """ceil(log2 m) for m >= 1 (scoring.py:89-93)."""
    if m < 1:
        raise ValueError("ceil_log2 needs m >= 1")
    return (m - 1).bit_length()


def bin_score(cardinality: int, upper: int, e_max: int, eps_eff: float) -> int:
    """ceil(log2 M) + u - e_max - floor(log2 eps) + 1 (scoring.py:96-105)."""
    if cardinality < 1:
        raise ValueError("score of an empty bin is -inf and never materialized")
    return ceil_log2(cardinality) + upper - e_max - floor_log2(eps_eff) + 1


def precision_of(score: int, input_mu: int) -> PrecisionLevel:
    """Coarsest level whose mantissa covers the score (scoring.py:108-123)."""
    if input_mu not in _MU_BELOW:
        raise ValueError("input_mu must be one of 10, 23, 52")
    if score < 0:
        return PrecisionLevel.PERFORATE
    for level in LEVELS_ASC[1:]:
        if level.mantissa_bits > input_mu:
            break
        if score < level.mantissa_bits:
            return level
    return PrecisionLevel.from_mu(input_mu)


def early_termination(e_min: int, e_max: int, input_mu: int, epsilon: float) -> bool:
    """e_max - e_min <= -floor(log2 eps) - mu_hat (scoring.py:126-136)."""
    if input_mu not in _MU_BELOW:
        raise ValueError("input_mu must be one of 10, 23, 52")
    return (e_max - e_min) <= (-floor_log2(epsilon) - _MU_BELOW[input_mu])


def relative_bound_term(b, e_max: int) -> float:
    """M * 2^(u - e_max + 1) * eps(precision) (scoring.py:171-173)."""
    return b.cardinality * math.ldexp(b.precision.eps, b.upper - e_max + 1)


def absolute_bound_term(b) -> float:
    """M * 2^(u + 1) * eps(precision) (scoring.py:176-178)."""
    return b.cardinality * math.ldexp(b.precision.eps, b.upper + 1)


@dataclass
class ParameterSet:
    """Scored, precision-assigned bins (scoring.py:139-168).

    ``zero_idx`` is materialised lazily from the device (only when read);
    ``zero_count`` is always available.
    """

    bins: list
    e_min: int
    e_max: int
    strategy: object
    tolerance: ToleranceConfig
    early_terminated: bool
    n: int
    eps_eff: float
    n_bins: int
    rel_bound: float = field(default=0.0)
    zero_count: int = 0
    _indexer: Optional[object] = field(default=None, repr=False)
    _zero_idx: Optional[np.ndarray] = field(default=None, repr=False)
    # bins=None with a _make_bins factory: the Bin objects are built on first
    # access (most callers only read the report's value, counts and bounds)
    _make_bins: Optional[object] = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.bins is None and self._make_bins is not None:
            del self.bins                       # resolved by __getattr__ on first read

    def __getattr__(self, name):
        if name == "bins":
            make = self.__dict__.get("_make_bins")
            value = make(self) if make is not None else []
            self.__dict__["bins"] = value
            return value
        raise AttributeError(name)

    @property
    def zero_idx(self) -> np.ndarray:
        if self._zero_idx is None:
            if self._indexer is None or self.zero_count == 0:
                self._zero_idx = np.empty(0, dtype=np.int64)
            else:
                self._indexer.materialize(self)
        return self._zero_idx

    @property
    def nonzero_count(self) -> int:
        return self.n - self.zero_count

    @property
    def rel_guarantee(self) -> float:
        """N_bins * eps_eff (scoring.py:159-168)."""
        return self.n_bins * self.eps_eff
