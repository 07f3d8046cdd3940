"""Binning strategies and the Bin record.

Host-side mirror of the reference's qdot.binning interface
(binning.py:119-188): the three strategy dataclasses, their text form and the
Bin record.  The partition itself is computed on the device from the
exponent-sum histogram (csrc/qdot_kernels.cu, k_score), so ``Bin.indices``
is materialised lazily -- on first access -- by a device pass
(qdot_b200_bin_ids) instead of an n-sized sort on every call.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Union

import numpy as np

from . import _lib


@dataclass
class ExactBinning:
    name: str = field(default="exact", init=False)


@dataclass
class RangedBinning:
    width: int
    name: str = field(default="ranged", init=False)

    def __post_init__(self):
        if self.width < 1:
            raise ValueError("ranged binning needs width >= 1")


@dataclass
class BinSplitting:
    levels: int
    name: str = field(default="split", init=False)

    def __post_init__(self):
        if self.levels < 0:
            raise ValueError("split levels must be >= 0")


Strategy = Union[ExactBinning, RangedBinning, BinSplitting]


def parse_strategy(text: str) -> Strategy:
    """Parse 'exact', 'ranged:W' or 'split:S' (binning.py:147-157)."""
    head, _, arg = text.partition(":")
    head = head.strip().lower()
    if head == "exact":
        return ExactBinning()
    if head == "ranged":
        return RangedBinning(width=int(arg))
    if head == "split":
        return BinSplitting(levels=int(arg))
    raise ValueError(f"unknown binning strategy {text!r}")


def strategy_label(strategy: Strategy) -> str:
    if isinstance(strategy, ExactBinning):
        return "exact"
    if isinstance(strategy, RangedBinning):
        return f"ranged:{strategy.width}"
    return f"split:{strategy.levels}"


def strategy_code(strategy: Strategy):
    """(qdot_strategy, param) for the C ABI; TypeError like binning.py:284."""
    if strategy is None or isinstance(strategy, ExactBinning):
        return _lib.STRATEGY_EXACT, 0
    if isinstance(strategy, RangedBinning):
        if strategy.width < 1:
            raise ValueError("ranged binning needs width >= 1")
        if strategy.width > (1 << 60):
            raise ValueError("ranged width beyond 2^60 is not supported")
        return _lib.STRATEGY_RANGED, int(strategy.width)
    if isinstance(strategy, BinSplitting):
        if strategy.levels < 0:
            raise ValueError("split levels must be >= 0")
        return _lib.STRATEGY_SPLIT, min(int(strategy.levels), 1 << 20)
    raise TypeError(f"unknown strategy {strategy!r}")


class Bin:
    """One (lower, upper] exponent bin with its score and precision.

    Same fields as the reference Bin (binning.py:168-177).  ``indices`` (the
    ascending member indices) is computed on first access for all bins of the
    report at once; ``value`` is the per-bin dot (what emulate.bin_dot
    returns for this bin).
    """

    __slots__ = ("lower", "upper", "_cardinality", "score", "precision", "value", "flags",
                 "first_key", "last_key", "_indices", "_indexer", "_owner")

    def __init__(self, lower: int, upper: int, cardinality: int, score: Optional[int] = None,
                 precision=None, value: float = 0.0, flags: int = 0, first_key: int = -1,
                 last_key: int = -1, indices: Optional[np.ndarray] = None, indexer=None, owner=None):
        self.lower = lower
        self.upper = upper
        self._cardinality = cardinality
        self.score = score
        self.precision = precision
        self.value = value
        self.flags = flags
        self.first_key = first_key
        self.last_key = last_key
        self._indices = indices
        self._indexer = indexer
        self._owner = owner

    @property
    def cardinality(self) -> int:
        return self._cardinality

    @property
    def indices(self) -> np.ndarray:
        if self._indices is None:
            if self._indexer is None:
                raise RuntimeError("bin indices are not available for this report")
            self._indexer.materialize(self._owner)
        return self._indices

    @indices.setter
    def indices(self, value):
        self._indices = value

    def __repr__(self) -> str:
        p = self.precision.label if self.precision is not None else None
        return (f"Bin(lower={self.lower}, upper={self.upper}, cardinality={self.cardinality}, "
                f"score={self.score}, precision={p})")


@dataclass
class BinPartition:
    bins: List[Bin]
    strategy: Strategy
    e_min: int
    e_max: int
