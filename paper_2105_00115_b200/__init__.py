"""paper_2105_00115_b200 -- B200-native qdot (arXiv 2105.00115) hot path.

Drop-in for the reference package's qdot entry point (qdot 0.1.0,
kernel.py:179): same names, arguments, report fields and exceptions; the
work runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/qdot_b200.h (lib/libqdot_b200.so).  No CPU fallback.
"""

from .binning import (Bin, BinPartition, BinSplitting, ExactBinning, RangedBinning, Strategy,
                      parse_strategy, strategy_label)
from .batched import BatchedReport, qdot_batched
from .kernel import QdotReport, ReferenceResult, qdot, reference_dot, select_parameters
from .scoring import (ParameterSet, PrecisionLevel, SplitMode, ToleranceConfig, bin_score, ceil_log2,
                      early_termination, floor_log2, precision_of)

__version__ = "0.1.0"

__all__ = [
    "Bin", "BinPartition", "BinSplitting", "ExactBinning", "RangedBinning", "Strategy",
    "parse_strategy", "strategy_label", "QdotReport", "qdot", "select_parameters", "ReferenceResult", "reference_dot",
    "BatchedReport", "qdot_batched",
    "ParameterSet", "PrecisionLevel", "SplitMode", "ToleranceConfig", "bin_score", "ceil_log2",
    "early_termination", "floor_log2", "precision_of",
]
