"""Batched qdot: many independent dot products (rows of X and Y) in one launch.

    qdot_batched(X, Y, cfg, strategy=None) -> BatchedReport

Row r of the result equals qdot(X[r], Y[r], cfg, strategy) (kernel.py:179-240)
-- same value, precision counts, bin count and exponent range.  The reference
has no batched entry point (SURVEY.md §7.1 adds it; BASELINE.json configs[3]
is 65,536 dots of length 4,096); its oracle is a per-row loop of qdot.

One warp per row streams the row once and finishes the whole pipeline in
registers and shared memory (csrc/qdot_batched.cuh); ranged and split
strategies too (a second pass over the row for the HALF / SINGLE members whose
products depend on the partition).  Rows the fused kernel flags
QDOT_BATCH_GENERAL (exponents spread over more than 64 values, DOUBLE
overflow, rows longer than 2^16, ...) are recomputed here through the
single-vector device pipeline, so results never depend on that split; so are
rows with a HALF bin whose fp32 sequential sum is order-sensitive (that
pipeline replays it in index order, qdot_b200_half_ordered).

bins=True also returns every row's bin table (QdotReport.params.bins per row:
lower, upper, cardinality, score, precision, value), from the kernel
(qdot_b200_batched_bins) or, for recomputed rows, from the single-vector run.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .binning import ExactBinning, Strategy
from .device import config_struct, require_cuda, stream_handle
from .kernel import _raise_status, run_device
from .scoring import LEVELS_ASC, PrecisionLevel, ToleranceConfig

GENERAL, NONFINITE, OVERFLOW, EPS, EARLY, HALF_ORDER = 8, 1, 2, 4, 16, 32
MAX_BINS = 64            # QDOT_BATCH_MAX_BINS: row stride of the device bin tables

# qdot_bin (include/qdot_b200.h) as a numpy record
BIN_DTYPE = np.dtype([("lower", "<i8"), ("upper", "<i8"), ("cardinality", "<i8"), ("score", "<i8"),
                      ("precision", "<i4"), ("first_key", "<i4"), ("last_key", "<i4"), ("flags", "<i4"),
                      ("value", "<f8")])
assert BIN_DTYPE.itemsize == ctypes.sizeof(_lib.QdotBin)


@dataclass
class BatchedReport:
    values: np.ndarray          # float64[rows]
    counts: np.ndarray          # int64[rows, 4]: PERFORATE (incl. zero products), HALF, SINGLE, DOUBLE
    n_bins: np.ndarray          # int32[rows]
    e_min: np.ndarray           # int32[rows]
    e_max: np.ndarray           # int32[rows]
    early_terminated: np.ndarray  # bool[rows]
    half_order_sensitive: np.ndarray  # bool[rows]
    general_rows: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    bin_table: np.ndarray = None          # BIN_DTYPE[rows, MAX_BINS] (bins=True)
    _rerun_bins: dict = field(default_factory=dict, repr=False)

    def count(self, level: PrecisionLevel) -> np.ndarray:
        return self.counts[:, LEVELS_ASC.index(level)]

    def row_bins(self, r: int) -> np.ndarray:
        """Bin table of row r (BIN_DTYPE records, ascending upper); needs bins=True."""
        if self.bin_table is None:
            raise ValueError("qdot_batched(..., bins=True) keeps the bin tables")
        if r in self._rerun_bins:
            return self._rerun_bins[r]
        return self.bin_table[r, :int(self.n_bins[r])]


def _as_matrix(A, device):
    import torch
    if isinstance(A, torch.Tensor):
        t = A
        if t.dim() != 2:
            raise ValueError("batched inputs must be 2-D (rows, length)")
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        if t.device != device:
            t = t.to(device)
        if t.stride(1) != 1:
            t = t.contiguous()
        return t
    a = np.asarray(A, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("batched inputs must be 2-D (rows, length)")
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def qdot_batched(X, Y, cfg: ToleranceConfig, strategy: Strategy = None, bins: bool = False) -> BatchedReport:
    """Row-wise qdot of two (rows, length) fp64 matrices (same result as a loop of qdot)."""
    torch = require_cuda()
    if strategy is None:
        strategy = ExactBinning()
    norm = X is Y
    device = torch.device("cuda", torch.cuda.current_device())
    Xd = _as_matrix(X, device)
    Yd = Xd if norm else _as_matrix(Y, device)
    if Xd.shape != Yd.shape:
        raise ValueError(f"shape mismatch: {tuple(Xd.shape)} vs {tuple(Yd.shape)}")
    rows, length = int(Xd.shape[0]), int(Xd.shape[1])

    def row_stride(t):   # size-1 leading dims may carry any stride
        return length if rows <= 1 else int(t.stride(0))

    ld = row_stride(Xd)
    if ld < length or (not norm and row_stride(Yd) != ld):
        Xd = Xd.contiguous()
        Yd = Xd if norm else Yd.contiguous()
        ld = length
    lib = _lib.load()
    c = config_struct(cfg, strategy)
    s = stream_handle(device)
    values = torch.empty(max(rows, 1), dtype=torch.float64, device=device)
    counts = torch.empty((max(rows, 1), 4), dtype=torch.int64, device=device)
    info = torch.empty((max(rows, 1), 4), dtype=torch.int32, device=device)
    if bins:
        btab = torch.empty(max(rows, 1) * MAX_BINS * BIN_DTYPE.itemsize, dtype=torch.uint8, device=device)
        _lib.check(lib.qdot_b200_batched_bins(Xd.data_ptr(), Yd.data_ptr(), rows, length, ld, int(norm),
                                              ctypes.byref(c), values.data_ptr(), counts.data_ptr(),
                                              info.data_ptr(), btab.data_ptr(), s), lib)
    else:
        _lib.check(lib.qdot_b200_batched(Xd.data_ptr(), Yd.data_ptr(), rows, length, ld, int(norm),
                                         ctypes.byref(c), values.data_ptr(), counts.data_ptr(), info.data_ptr(),
                                         s), lib)
    v = values[:rows].cpu().numpy()
    cn = counts[:rows].cpu().numpy()
    inf = info[:rows].cpu().numpy()
    st = inf[:, 3]
    if np.any(st & NONFINITE):
        raise ValueError("inputs must be finite")                       # floatbits.py:70-71
    # rows with a HALF bin the reference sums order-sensitively are redone by
    # the single-vector pipeline, which replays that fp32 sum in index order
    general = np.flatnonzero(st & (GENERAL | HALF_ORDER))
    rep = BatchedReport(values=v.copy(), counts=cn.copy(), n_bins=inf[:, 0].copy(), e_min=inf[:, 1].copy(),
                        e_max=inf[:, 2].copy(), early_terminated=(st & EARLY) != 0,
                        half_order_sensitive=(st & HALF_ORDER) != 0, general_rows=general)
    if bins:
        rep.bin_table = btab[:rows * MAX_BINS * BIN_DTYPE.itemsize].cpu().numpy().view(BIN_DTYPE).reshape(
            rows, MAX_BINS)
    if np.any((st & OVERFLOW) & ~(st & GENERAL)):
        raise OverflowError("math range error")
    if np.any((st & EPS) & ~(st & GENERAL)):
        raise ValueError("floor_log2 needs a positive finite value")
    for r in general.tolist():
        xr = Xd[r]
        yr = xr if norm else Yd[r]
        res, rb, _ = run_device(xr, yr, length, norm, cfg, strategy, timing=False)
        _raise_status(res)
        rep.values[r] = res.value
        rep.counts[r] = [res.counts[i] for i in range(4)]
        rep.n_bins[r] = res.n_bins
        rep.e_min[r] = res.e_min
        rep.e_max[r] = res.e_max
        rep.early_terminated[r] = bool(res.early_terminated)
        rep.half_order_sensitive[r] = bool(res.half_order_sensitive)
        if bins:
            nb = int(res.n_bins)
            rep._rerun_bins[r] = np.frombuffer(ctypes.string_at(ctypes.addressof(rb), nb * BIN_DTYPE.itemsize),
                                               dtype=BIN_DTYPE).copy() if nb else np.empty(0, dtype=BIN_DTYPE)
    return rep
