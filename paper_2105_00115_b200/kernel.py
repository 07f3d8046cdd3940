"""qdot entry point: the drop-in replacement for the reference's kernel.qdot.

    qdot(x, y, cfg, strategy=None, reference=None) -> QdotReport   (kernel.py:179-240)
    select_parameters(x, y, cfg, strategy=None) -> ParameterSet    (kernel.py:34-72)

Same signature, argument meaning, report fields and exception types as the
reference.  Underneath, one call is (csrc/, include/qdot_b200.h):

    begin -> pass1 (stream x, y once: histogram + exact per-key partials)
          -> score (one CTA: partition, scores, precisions)
          -> pass2 (only if a HALF/SINGLE bin has upper != e for a member)
          -> finalize (per-bin values, Neumaier fold) -> fetch (small D2H)

The report's bounds are the fsum / left-to-right sums of the per-bin terms of
kernel.py:205-222, computed by the library's host code over the fetched bin
table (qdot_b200_bound_sums: exact, rounded once -- math.fsum's result).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

from . import _lib
from .binning import Bin, ExactBinning, Strategy, strategy_label
from .device import as_device_vector, config_struct, require_cuda, stream_handle, thread_state
from .exact import ReferenceResult, reference_dot  # noqa: F401  (kernel.py:75-133 live here in the reference)
from .scoring import ParameterSet, PrecisionLevel, SplitMode, ToleranceConfig

__all__ = ["QdotReport", "qdot", "select_parameters", "run_device", "ReferenceResult", "reference_dot"]


@dataclass
class QdotReport:
    """Value plus everything needed to audit it (kernel.py:136-168)."""

    value: float
    counts: Dict[PrecisionLevel, int]
    abs_bound: float
    rel_bound: float
    abs_cap: float
    rel_guarantee: float
    rel_hypothesis: str
    rel_bound_e: Optional[float]
    early_terminated: bool
    n: int
    epsilon: float
    split: SplitMode
    strategy: str
    phase_ns: Dict[str, int] = field(default_factory=dict)
    params: Optional[ParameterSet] = None
    # B200 extras (not in the reference report)
    pass2_needed: bool = False
    half_order_sensitive: bool = False   # a HALF bin's fp32 sequential sum depends on order ...
    half_ordered: bool = False           # ... and was replayed in index order (the value is the reference's)

    def count(self, level: PrecisionLevel) -> int:
        return self.counts.get(level, 0)

    def fraction(self, level: PrecisionLevel) -> float:
        return self.count(level) / self.n if self.n else 0.0


class _Indexer:
    """Materialises Bin.indices / ParameterSet.zero_idx on first access with
    the device counting-sort scatter (qdot_b200_bin_order: members of every
    bin in ascending index order, binning.py:46-55,88-116) and one D2H copy.

    Device inputs the caller owns are re-read at that point: an in-place
    modification after qdot() returned is detected (tensor version counter)
    and raises instead of slicing stale cardinalities.  Host inputs are kept
    as host tensors (no device copy stays alive) and uploaded again."""

    def __init__(self, xd, yd, n, norm, device, host=None):
        self.n, self.norm, self.device = n, norm, device
        if host is not None:                      # (xh, yh) host tensors
            self.xd = self.yd = None
            self.host = host
            self.version = None
        else:
            self.xd, self.yd, self.host = xd, yd, None
            self.version = (xd._version, yd._version)
        self.done = False

    def _inputs(self):
        import torch
        if self.host is not None:
            xh, yh = self.host
            xd = xh.to(self.device)
            return xd, (xd if self.norm else yh.to(self.device))
        if (self.xd._version, self.yd._version) != self.version:
            raise RuntimeError("qdot inputs were modified in place after the call; "
                               "Bin.indices would not match the report's bins")
        return self.xd, self.yd

    def materialize(self, params: ParameterSet) -> None:
        if self.done:
            return
        import torch
        lib = _lib.load()
        xd, yd = self._inputs()
        lut = np.full(_lib.KEYS, -1, dtype=np.int32)
        for b_id, b in enumerate(params.bins):
            lut[b.first_key:b.last_key + 1] = b_id
        nb = len(params.bins)
        lut_d = torch.from_numpy(lut).to(self.device)
        nbytes = int(lib.qdot_b200_order_scratch_bytes(self.n, nb))
        scratch = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=self.device)
        starts_d = torch.empty(nb + 2, dtype=torch.int64, device=self.device)
        order_d = torch.empty(max(self.n, 1), dtype=torch.int64, device=self.device)
        st = stream_handle(self.device)
        _lib.check(lib.qdot_b200_bin_order(xd.data_ptr(), yd.data_ptr(), self.n, int(self.norm), lut_d.data_ptr(),
                                           nb, None, starts_d.data_ptr(), order_d.data_ptr(), scratch.data_ptr(),
                                           nbytes, st), lib)
        starts = starts_d.cpu().numpy()
        order = order_d[:self.n].cpu().numpy()
        params._zero_idx = order[starts[0]:starts[1]]
        for i, b in enumerate(params.bins):
            b.indices = order[starts[i + 1]:starts[i + 2]]
        self.done = True
        self.xd = self.yd = self.host = None


def resolve_half_order(xd, yd, n: int, norm: bool, st, stream: int) -> None:
    """HALF bins finalize flagged order-sensitive: replay the reference's
    sequential fp32 sum in index order on the device (emulate.py:150-151),
    re-fold, and refresh st.result / st.bins (qdot_b200_half_ordered)."""
    import torch
    lib = _lib.load()
    res = st.result
    nb = int(res.n_bins)
    rows = _bin_rows(st.bins, nb)
    flagged = rows[(rows["precision"] == PrecisionLevel.HALF.code) & ((rows["flags"] & 1) != 0)]
    m = int(flagged["cardinality"].sum()) if flagged.size else 0
    nbytes = int(lib.qdot_b200_order_scratch_bytes(n, nb))
    scratch = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=xd.device)
    order = torch.empty(max(m, 1), dtype=torch.int64, device=xd.device)
    chain = torch.empty(max(nb, 1), dtype=torch.float32, device=xd.device)
    xp = xd.data_ptr()
    yp = xp if norm else yd.data_ptr()
    _lib.check(lib.qdot_b200_half_ordered(xp, yp, n, int(norm), st.ws_ptr, nb, order.data_ptr(), m,
                                          chain.data_ptr(), scratch.data_ptr(), nbytes, 7, stream), lib)
    _lib.check(lib.qdot_b200_fetch(st.ws_ptr, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, stream), lib)


def run_device(xd, yd, n: int, norm: bool, cfg: ToleranceConfig, strategy, st=None, timing: bool = True,
               stream=None):
    """Launch the whole device pipeline on device vectors; returns (result, bins, phase_ns)."""
    lib = _lib.load()
    if st is None:
        st = thread_state(xd.device)
    c = config_struct(cfg, strategy)
    s = stream_handle(xd.device) if stream is None else int(stream)
    ws = st.ws_ptr
    xp = xd.data_ptr()
    yp = xp if norm else yd.data_ptr()
    if not timing:
        # one C call: a cached CUDA graph of the whole pipeline, result published
        # to host-mapped memory (qdot_b200_dot)
        _lib.check(lib.qdot_b200_dot(xp, yp, n, int(norm), ctypes.byref(c), ws, ctypes.byref(st.result), st.bins,
                                     _lib.KEYS + 1, s), lib)
        res = st.result
        if res.half_order_sensitive == 1 and res.status == _lib.QDOT_OK:
            resolve_half_order(xd, yd, n, norm, st, s)
        return res, st.bins, {"select": int(res.select_ns), "compute": int(res.compute_ns), "reference": 0}
    torch_stream = None
    if timing:
        import torch
        torch_stream = torch.cuda.current_stream(xd.device) if stream is None else None
        if torch_stream is not None:
            st.ev[0].record(torch_stream)
    _lib.check(lib.qdot_b200_begin(ws, s), lib)
    _lib.check(lib.qdot_b200_pass1(xp, yp, n, int(norm), ctypes.byref(c), n, ws, s), lib)
    _lib.check(lib.qdot_b200_score_finalize(ws, n, ctypes.byref(c), s), lib)
    if torch_stream is not None:
        st.ev[1].record(torch_stream)
    _lib.check(lib.qdot_b200_pass2_finalize(xp, yp, n, int(norm), ws, s), lib)
    if torch_stream is not None:
        st.ev[2].record(torch_stream)
    _lib.check(lib.qdot_b200_fetch(ws, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, s), lib)
    if st.result.half_order_sensitive == 1 and st.result.status == _lib.QDOT_OK:
        resolve_half_order(xd, yd, n, norm, st, s)
    phase = {"select": 0, "compute": 0, "reference": 0}
    if torch_stream is not None:
        phase["select"] = int(st.ev[0].elapsed_time(st.ev[1]) * 1e6)
        phase["compute"] = int(st.ev[1].elapsed_time(st.ev[2]) * 1e6)
    return st.result, st.bins, phase


_BIN_DTYPE = np.dtype([("lower", "<i8"), ("upper", "<i8"), ("cardinality", "<i8"), ("score", "<i8"),
                       ("precision", "<i4"), ("first_key", "<i4"), ("last_key", "<i4"), ("flags", "<i4"),
                       ("value", "<f8")])
assert _BIN_DTYPE.itemsize == ctypes.sizeof(_lib.QdotBin)


def _bin_rows(cbins, n_bins: int) -> np.ndarray:
    """A private, read-only copy of the first n_bins device bin records (the
    ctypes table is reused by the next call on this thread); string_at copies
    the bytes without the buffer protocol's per-call format parsing."""
    if n_bins <= 0:
        return np.zeros(0, dtype=_BIN_DTYPE)
    return np.frombuffer(ctypes.string_at(ctypes.addressof(cbins), n_bins * _BIN_DTYPE.itemsize), dtype=_BIN_DTYPE)


def _bound_sums(cbins, n_bins: int, shift: int):
    """(fsum, left-to-right sum) of M * ldexp(eps(precision), upper - shift + 1)
    over the fetched bin table (scoring.py:171-199, kernel.py:205-222), in the
    library's host code (qdot_b200_bound_sums: exact big-integer sum rounded
    once, i.e. math.fsum).  OverflowError where math.ldexp / fsum raise it."""
    lib = _lib.load()
    out = (ctypes.c_double * 2)()
    rc = lib.qdot_b200_bound_sums(cbins, int(n_bins), int(shift), out)
    if rc == _lib.QDOT_ERR_OVERFLOW:
        raise OverflowError("math range error")
    _lib.check(rc, lib)
    return out[0], out[1]


def _bound_sums2(cbins, n_bins: int, shift_a: int, shift_b: int):
    """_bound_sums for two shifts in one library call: (fsum_a, plain_a, fsum_b, plain_b)."""
    lib = _lib.load()
    out = (ctypes.c_double * 4)()
    rc = lib.qdot_b200_bound_sums2(cbins, int(n_bins), int(shift_a), int(shift_b), out)
    if rc == _lib.QDOT_ERR_OVERFLOW:
        raise OverflowError("math range error")
    _lib.check(rc, lib)
    return out[0], out[1], out[2], out[3]


def _make_bin_objects(rows: np.ndarray, indexer):
    def make(ps):
        return [Bin(lower=int(r["lower"]), upper=int(r["upper"]), cardinality=int(r["cardinality"]),
                    score=int(r["score"]), precision=PrecisionLevel.from_code(int(r["precision"])),
                    value=float(r["value"]), flags=int(r["flags"]), first_key=int(r["first_key"]),
                    last_key=int(r["last_key"]), indexer=indexer, owner=ps) for r in rows]
    return make


def _build_params(res, cbins, cfg, strategy, indexer, rows=None, rel=None) -> ParameterSet:
    if rows is None:
        rows = _bin_rows(cbins, int(res.n_bins))
    ps = ParameterSet(bins=None, e_min=int(res.e_min), e_max=int(res.e_max), strategy=strategy, tolerance=cfg,
                      early_terminated=bool(res.early_terminated), n=int(res.n), eps_eff=float(res.eps_eff),
                      n_bins=int(res.n_bins), zero_count=int(res.zero_count), _indexer=indexer,
                      _make_bins=_make_bin_objects(rows, indexer))
    # ParameterSet.rel_bound: plain left-to-right sum from 0.0 (scoring.py:195-199);
    # the report's rel_bound: fsum of the same terms (kernel.py:213)
    ps._rel_fsum, ps.rel_bound = rel if rel is not None else _bound_sums(cbins, int(res.n_bins), int(res.e_max))
    return ps


def _prepare(x, y):
    torch = require_cuda()
    is_norm = x is y                                           # kernel.py:194
    # fast path: 1-D contiguous float64 tensors already on the current device
    if type(x) is torch.Tensor and (is_norm or type(y) is torch.Tensor):
        dev = x.device
        if (x.is_cuda and x.dtype is torch.float64 and x.dim() == 1 and x.is_contiguous()
                and dev.index == torch.cuda.current_device()
                and (is_norm or (y.device == dev and y.dtype is torch.float64 and y.dim() == 1
                                 and y.is_contiguous()))):
            if not is_norm and x.shape[0] != y.shape[0]:       # floatbits.py:68-69
                raise ValueError(f"length mismatch: {x.shape[0]} vs {y.shape[0]}")
            return is_norm, x, (x if is_norm else y)
    device = torch.device("cuda", torch.cuda.current_device())
    xd, _ = as_device_vector(x, device)
    yd = xd if is_norm else as_device_vector(y, device)[0]
    if xd.shape[0] != yd.shape[0]:                             # floatbits.py:68-69
        raise ValueError(f"length mismatch: {xd.shape[0]} vs {yd.shape[0]}")
    return is_norm, xd, yd


def select_parameters(x, y, cfg: ToleranceConfig, strategy: Strategy = None) -> ParameterSet:
    """Parameter selection only (kernel.py:34-72): pass1 + score on the device."""
    if strategy is None:
        strategy = ExactBinning()
    is_norm, xd, yd = _prepare(x, y)
    n = int(xd.shape[0])
    lib = _lib.load()
    st = thread_state(xd.device)
    c = config_struct(cfg, strategy)
    s = stream_handle(xd.device)
    ws = st.ws_ptr
    _lib.check(lib.qdot_b200_begin(ws, s), lib)
    _lib.check(lib.qdot_b200_pass1(xd.data_ptr(), yd.data_ptr(), n, int(is_norm), ctypes.byref(c), n, ws, s), lib)
    _lib.check(lib.qdot_b200_score_finalize(ws, n, ctypes.byref(c), s), lib)
    # finalize also fills the result header and per-bin values; cheap (1 CTA)
    _lib.check(lib.qdot_b200_pass2_finalize(xd.data_ptr(), yd.data_ptr(), n, int(is_norm), ws, s), lib)
    _lib.check(lib.qdot_b200_fetch(ws, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, s), lib)
    res = st.result
    _raise_status(res)
    indexer = _Indexer(xd, yd, n, is_norm, xd.device)
    return _build_params(res, st.bins, cfg, strategy, indexer)


def _raise_status(res) -> None:
    if res.status == _lib.QDOT_ERR_OVERFLOW:
        raise OverflowError("math range error")
    _lib.check(int(res.status))


_LEVELS4 = (PrecisionLevel.PERFORATE, PrecisionLevel.HALF, PrecisionLevel.SINGLE, PrecisionLevel.DOUBLE)


def report_from_result(res, cbins, cfg, strategy, is_norm, reference, phase, indexer) -> QdotReport:
    """Host-side report assembly (kernel.py:205-240)."""
    rows = _bin_rows(cbins, int(res.n_bins))
    # the rel terms at e_max (params), then the abs terms: one library call, same order
    rf, rp, abs_bound, _ = _bound_sums2(cbins, int(res.n_bins), int(res.e_max), 0)
    params = _build_params(res, cbins, cfg, strategy, indexer, rows, rel=(rf, rp))
    rel_bound = params._rel_fsum
    rel_hypothesis = "assumed"
    rel_bound_e = None
    if is_norm:
        rel_hypothesis = "holds"
    if reference is not None:
        fe = getattr(reference, "flexp_e", None)
        if fe is None:
            rel_hypothesis = "violated" if not is_norm else rel_hypothesis
        else:
            holds = params.e_max <= fe or rows.size == 0
            rel_hypothesis = "holds" if (holds or is_norm) else "violated"
            rel_bound_e = _bound_sums(cbins, int(res.n_bins), int(fe))[0]
    counts = dict(zip(_LEVELS4, res.counts))                  # PERFORATE, HALF, SINGLE, DOUBLE
    return QdotReport(
        value=float(res.value), counts=counts, abs_bound=abs_bound, rel_bound=rel_bound,
        abs_cap=2.0 * abs_bound, rel_guarantee=params.rel_guarantee, rel_hypothesis=rel_hypothesis,
        rel_bound_e=rel_bound_e, early_terminated=params.early_terminated, n=params.n,
        epsilon=cfg.epsilon, split=cfg.split, strategy=strategy_label(params.strategy),
        phase_ns=phase, params=params, pass2_needed=bool(res.pass2_needed),
        half_order_sensitive=bool(res.half_order_sensitive), half_ordered=int(res.half_order_sensitive) == 2)


# host inputs at least this long are streamed to the device in chunks that
# pass 1 consumes while the next chunk is in flight (copy / compute overlap;
# pageable memory through the library's pinned staging ring, csrc/qdot_host.cu)
PIPELINE_MIN = 1 << 22


def _host_vector(a):
    """1-D float64 contiguous CPU torch tensor for a host input, or None when `a`
    is already on a CUDA device."""
    import torch
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            return None
        t = a
        if t.dim() != 1:
            raise ValueError("inputs must be 1-D arrays")
        return t.to(torch.float64).contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError("inputs must be 1-D arrays")
    return torch.from_numpy(arr)


def h2d_pass1(xh, yh, norm: bool, c, n_total: int, st, device):
    """Copy host vectors (pageable or pinned) into new device buffers chunk by
    chunk while pass 1 consumes each landed chunk on the current stream
    (workspace already begun): qdot_b200_pass1_host.  Returns the device vectors."""
    import torch
    n = int(xh.shape[0])
    lib = _lib.load()
    s = torch.cuda.current_stream(device).cuda_stream
    xd = torch.empty(n, dtype=torch.float64, device=device)
    yd = xd if norm else torch.empty(n, dtype=torch.float64, device=device)
    _lib.check(lib.qdot_b200_pass1_host(xh.data_ptr(), xh.data_ptr() if norm else yh.data_ptr(), n, int(norm),
                                        ctypes.byref(c), n_total, st.ws_ptr, xd.data_ptr(),
                                        xd.data_ptr() if norm else yd.data_ptr(), s), lib)
    return xd, yd


def _run_host_pipelined(xh, yh, norm: bool, cfg: ToleranceConfig, strategy):
    """H2D of chunk k+1 (copy stream) overlaps pass 1 on chunk k (compute
    stream); then score / pass 2 / finalize on the resident vectors.
    Returns (result, bins, phase_ns, xd, yd)."""
    import torch
    device = torch.device("cuda", torch.cuda.current_device())
    n = int(xh.shape[0])
    lib = _lib.load()
    st = thread_state(device)
    c = config_struct(cfg, strategy)
    comp = torch.cuda.current_stream(device)
    s = comp.cuda_stream
    ws = st.ws_ptr
    _lib.check(lib.qdot_b200_begin(ws, s), lib)
    xd, yd = h2d_pass1(xh, yh, norm, c, n, st, device)
    _lib.check(lib.qdot_b200_score_finalize(ws, n, ctypes.byref(c), s), lib)
    _lib.check(lib.qdot_b200_pass2_finalize(xd.data_ptr(), yd.data_ptr(), n, int(norm), ws, s), lib)
    _lib.check(lib.qdot_b200_fetch(ws, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, s), lib)
    res = st.result
    if res.half_order_sensitive == 1 and res.status == _lib.QDOT_OK:
        resolve_half_order(xd, yd, n, norm, st, s)
    phase = {"select": int(res.select_ns), "compute": int(res.compute_ns), "reference": 0}
    return res, st.bins, phase, xd, yd


def qdot(x, y, cfg: ToleranceConfig, strategy: Strategy = None, reference=None) -> QdotReport:
    """Approximate dot product with audit report (kernel.py:179-240).

    x, y: array-likes (coerced like np.ascontiguousarray(float64) and copied
    to the current CUDA device) or CUDA/CPU torch tensors (float64 CUDA
    tensors are used in place).  ``x is y`` selects norm mode (one read).
    Long host inputs are streamed in chunks with the copy overlapping pass 1.
    """
    if strategy is None:
        strategy = ExactBinning()
    torch = require_cuda()
    is_norm = x is y                                           # kernel.py:194
    xh = None if (type(x) is torch.Tensor and x.is_cuda) else _host_vector(x)   # device tensors: no host staging
    if xh is not None and xh.shape[0] >= PIPELINE_MIN:
        yh = xh if is_norm else _host_vector(y)
        if yh is not None:
            if xh.shape[0] != yh.shape[0]:                     # floatbits.py:68-69
                raise ValueError(f"length mismatch: {xh.shape[0]} vs {yh.shape[0]}")
            n = int(xh.shape[0])
            res, cbins, phase, xd, yd = _run_host_pipelined(xh, yh, is_norm, cfg, strategy)
            _raise_status(res)
            indexer = _Indexer(None, None, n, is_norm, xd.device, host=(xh, yh))
            del xd, yd
            return report_from_result(res, cbins, cfg, strategy, is_norm, reference, phase, indexer)
    is_norm, xd, yd = _prepare(x, y)
    n = int(xd.shape[0])
    # one C call (cached CUDA graph, host-mapped result); phase_ns comes from
    # device timestamps (select: pass 1 + scoring, compute: pass 2 + finalize)
    res, cbins, phase = run_device(xd, yd, n, is_norm, cfg, strategy, timing=False)
    _raise_status(res)
    indexer = _Indexer(xd, yd, n, is_norm, xd.device)
    return report_from_result(res, cbins, cfg, strategy, is_norm, reference, phase, indexer)
