"""Exact dot product on the device: the verification oracle
kernel.reference_dot (kernel.py:75-133) re-done B200-side.

    reference_dot(x, y, plain=True) -> ReferenceResult(value, flexp_e, plain)

value is the correctly rounded x.y (the reference's Dekker + math.fsum /
Fraction result), flexp_e = flexp(value) or None for a zero dot, plain the
left-to-right double sum of the rounded products.  Same ValueError /
OverflowError behaviour.  Computed by csrc/qdot_exact.cu: one streaming pass
accumulating every exact product mx*my*2^q in integer limbs per exponent,
one rounding at the end -- so it verifies qdot at 2^28..2^31 elements
without a 150 GB host run.  `plain` is a serial one-thread sum (about 1 ns
per element); pass plain=False to skip it (then plain is NaN).

reference_dot_sharded(x_local, y_local) is the multi-GPU form: every rank
accumulates its contiguous shard, the integer accumulator region is
SUM-allreduced (exact for any rank count), every rank rounds the same total.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

from . import _lib
from .device import as_device_vector, require_cuda, stream_handle

__all__ = ["ReferenceResult", "reference_dot", "reference_dot_sharded"]


@dataclass
class ReferenceResult:
    """Verification-grade dot product: value is correctly rounded (<1 ulp)."""

    value: float
    flexp_e: Optional[int]       # flexp(x . y), None when the dot is 0
    plain: float                 # left-to-right double dot, the baseline kernel


class _ExactWs:
    def __init__(self, device):
        torch = require_cuda()
        lib = _lib.load()
        self.buf = torch.empty(int(lib.qdot_b200_exact_workspace_bytes()) // 8, dtype=torch.int64, device=device)
        self.region_words = int(lib.qdot_b200_exact_region_words())

    @property
    def ptr(self):
        return self.buf.data_ptr()


def _prepare(x, y):
    torch = require_cuda()
    norm = x is y
    device = torch.device("cuda", torch.cuda.current_device())
    xd, _ = as_device_vector(x, device)
    yd = xd if norm else as_device_vector(y, device)[0]
    if xd.shape != yd.shape:                                    # kernel.py:106-107
        raise ValueError("reference_dot needs equal-length 1-D arrays")
    return norm, xd, yd, device


def _finish(lib, ws, xd, yd, n, norm, plain, s) -> ReferenceResult:
    if plain and n:
        _lib.check(lib.qdot_b200_exact_plain(xd.data_ptr(), yd.data_ptr(), n, int(norm), ws.ptr, s), lib)
    _lib.check(lib.qdot_b200_exact_finalize(ws.ptr, s), lib)
    r = _lib.QdotExactResult()
    _lib.check(lib.qdot_b200_exact_fetch(ws.ptr, ctypes.byref(r), s), lib)
    if r.status == _lib.QDOT_ERR_NONFINITE:
        raise ValueError("inputs must be finite")               # kernel.py:112-113
    if r.status == _lib.QDOT_ERR_OVERFLOW:
        raise OverflowError("true dot product overflows double")  # kernel.py:130-131
    _lib.check(int(r.status), lib)
    value = float(r.value)
    return ReferenceResult(value=value, flexp_e=None if r.is_zero else int(r.flexp_e),
                           plain=float(r.plain) if plain else math.nan)


def reference_dot(x, y, plain: bool = True) -> ReferenceResult:
    """Correctly rounded dot product of two equal-length 1-D vectors (kernel.py:98-133)."""
    norm, xd, yd, device = _prepare(x, y)
    n = int(xd.shape[0])
    if n == 0:
        return ReferenceResult(value=0.0, flexp_e=None, plain=0.0)
    lib = _lib.load()
    ws = _ExactWs(device)
    s = stream_handle(device)
    _lib.check(lib.qdot_b200_exact_begin(ws.ptr, s), lib)
    _lib.check(lib.qdot_b200_exact_accumulate(xd.data_ptr(), yd.data_ptr(), n, int(norm), ws.ptr, s), lib)
    return _finish(lib, ws, xd, yd, n, norm, plain, s)


def reference_dot_sharded(x_local, y_local, group=None) -> ReferenceResult:
    """Exact dot of vectors sharded contiguously over the ranks of `group`.
    plain (a serial left-to-right sum over all ranks) is not formed: NaN."""
    import torch.distributed as dist
    norm, xd, yd, device = _prepare(x_local, y_local)
    n = int(xd.shape[0])
    lib = _lib.load()
    ws = _ExactWs(device)
    s = stream_handle(device)
    _lib.check(lib.qdot_b200_exact_begin(ws.ptr, s), lib)
    _lib.check(lib.qdot_b200_exact_accumulate(xd.data_ptr(), yd.data_ptr(), n, int(norm), ws.ptr, s), lib)
    region = ws.buf[:ws.region_words]
    dist.all_reduce(region, op=dist.ReduceOp.SUM, group=group)
    return _finish(lib, ws, xd, yd, n, norm, False, s)
