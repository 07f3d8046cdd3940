"""Device plumbing: input staging, per-thread workspaces, streams, events.

torch is used only for device memory, streams and (in dist.py) collectives;
all arithmetic on the vectors happens in lib/libqdot_b200.so.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .binning import strategy_code
from .scoring import SplitMode

_tls = threading.local()

# pass-1 lean/full choice: 0 = per-CTA auto (default), 1 = force lean, 2 = force
# full variants.  Only speed depends on it (tests run all three).
PASS1_MODE = int(os.environ.get("QDOT_B200_PASS1_MODE", "0"))


def _torch():
    import torch
    return torch


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    torch = _torch()
    if not _CUDA_OK:                      # a success is cached; a failure raises every time
        if not torch.cuda.is_available():
            raise RuntimeError("qdot_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
        _CUDA_OK = True
    return torch


def as_device_vector(a, device):
    """1-D contiguous float64 CUDA tensor for `a`, plus the host array it came
    from (numpy inputs) so lazy index materialisation can re-read it.

    Array-likes are coerced exactly like the reference (np.ascontiguousarray
    with dtype float64, kernel.py:195-196)."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t = a
        if t.dim() != 1:
            raise ValueError("inputs must be 1-D arrays")
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        if t.device != device:
            t = t.to(device)
        return t.contiguous(), None
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError("inputs must be 1-D arrays")
    t = torch.from_numpy(arr).to(device, non_blocking=False)
    return t, arr


class ThreadState:
    """Per host thread and device: workspace, result buffers, timing events."""

    def __init__(self, device):
        torch = _torch()
        lib = _lib.load()
        self.device = device
        self.ws_bytes = int(lib.qdot_b200_workspace_bytes())
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        self.layout = _lib.layout()
        self.result = _lib.QdotResult()
        self.bins = (_lib.QdotBin * (_lib.KEYS + 1))()
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    @property
    def ws_ptr(self) -> int:
        return self.ws.data_ptr()

    def region_a(self):
        lay = self.layout
        return self.ws[lay.a_offset:lay.a_offset + 8 * lay.a_len].view(_torch().int64)

    def region_b(self):
        lay = self.layout
        return self.ws[lay.b_offset:lay.b_offset + 8 * lay.b_len].view(_torch().int64)


def thread_state(device=None) -> ThreadState:
    torch = require_cuda()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    states = getattr(_tls, "states", None)
    if states is None:
        states = _tls.states = {}
    key = (device.type, device.index)
    st = states.get(key)
    if st is None:
        st = states[key] = ThreadState(device)
    return st


def stream_handle(device) -> int:
    """The current CUDA stream of `device` (torch's raw getter: the Stream
    object of torch.cuda.current_stream costs several microseconds per call)."""
    torch = _torch()
    idx = device.index if getattr(device, "index", None) is not None else torch.cuda.current_device()
    return int(torch._C._cuda_getCurrentRawStream(idx))


def config_struct(cfg, strategy) -> _lib.QdotConfig:
    code, param = strategy_code(strategy)
    return _lib.QdotConfig(float(cfg.epsilon), 1 if cfg.split == SplitMode.PER_BIN else 0, int(cfg.input_mu), code,
                           PASS1_MODE, param)
