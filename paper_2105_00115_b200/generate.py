"""Synthetic input vectors generated on the device (csrc/qdot_gen.cu).

    device_vectors(law, n, seed=0, offset=0, param=0.0, norm=False) -> (x, y)

Each element is a pure function of (law, param, seed, global index), so
rank r of G can generate exactly its contiguous shard [offset, offset + n)
of one global vector pair -- sharded runs see the same data as one device.
Laws follow the numpy generators of SURVEY.md §8d and harness.py:61-76 but
are not their bytes (the host generators stay for golden / CSV parity).
"""

from __future__ import annotations

from . import _lib
from .device import require_cuda, stream_handle

LAWS = {"normal": 0, "illcond": 1, "A": 2, "B": 3}


def device_vectors(law: str, n: int, seed: int = 0, offset: int = 0, param: float = 0.0, norm: bool = False,
                   device=None):
    """float64 CUDA tensors x, y (y is x when norm) for elements
    [offset, offset + n) of the law's global vector pair."""
    torch = require_cuda()
    if law not in LAWS:
        raise ValueError(f"unknown law {law!r}; one of {sorted(LAWS)}")
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    x = torch.empty(n, dtype=torch.float64, device=device)
    y = x if norm else torch.empty(n, dtype=torch.float64, device=device)
    lib = _lib.load()
    _lib.check(lib.qdot_b200_generate(LAWS[law], float(param), int(seed) & (2**64 - 1), int(offset), int(n),
                                      x.data_ptr() if n else None, None if norm or not n else y.data_ptr(),
                                      stream_handle(device)), lib)
    return x, y
