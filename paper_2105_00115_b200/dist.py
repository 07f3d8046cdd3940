"""Multi-GPU qdot: one process per GPU, contiguous shards, two integer allreduces.

    qdot_sharded(x_local, y_local, cfg, strategy=None, group=None) -> QdotReport

Every rank holds a contiguous shard [lo, hi) of the two vectors (see
shard_bounds).  Per call and rank (all stream-ordered, one host sync at the end):

    begin -> pass1(local shard)                      histogram + exact partials
          -> allreduce(region A, SUM)  [NCCL]        ~67 KB: histogram, zero count,
                                                      non-finite count, hot flags
          -> score (identical inputs on every rank -> identical bins everywhere)
          -> pass2(local shard)                      only if scoring asked for it
          -> allreduce(region B, SUM)  [NCCL]        ~300 KB: exact per-key partials
          -> finalize -> fetch

Both regions hold integers (counts and 32-bit limbs in int64 words), so the
sums are exact and the result is bit-identical for any number of ranks and
any reduction order -- the same bins, precisions and value as one device
running over the concatenated vectors.  The reference has no distributed
path; this is the B200 build's sharding of the same result.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Tuple

from . import _lib
from .binning import ExactBinning, Strategy
from .device import as_device_vector, config_struct, require_cuda, stream_handle, thread_state
from .kernel import QdotReport, _raise_status, report_from_result
from .scoring import ToleranceConfig


def shard_bounds(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced shard [lo, hi) of n elements for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def reduce_regions(region_a, region_b=None, group=None) -> None:
    """In-place SUM allreduce of the workspace regions (int64 tensors).

    Backend-agnostic (NCCL for CUDA tensors, gloo for CPU tensors in tests);
    exactness relies only on integer addition."""
    import torch.distributed as dist
    dist.all_reduce(region_a, op=dist.ReduceOp.SUM, group=group)
    if region_b is not None:
        dist.all_reduce(region_b, op=dist.ReduceOp.SUM, group=group)


def _p2p(tensor, peer: int, send: bool, group) -> None:
    """send / recv of a small tensor; gloo groups move it through host memory."""
    import torch.distributed as dist
    if group is not None:
        peer = dist.get_global_rank(group, peer)
    if dist.get_backend(group) == "gloo" and tensor.is_cuda:
        h = tensor.cpu()
        if send:
            dist.send(h, dst=peer, group=group)
        else:
            dist.recv(h, src=peer, group=group)
            tensor.copy_(h)
        return
    (dist.send if send else dist.recv)(tensor, peer, group=group)


def chain_in_rank_order(chain, run, group=None) -> None:
    """Run `run(chain)` rank after rank: rank r receives rank r-1's chain
    values into `chain` before its run and sends them on after it; then every
    rank receives the last rank's values (broadcast)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if rank > 0:
        _p2p(chain, rank - 1, False, group)
    run(chain)
    if rank < world - 1:
        _p2p(chain, rank + 1, True, group)
    last = dist.get_global_rank(group, world - 1) if group is not None else world - 1
    if dist.get_backend(group) == "gloo" and chain.is_cuda:
        h = chain.cpu()
        dist.broadcast(h, src=last, group=group)
        chain.copy_(h)
    else:
        dist.broadcast(chain, src=last, group=group)


def half_chain_sharded(xd, yd, n: int, norm: bool, st, stream: int, group=None) -> None:
    """HALF bins flagged order-sensitive over contiguous shards: every rank
    orders its members of those bins (stage 1), then the fp32 running sums
    run rank after rank -- rank r continues from rank r-1's chain values
    (stage 2, a send/recv of n_bins floats) -- and every rank applies the last
    rank's chains (stage 4).  The value equals one device's on the
    concatenated vectors (the reference's index-order fp32 sum)."""
    import torch
    from .kernel import _bin_rows
    from .scoring import PrecisionLevel
    lib = _lib.load()
    nb = int(st.result.n_bins)
    rows = _bin_rows(st.bins, nb)
    flagged = rows[(rows["precision"] == PrecisionLevel.HALF.code) & ((rows["flags"] & 1) != 0)]
    m = min(n, int(flagged["cardinality"].sum())) if flagged.size else 0
    nbytes = int(lib.qdot_b200_order_scratch_bytes(n, nb))
    scratch = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=xd.device)
    order = torch.empty(max(m, 1), dtype=torch.int64, device=xd.device)
    chain = torch.zeros(max(nb, 1), dtype=torch.float32, device=xd.device)
    xp = xd.data_ptr()
    yp = xp if norm else yd.data_ptr()

    def stage(k):
        _lib.check(lib.qdot_b200_half_ordered(xp, yp, n, int(norm), st.ws_ptr, nb, order.data_ptr(), m,
                                              chain.data_ptr(), scratch.data_ptr(), nbytes, k, stream), lib)
    stage(1)
    chain_in_rank_order(chain, lambda c: stage(2), group)
    stage(4)
    del order, scratch
    _lib.check(lib.qdot_b200_fetch(st.ws_ptr, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, stream), lib)


class _ShardedIndexer:
    """Bin.indices of a sharded report would need an all-gather; refuse loudly."""

    def materialize(self, params):
        raise RuntimeError("Bin.indices is not materialised for sharded qdot reports "
                           "(each rank holds only its shard)")


def qdot_sharded(x_local, y_local, cfg: ToleranceConfig, strategy: Strategy = None, group=None,
                 n_total: Optional[int] = None, reference=None) -> QdotReport:
    """qdot over vectors sharded across the ranks of `group` (collective call).

    x_local, y_local: this rank's contiguous shard (CUDA tensors or
    array-likes).  Returns the same report on every rank, equal to
    qdot(concat(x), concat(y), cfg, strategy) on one device.
    """
    import torch
    import torch.distributed as dist
    require_cuda()
    if strategy is None:
        strategy = ExactBinning()
    is_norm = x_local is y_local
    device = torch.device("cuda", torch.cuda.current_device())
    from .kernel import PIPELINE_MIN, _host_vector, h2d_pass1
    xh = _host_vector(x_local)
    yh = None if xh is None else (xh if is_norm else _host_vector(y_local))
    if xh is not None and yh is not None and xh.shape[0] != yh.shape[0]:
        raise ValueError(f"length mismatch: {xh.shape[0]} vs {yh.shape[0]}")
    streamed = xh is not None and yh is not None and xh.shape[0] >= PIPELINE_MIN
    if not streamed:
        xd, _ = as_device_vector(x_local, device)
        yd = xd if is_norm else as_device_vector(y_local, device)[0]
        if xd.shape[0] != yd.shape[0]:
            raise ValueError(f"length mismatch: {xd.shape[0]} vs {yd.shape[0]}")
    n = int(xh.shape[0]) if streamed else int(xd.shape[0])
    if n_total is None:
        t = torch.tensor([n], dtype=torch.int64, device=device)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())
    lib = _lib.load()
    st = thread_state(device)
    c = config_struct(cfg, strategy)
    s = stream_handle(device)
    ws = st.ws_ptr
    _lib.check(lib.qdot_b200_begin(ws, s), lib)
    if streamed:        # host shard: H2D in chunks overlapping pass 1
        xd, yd = h2d_pass1(xh, yh, is_norm, c, n_total, st, device)
    xp = xd.data_ptr()
    yp = xp if is_norm else yd.data_ptr()
    if not streamed:
        _lib.check(lib.qdot_b200_pass1(xp, yp, n, int(is_norm), ctypes.byref(c), n_total, ws, s), lib)
    reduce_regions(st.region_a(), None, group)
    _lib.check(lib.qdot_b200_score(ws, n_total, ctypes.byref(c), s), lib)
    _lib.check(lib.qdot_b200_pass2(xp, yp, n, int(is_norm), ws, s), lib)
    dist.all_reduce(st.region_b(), op=dist.ReduceOp.SUM, group=group)
    _lib.check(lib.qdot_b200_finalize(ws, s), lib)
    _lib.check(lib.qdot_b200_fetch(ws, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, s), lib)
    if st.result.half_order_sensitive == 1 and st.result.status == _lib.QDOT_OK:
        half_chain_sharded(xd, yd, n, is_norm, st, s, group)
    _raise_status(st.result)
    phase = {"select": 0, "compute": 0, "reference": 0}
    return report_from_result(st.result, st.bins, cfg, strategy, is_norm, reference, phase, _ShardedIndexer())
