"""Multi-rank host logic on CPU (gloo, world_size 2).

The N-GPU path exchanges two int64 workspace regions with a SUM allreduce
(paper_2105_00115_b200.dist).  These tests run that exchange with real
torch.distributed processes over gloo: each rank builds its shard's region
contents with a numpy model of the device format (exponent histogram, zero
count, DOUBLE partials as 32-bit limbs), the product's reduce_regions sums
them, and the decoded totals must equal the whole-vector values -- including
the oracle's histogram.  The CUDA kernels themselves are covered by the GPU
tests (tests/test_gpu_parity.py::test_sharded_tables_sum_like_one_device).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.dist import chain_in_rank_order, reduce_regions, shard_bounds

KEYS, KOFF = _lib.KEYS, _lib.KEY_OFFSET


def _flexp(a):
    return np.frexp(np.abs(a))[1].astype(np.int64) - 1


def model_regions(x, y, a_len, b_len):
    """numpy model of pass-1 regions A and B for one shard (device format)."""
    A = np.zeros(a_len, dtype=np.int64)
    B = np.zeros(b_len, dtype=np.int64)
    z = (x == 0) | (y == 0)
    A[KEYS] = int(z.sum())
    xs, ys = x[~z], y[~z]
    e = _flexp(xs) + _flexp(ys)
    keys = e + KOFF
    np.add.at(A, keys, 1)
    p = xs * ys
    qd = np.maximum(e - 52, -1074)
    k = np.ldexp(p, -qd).astype(np.int64)           # exact integer units
    np.add.at(B, keys, k & 0xFFFFFFFF)              # D0 limb
    np.add.at(B, KEYS + keys, k >> 32)              # D1 limb
    return A, B


def decode_d(B, key):
    return (int(B[key]) + (int(B[KEYS + key]) << 32) + (int(B[2 * KEYS + key]) << 64)
            + (int(B[3 * KEYS + key]) << 96))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        x = np.ldexp(rng.uniform(0.5, 1, n) * rng.choice([-1, 1], n), rng.integers(-40, 40, n))
        y = np.ldexp(rng.uniform(0.5, 1, n), rng.integers(-40, 40, n))
        x[rng.integers(0, n, n // 20)] = 0.0
        lo, hi = shard_bounds(n, rank, world)
        a_len, b_len = 12672, 37760
        A, B = model_regions(x[lo:hi], y[lo:hi], a_len, b_len)
        ta, tb = torch.from_numpy(A), torch.from_numpy(B)
        reduce_regions(ta, tb)
        if rank == 0:
            FA, FB = model_regions(x, y, a_len, b_len)
            ok_a = bool(torch.equal(ta, torch.from_numpy(FA)))
            ok_b = all(decode_d(tb.numpy(), k) == decode_d(FB, k) for k in np.flatnonzero(FA[:KEYS]))
            from oracle import oracle as O
            hist, zc = O.hist(x, y)
            ok_o = bool(np.array_equal(ta.numpy()[:KEYS], hist)) and int(ta[KEYS]) == zc
            q.put((ok_a, ok_b, ok_o))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 10001), (3, 4099)])
def test_gloo_region_exchange_is_exact(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == (True, True, True)


def _chain_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        vals = np.abs(rng.standard_normal((3, n))).astype(np.float16).astype(np.float32)   # 3 "bins"
        lo, hi = shard_bounds(n, rank, world)
        chain = torch.zeros(3, dtype=torch.float32)

        def run(c):                                  # this rank's part of each fp32 running sum
            for b in range(3):
                s = np.float32(c[b].item())
                for v in vals[b, lo:hi]:
                    s = np.float32(s + v)
                c[b] = float(s)
        chain_in_rank_order(chain, run)
        want = []
        for b in range(3):                           # emulate.py:105-108 over the whole vector
            s = np.float32(0.0)
            for v in vals[b]:
                s = np.float32(s + v)
            want.append(float(s))
        q.put((rank, chain.tolist() == want))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_half_chain_runs_in_rank_order(world):
    """The HALF order-sensitive fallback over shards (dist.half_chain_sharded):
    fp32 running sums continued rank after rank equal the single sequential sum."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, world, port, 30011, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res.values()) and len(res) == world


def test_shard_bounds_partition():
    for n in [0, 1, 7, 1000, (1 << 31) + 5]:
        for world in [1, 2, 3, 8]:
            prev = 0
            sizes = []
            for r in range(world):
                lo, hi = shard_bounds(n, r, world)
                assert lo == prev
                prev = hi
                sizes.append(hi - lo)
            assert prev == n and max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_d_limb_encoding_survives_large_sums():
    """Per-key DOUBLE partials beyond 2^63 (n * 2^54) decode exactly from 32-bit limbs."""
    big = (1 << 54) - 1
    B = np.zeros(37760, dtype=np.int64)
    total = 0
    for _ in range(3):                   # three "ranks" each adding 2^20 maximal products
        v = big << 20
        total += v
        B[5] += v & 0xFFFFFFFF
        B[KEYS + 5] += (v >> 32) & 0xFFFFFFFF
        B[2 * KEYS + 5] += (v >> 64) & 0xFFFFFFFF
        B[3 * KEYS + 5] += v >> 96
    assert decode_d(B, 5) == total and total > (1 << 63)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_sharded_needs_cuda():
    import paper_2105_00115_b200 as Q
    from paper_2105_00115_b200.dist import qdot_sharded
    with pytest.raises(RuntimeError):
        qdot_sharded(np.ones(4), np.ones(4), Q.ToleranceConfig(1e-6))
