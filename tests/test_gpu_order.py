"""Member order on the device (csrc/qdot_order.cu).

* Bin.indices / zero_idx from the stable counting-sort scatter equal the
  reference's order (binning.py:46-55, 88-116, 218, 270; floatbits.py:74-76):
  against the oracle's members on inputs with many bins, many segments,
  ragged lengths, zeros, every strategy and the early-terminated bin.
* HALF bins whose fp32 sequential sum is order-sensitive are replayed in
  index order (emulate.py:150-151): the value is the reference's bit for bit,
  also on several emulated contiguous shards chaining their fp32 sums.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_00115_b200 as Q  # noqa: E402
from paper_2105_00115_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402


def members_equal(rep, ref, x, y):
    assert rep.params.zero_idx.tolist() == np.flatnonzero((x == 0) | (y == 0)).tolist()
    assert len(rep.params.bins) == len(ref.bins)
    for b, w in zip(rep.params.bins, ref.bins):
        assert np.array_equal(b.indices, w.indices), (b.lower, b.upper)


@pytest.mark.parametrize("gen,n,strategy,eps", [
    ("illcond", (1 << 18) + 5, "exact", 1e-12),         # ~360 bins, wide keys
    ("illcond", (1 << 18) + 5, "ranged:7", 1e-12),
    ("illcond", 100003, "split:9", 1e-12),
    ("normal", (1 << 21) + 31, "exact", 1e-8),          # many segments per slot
    ("normal", 4097, "split:2", 1e-8),
    ("normal", 77, "exact", 1e-2),                      # early-terminated single bin
    ("normal", 1, "exact", 1e-8),
])
def test_indices_match_oracle(gen, n, strategy, eps):
    if gen == "illcond":
        x, y = O.gen_illcond(n - n % 2, seed=7)
        x = np.concatenate([x, np.ones(n % 2)])
        y = np.concatenate([y, np.ones(n % 2)])
    else:
        x, y = O.gen_normal(n, seed=8)
    x[::53] = 0.0
    y[5::71] = 0.0
    ref = O.qdot(x, y, eps, "none", 52, strategy, members=True)
    rep = Q.qdot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), Q.ToleranceConfig(eps),
                 strategy=Q.parse_strategy(strategy))
    members_equal(rep, ref, x, y)


def test_indices_norm_mode_and_host_inputs():
    x, _ = O.gen_normal((1 << 22) + 9, seed=2)          # host input above PIPELINE_MIN: streamed
    x[::1000] = 0.0
    ref = O.qdot(x, x, 1e-6, "none", 52, "ranged:3", members=True)
    rep = Q.qdot(x, x, Q.ToleranceConfig(1e-6), strategy=Q.RangedBinning(3))
    members_equal(rep, ref, x, x)


def test_indices_detect_in_place_modification():
    x, y = O.gen_normal(5000, seed=3)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    rep = Q.qdot(xd, yd, Q.ToleranceConfig(1e-6))
    xd.mul_(2.0)
    with pytest.raises(RuntimeError):
        rep.params.bins[0].indices


def test_bin_order_c_abi_want_mask_and_empty():
    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    # n == 0: all slots empty
    nbytes = int(lib.qdot_b200_order_scratch_bytes(0, 3))
    scratch = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
    starts = torch.full((5,), -1, dtype=torch.int64, device="cuda")
    lut = torch.zeros(_lib.KEYS, dtype=torch.int32, device="cuda")
    _lib.check(lib.qdot_b200_bin_order(None, None, 0, 0, lut.data_ptr(), 3, None, starts.data_ptr(), None,
                                       scratch.data_ptr(), nbytes, s), lib)
    assert starts.tolist() == [0, 0, 0, 0, 0]
    # a want mask selects slots; unwanted slots are empty
    x, y = O.gen_normal(50000, seed=4)
    x[::7] = 0.0
    rep = Q.qdot(x, y, Q.ToleranceConfig(1e-8))
    nb = len(rep.params.bins)
    lut_h = np.full(_lib.KEYS, -1, dtype=np.int32)
    for i, b in enumerate(rep.params.bins):
        lut_h[b.first_key:b.last_key + 1] = i
    want = np.zeros(nb + 1, dtype=np.uint8)
    want[0] = 1
    want[1 + nb // 2] = 1
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    nbytes = int(lib.qdot_b200_order_scratch_bytes(x.size, nb))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    starts = torch.empty(nb + 2, dtype=torch.int64, device="cuda")
    order = torch.full((x.size,), -1, dtype=torch.int64, device="cuda")
    lut_d = torch.from_numpy(lut_h).cuda()
    want_d = torch.from_numpy(want).cuda()
    _lib.check(lib.qdot_b200_bin_order(xd.data_ptr(), yd.data_ptr(), x.size, 0, lut_d.data_ptr(), nb,
                                       want_d.data_ptr(), starts.data_ptr(), order.data_ptr(), scratch.data_ptr(),
                                       nbytes, s), lib)
    st = starts.cpu().numpy()
    od = order.cpu().numpy()
    z = np.flatnonzero((x == 0) | (y == 0))
    mid = rep.params.bins[nb // 2].indices
    assert st[0] == 0 and st[1] == z.size
    assert np.all(st[2:2 + nb // 2] == z.size)
    assert st[2 + nb // 2] == z.size + mid.size and st[-1] == z.size + mid.size
    assert np.array_equal(od[:z.size], z) and np.array_equal(od[z.size:z.size + mid.size], mid)
    assert np.all(od[z.size + mid.size:] == -1)


def half_inputs(n, seed=21):
    rng = np.random.default_rng(seed)
    return np.abs(rng.standard_normal(n)), np.abs(rng.standard_normal(n))


@pytest.mark.parametrize("strategy", ["exact", "ranged:4", "split:3"])
@pytest.mark.parametrize("split", ["none", "per-bin"])
@pytest.mark.parametrize("n", [1 << 18, (1 << 20) + 77])
def test_half_order_sensitive_bins_are_replayed(strategy, split, n):
    x, y = half_inputs(n)
    x[::9] *= -1.0                                     # some cancellation inside the chains
    ref = O.qdot(x, y, 2.0**10, split, 52, strategy)
    rep = Q.qdot(x, y, Q.ToleranceConfig(2.0**10, Q.SplitMode(split)), strategy=Q.parse_strategy(strategy))
    assert rep.half_order_sensitive and rep.half_ordered
    assert [(b.lower, b.upper, b.cardinality, b.precision.code) for b in rep.params.bins] == \
        [(b.lower, b.upper, b.cardinality, b.precision) for b in ref.bins]
    for b, w in zip(rep.params.bins, ref.bins):
        assert b.value == w.value, (b.lower, b.upper, b.value, w.value)
    assert rep.value == ref.value


def test_half_order_norm_mode_and_batched_rows():
    x, _ = half_inputs(1 << 17, seed=5)
    ref = O.qdot(x, x, 2.0**8, "none", 52, "exact")
    rep = Q.qdot(x, x, Q.ToleranceConfig(2.0**8))
    assert rep.half_ordered and rep.value == ref.value
    X = np.stack([half_inputs(1 << 14, seed=s)[0] for s in range(4)])
    Y = np.stack([half_inputs(1 << 14, seed=s)[1] for s in range(4)])
    b = Q.qdot_batched(X, Y, Q.ToleranceConfig(2.0**10))
    for r in range(4):
        assert b.values[r] == O.qdot(X[r], Y[r], 2.0**10).value, r


@pytest.mark.parametrize("ranks", [2, 3])
def test_half_chain_across_emulated_shards(ranks):
    """Contiguous shards chain their fp32 sums in rank order (what
    dist.qdot_sharded does over the process group): the same value as one device."""
    from paper_2105_00115_b200.dist import shard_bounds
    from paper_2105_00115_b200.device import ThreadState, config_struct
    lib = _lib.load()
    n = (1 << 19) + 3
    x, y = half_inputs(n, seed=9)
    cfg = Q.ToleranceConfig(2.0**10)
    want = O.qdot(x, y, 2.0**10).value
    dev = torch.device("cuda", torch.cuda.current_device())
    xd, yd = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    s = torch.cuda.current_stream().cuda_stream
    c = config_struct(cfg, Q.ExactBinning())
    parts = [shard_bounds(n, r, ranks) for r in range(ranks)]
    sts = [ThreadState(dev) for _ in range(ranks)]
    for st, (a, b) in zip(sts, parts):
        _lib.check(lib.qdot_b200_begin(st.ws_ptr, s))
        _lib.check(lib.qdot_b200_pass1(xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, ctypes.byref(c), n,
                                       st.ws_ptr, s))
    ra = sum(st.region_a() for st in sts)
    for st in sts:
        st.region_a().copy_(ra)
    for st, (a, b) in zip(sts, parts):
        _lib.check(lib.qdot_b200_score(st.ws_ptr, n, ctypes.byref(c), s))
        _lib.check(lib.qdot_b200_pass2(xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, st.ws_ptr, s))
    rb = sum(st.region_b() for st in sts)
    for st in sts:
        st.region_b().copy_(rb)
        _lib.check(lib.qdot_b200_finalize(st.ws_ptr, s))
        _lib.check(lib.qdot_b200_fetch(st.ws_ptr, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, s))
    assert sts[0].result.half_order_sensitive == 1
    nb = sts[0].result.n_bins
    chain = torch.zeros(nb, dtype=torch.float32, device=dev)
    keep = []
    for st, (a, b) in zip(sts, parts):                # rank order: each continues the previous chain
        nbytes = int(lib.qdot_b200_order_scratch_bytes(b - a, nb))
        scr = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        order = torch.empty(b - a, dtype=torch.int64, device=dev)
        mine = torch.empty(nb, dtype=torch.float32, device=dev)
        keep.append((scr, nbytes, order, mine))
        args = (xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, st.ws_ptr, nb, order.data_ptr(), b - a,
                mine.data_ptr(), scr.data_ptr(), nbytes)
        _lib.check(lib.qdot_b200_half_ordered(*args, 1, s), lib)
        mine.copy_(chain)                              # "recv" from the previous rank
        _lib.check(lib.qdot_b200_half_ordered(*args, 2, s), lib)
        chain = mine.clone()                           # "send" to the next rank
    for st, (a, b), (scr, nbytes, order, mine) in zip(sts, parts, keep):
        mine.copy_(chain)                              # the last rank's chain, "broadcast"
        _lib.check(lib.qdot_b200_half_ordered(xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, st.ws_ptr, nb,
                                              order.data_ptr(), b - a, mine.data_ptr(), scr.data_ptr(), nbytes,
                                              4, s), lib)
        _lib.check(lib.qdot_b200_fetch(st.ws_ptr, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, s))
        assert st.result.half_order_sensitive == 2
        assert st.result.value == want


def _sharded_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    from paper_2105_00115_b200.dist import qdot_sharded, shard_bounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = (1 << 19) + 3
        x, y = half_inputs(n, seed=9)
        lo, hi = shard_bounds(n, rank, world)
        rep = qdot_sharded(torch.from_numpy(x[lo:hi]).cuda(), torch.from_numpy(y[lo:hi]).cuda(),
                           Q.ToleranceConfig(2.0**10))
        q.put((rank, rep.value, rep.half_ordered))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_qdot_sharded_half_chain_gloo_processes(world):
    """dist.qdot_sharded with ranks as real processes (gloo, all on cuda:0): the
    HALF fp32 chains pass rank to rank and every rank reports the reference value."""
    import socket
    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = (1 << 19) + 3
    x, y = half_inputs(n, seed=9)
    want = O.qdot(x, y, 2.0**10).value
    assert all(v == want and h for _, v, h in out), (out, want)
