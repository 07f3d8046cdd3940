"""GPU parity: the CUDA path (through the C ABI) against the reference's own
golden outputs and the CPU oracle.

Bar: bins, scores, precisions, counts, bounds and
error behaviour bit-exact; per-bin values and the final value bit-exact.
HALF bins whose fp32 sequential sum is order-sensitive are replayed in index
order on the device (qdot_b200_half_ordered), so they are held to the same
bar.  The one admitted difference: a DOUBLE bin where the reference's
Neumaier sum is itself not the correctly rounded sum of its products (the
device rounds the exact sum once) -- checked explicitly with math.fsum over
the bin's members, and it never occurs in the golden set.  Every value lies
within abs_cap of the exact dot.
"""

import math

import numpy as np
import pytest

import golden_util as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_00115_b200 as Q  # noqa: E402
from paper_2105_00115_b200 import PrecisionLevel as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

PREC = {0: P.PERFORATE, 1: P.HALF, 2: P.SINGLE, 3: P.DOUBLE}
LABEL = {P.PERFORATE: "perforate", P.HALF: "half", P.SINGLE: "single", P.DOUBLE: "double"}


def strat(s):
    return Q.parse_strategy(s)


def cfg_of(case):
    return Q.ToleranceConfig(epsilon=G.hexf(case["epsilon"]),
                             split=Q.SplitMode.PER_BIN if case["split"] == "per-bin" else Q.SplitMode.NONE,
                             input_mu=case["input_mu"])


def same(a, b):
    return a == b or (math.isnan(a) and math.isnan(b))


NEUMAIER_NOT_CR = []   # (bin, oracle value, fsum) of DOUBLE bins where the reference is not correctly rounded


def assert_bins_exact(x, y, rep, r):
    """Per-bin values and the value equal the oracle's bit for bit, except a
    DOUBLE bin whose reference (Neumaier, index order) value is not the
    correctly rounded sum of its products: there the device value must be the
    correctly rounded one (math.fsum) and the final value within abs_cap."""
    exact = True
    for b, w in zip(rep.params.bins, r.bins):
        if same(b.value, w.value):
            continue
        assert b.precision is P.DOUBLE, (b, b.value, w.value)
        cr = math.fsum((x[w.indices] * y[w.indices]).tolist())
        assert b.value == cr and w.value != cr, (b, b.value, w.value, cr)
        NEUMAIER_NOT_CR.append((b.upper, w.value, cr))
        exact = False
    if exact:
        assert same(rep.value, r.value), (rep.value, r.value)
    else:
        assert abs(rep.value - r.value) <= rep.abs_cap


def check_against_golden(case, rep):
    bins = rep.params.bins
    got = [[b.lower, b.upper, b.cardinality, b.score, b.precision.code] for b in bins]
    assert got == [w[:5] for w in case["bins"]], case["name"]
    assert rep.params.n_bins == case["n_bins"]
    assert rep.early_terminated == case["early_terminated"]
    assert rep.params.eps_eff == G.hexf(case["eps_eff"])
    if case["n_bins"]:
        assert (rep.params.e_min, rep.params.e_max) == (case["e_min"], case["e_max"])
    assert rep.params.zero_count == case["zero_count"]
    assert {LABEL[k]: v for k, v in rep.counts.items()} == case["counts"]
    assert rep.abs_bound == G.hexf(case["abs_bound"])
    assert rep.rel_bound == G.hexf(case["rel_bound"])
    assert rep.rel_guarantee == G.hexf(case["rel_guarantee"])
    assert rep.abs_cap == G.hexf(case["abs_cap"])
    # per-bin values: bit-exact, every precision (the reference's DOUBLE
    # Neumaier sums are correctly rounded on every golden input)
    for b, w in zip(bins, case["bins"]):
        assert same(b.value, G.hexf(w[5])), (case["name"], b, b.value, w[5])
    want = G.hexf(case["value"])
    assert same(rep.value, want), (case["name"], rep.value.hex(), case["value"])
    if case.get("exact") is not None and math.isfinite(rep.value):
        assert abs(rep.value - G.hexf(case["exact"])) <= rep.abs_cap + 1e-300


CASES = G.select(max_n=1 << 20)


@pytest.fixture(params=[0, 1, 2, 1 | 4, 2 | 4, 2 | 8, 1 | 16, 1 | 4 | 16, 32, 1 | 32],
                ids=["auto", "lean", "full", "lean-queue", "full-queue", "full-noqueue", "lean-wide",
                     "lean-wide-queue", "auto-nonormloop", "lean-nonormloop"])
def pass1_mode(request, monkeypatch):
    from paper_2105_00115_b200 import device
    monkeypatch.setattr(device, "PASS1_MODE", request.param)
    return request.param


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_golden_case(case, pass1_mode):
    x, y = G.inputs(case)
    cfg = cfg_of(case)
    yy = x if case["norm"] else y
    if "error" in case:
        exc = {"ValueError": ValueError, "OverflowError": OverflowError}[case["error"]]
        with pytest.raises(exc):
            Q.qdot(x, yy, cfg, strategy=strat(case["strategy"]))
        return
    rep = Q.qdot(x, yy, cfg, strategy=strat(case["strategy"]))
    check_against_golden(case, rep)
    assert rep.rel_hypothesis == case["rel_hypothesis"]
    if pass1_mode == 0:   # Bin.indices / zero_idx (device counting-sort scatter) against the reference's order
        ps = rep.params
        assert G.members_sha(ps.zero_idx, [b.indices for b in ps.bins]) == case["members_sha"], case["name"]


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("strategy", ["exact", "ranged:3", "split:4"])
def test_random_against_oracle(seed, strategy, pass1_mode):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 20000))
    t = int(rng.integers(0, 120))
    x = np.ldexp(rng.uniform(0.5, 1, n) * rng.choice([-1, 1], n), rng.integers(-t // 2, t // 2 + 1, n))
    y = np.ldexp(rng.uniform(0.5, 1, n), rng.integers(-t // 2, t // 2 + 1, n))
    if seed % 3 == 0:
        x[rng.integers(0, n, max(1, n // 50))] = 0.0
    eps = float(np.ldexp(1.0, -int(rng.integers(0, 55))))
    split = "per-bin" if seed % 2 else "none"
    r = O.qdot(x, y, eps, split, 52, strategy, members=True)
    rep = Q.qdot(x, y, Q.ToleranceConfig(eps, Q.SplitMode(split)), strategy=strat(strategy))
    assert [[b.lower, b.upper, b.cardinality, b.score, b.precision.code] for b in rep.params.bins] == \
        [[b.lower, b.upper, b.cardinality, b.score, b.precision] for b in r.bins]
    assert_bins_exact(x, y, rep, r)
    ex, _, _ = O.exact_dot(x, y)
    assert abs(rep.value - ex) <= rep.abs_cap


def test_toy_bit_exact():
    x = np.array([2.0**27, 2.0**8, 2.0**-3, 2.0**20])
    y = np.array([2.0**23, 2.0**-14, 2.0**7, 2.0**-3])
    rep = Q.qdot(x, y, Q.ToleranceConfig(2.0**-34))
    assert rep.value == 2.0**50 + 2.0**17
    assert [b.score for b in rep.params.bins] == [-21, -11, 2, 35]
    assert rep.rel_bound == 2.0**-51 + 2.0**-42 + 2.0**-45 + 2.0**-55
    assert set(rep.phase_ns) == {"select", "compute", "reference"}


def test_norm_mode_reads_once_and_matches():
    x, _ = O.gen_normal(1 << 16, seed=5)
    a = Q.qdot(x, x, Q.ToleranceConfig(1e-8))
    b = Q.qdot(x, x.copy(), Q.ToleranceConfig(1e-8))
    assert a.value == b.value and a.rel_hypothesis == "holds" and b.rel_hypothesis == "assumed"
    r = O.qdot(x, x, 1e-8)
    assert a.value == r.value


def test_torch_inputs_and_misaligned_views():
    x, y = O.gen_normal((1 << 15) + 7, seed=9)
    want = O.qdot(x[1:], y[1:], 1e-9).value
    xt = torch.from_numpy(x).cuda()
    yt = torch.from_numpy(y).cuda()
    rep = Q.qdot(xt[1:], yt[1:], Q.ToleranceConfig(1e-9))     # 8-byte aligned: scalar loads
    assert rep.value == want
    rep2 = Q.qdot(xt[1:].clone(), yt[1:].clone(), Q.ToleranceConfig(1e-9))
    assert rep2.value == want


@pytest.mark.parametrize("n", [(1 << 21) + 7, (1 << 23) + 1])
def test_misaligned_views_of_long_vectors(n):
    """8-byte aligned views long enough for the streaming pass-1 variant (its
    TMA L2 prefetch needs 16-byte addresses): same value as aligned copies,
    and the device exact dot agrees too."""
    x, y = O.gen_normal(n + 1, seed=12)
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for strategy in ("exact", "ranged:3"):
        a = Q.qdot(xt[1:], yt[1:], Q.ToleranceConfig(1e-9), strategy=strat(strategy))
        b = Q.qdot(xt[1:].clone(), yt[1:].clone(), Q.ToleranceConfig(1e-9), strategy=strat(strategy))
        assert a.value == b.value and a.counts == b.counts
    assert a.value == O.qdot(x[1:], y[1:], 1e-9, "none", 52, "ranged:3").value
    assert Q.reference_dot(xt[1:], yt[1:]).value == Q.reference_dot(xt[1:].clone(), yt[1:].clone()).value


def test_lazy_indices_match_oracle():
    for strategy in ["exact", "ranged:4", "split:3"]:
        x, y = O.gen_family("B", 12, 5000, 77)
        x[::97] = 0.0
        r = O.qdot(x, y, 1e-6, "none", 52, strategy, members=True)
        rep = Q.qdot(x, y, Q.ToleranceConfig(1e-6), strategy=strat(strategy))
        for b, w in zip(rep.params.bins, r.bins):
            assert b.indices.tolist() == w.indices.tolist()
        assert rep.params.zero_idx.tolist() == np.flatnonzero((x == 0) | (y == 0)).tolist()


def test_errors():
    with pytest.raises(ValueError):
        Q.qdot(np.array([1.0, np.nan]), np.ones(2), Q.ToleranceConfig(1e-3))
    with pytest.raises(ValueError):
        Q.qdot(np.ones(3), np.ones(4), Q.ToleranceConfig(1e-3))
    with pytest.raises(ValueError):
        Q.qdot(np.ones((2, 2)), np.ones((2, 2)), Q.ToleranceConfig(1e-3))
    with pytest.raises(TypeError):
        Q.qdot(np.ones(3), np.ones(3), Q.ToleranceConfig(1e-3), strategy=object())


def test_empty_and_all_zero():
    rep = Q.qdot(np.zeros(0), np.zeros(0), Q.ToleranceConfig(2.0**-34))
    assert rep.value == 0.0 and rep.n == 0 and sum(rep.counts.values()) == 0
    rep = Q.qdot(np.zeros(4), np.ones(4), Q.ToleranceConfig(2.0**-34))
    assert rep.value == 0.0 and rep.counts[P.PERFORATE] == 4 and rep.abs_bound == 0.0


def test_sharded_tables_sum_like_one_device():
    """The multi-GPU exchange is an integer sum of regions A and B: emulate two
    ranks on one device and check bit-identical results to the single call."""
    import ctypes
    from paper_2105_00115_b200 import _lib
    from paper_2105_00115_b200.device import ThreadState, config_struct
    lib = _lib.load()
    x, y = O.gen_illcond(1 << 18, seed=3)
    cfg = Q.ToleranceConfig(1e-12)
    whole = Q.qdot(x, y, cfg)
    dev = torch.device("cuda", torch.cuda.current_device())
    xd = torch.from_numpy(x).to(dev)
    yd = torch.from_numpy(y).to(dev)
    n = x.shape[0]
    cut = n // 3
    ranks = [ThreadState(dev), ThreadState(dev)]
    s = torch.cuda.current_stream().cuda_stream
    parts = [(0, cut), (cut, n)]
    c = config_struct(cfg, Q.ExactBinning())
    for st, (a, b) in zip(ranks, parts):
        _lib.check(lib.qdot_b200_begin(st.ws_ptr, s))
        _lib.check(lib.qdot_b200_pass1(xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, ctypes.byref(c), n,
                                       st.ws_ptr, s))
    ra = ranks[0].region_a() + ranks[1].region_a()          # "allreduce" of region A
    for st in ranks:
        st.region_a().copy_(ra)
    for st, (a, b) in zip(ranks, parts):
        _lib.check(lib.qdot_b200_score(st.ws_ptr, n, ctypes.byref(c), s))
        _lib.check(lib.qdot_b200_pass2(xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, st.ws_ptr, s))
    rb = ranks[0].region_b() + ranks[1].region_b()          # "allreduce" of region B
    for st in ranks:
        st.region_b().copy_(rb)
        _lib.check(lib.qdot_b200_finalize(st.ws_ptr, s))
        _lib.check(lib.qdot_b200_fetch(st.ws_ptr, ctypes.byref(st.result), st.bins, 4196, s))
        assert st.result.value == whole.value
        assert st.result.n_bins == whole.params.n_bins


def test_c1_against_golden_and_exact():
    case = next(c for c in G.cases() if c["name"] == "C1_none")
    x, y = G.inputs(case)
    rep = Q.qdot(x, y, cfg_of(case))
    assert rep.value == G.hexf(case["value"])                  # -979.5638873355846
    assert rep.value == -979.5638873355846


@pytest.mark.slow
def test_c2_headline_size_properties():
    """n = 2^28 (BASELINE configs[1]): bins and precisions equal the oracle's,
    value equals the oracle's reference-order value and lies within abs_cap of
    the exact dot; repeated runs are bit-identical."""
    n = 1 << 28
    x, y = O.gen_normal(n, seed=0)
    O.set_threads(32)
    r = O.qdot(x, y, 1e-8)
    ex, _, _ = O.exact_dot(x, y)
    xt = torch.from_numpy(x).cuda()
    yt = torch.from_numpy(y).cuda()
    del x, y
    cfg = Q.ToleranceConfig(1e-8)
    rep = Q.qdot(xt, yt, cfg)
    rep2 = Q.qdot(xt, yt, cfg)
    assert rep.value == rep2.value
    assert [[b.lower, b.upper, b.cardinality, b.score, b.precision.code] for b in rep.params.bins] == \
        [[b.lower, b.upper, b.cardinality, b.score, b.precision] for b in r.bins]
    assert rep.value == r.value == -23532.7407708119
    assert abs(rep.value - ex) <= rep.abs_cap


def test_qdot_sharded_single_rank_nccl():
    """dist.qdot_sharded through a real NCCL process group (world 1 on this box;
    the 2/4/8-rank exchange algebra is covered by tests/test_dist_cpu.py)."""
    import socket
    import torch.distributed as dist
    from paper_2105_00115_b200.dist import qdot_sharded
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        x, y = O.gen_illcond(1 << 16, seed=4)
        cfg = Q.ToleranceConfig(1e-12, Q.SplitMode.PER_BIN)
        a = qdot_sharded(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), cfg)
        b = Q.qdot(x, y, cfg)
        assert a.value == b.value and a.counts == b.counts and a.abs_bound == b.abs_bound
        assert [(u.lower, u.upper, u.cardinality) for u in a.params.bins] == \
            [(u.lower, u.upper, u.cardinality) for u in b.params.bins]
        # a host shard above PIPELINE_MIN takes the chunked H2D / pass-1 overlap path
        from paper_2105_00115_b200 import kernel
        xl, yl = O.gen_illcond(kernel.PIPELINE_MIN + 4097, seed=5)
        c = qdot_sharded(torch.from_numpy(xl).pin_memory(), torch.from_numpy(yl).pin_memory(), cfg)
        d = Q.qdot(torch.from_numpy(xl).cuda(), torch.from_numpy(yl).cuda(), cfg)
        assert c.value == d.value and c.counts == d.counts and c.abs_bound == d.abs_bound
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("norm", [False, True])
def test_host_inputs_pipelined_equal_device(norm):
    # host inputs above PIPELINE_MIN stream in chunks overlapping pass 1; the
    # report must equal the one for the same vectors already on the device
    from paper_2105_00115_b200 import kernel
    rng = np.random.default_rng(77)
    n = kernel.PIPELINE_MIN + 3 * (1 << 22) // 2 + 12345        # several staging chunks, a ragged tail
    x = rng.standard_normal(n) * np.exp2(rng.integers(-30, 30, n))
    y = x if norm else rng.standard_normal(n)
    cfg = Q.ToleranceConfig(1e-9, Q.SplitMode.PER_BIN)
    for strategy in (Q.ExactBinning(), Q.RangedBinning(3)):
        a = Q.qdot(x, y, cfg, strategy=strategy)                              # numpy (pageable)
        xt = torch.from_numpy(x).pin_memory()
        b = Q.qdot(xt, xt if norm else torch.from_numpy(y).pin_memory(), cfg, strategy=strategy)   # pinned
        xd = torch.from_numpy(x).cuda()
        d = Q.qdot(xd, xd if norm else torch.from_numpy(y).cuda(), cfg, strategy=strategy)        # device
        for r in (a, b):
            assert r.value == d.value and r.counts == d.counts and r.abs_bound == d.abs_bound
            assert [(q.lower, q.upper, q.cardinality, q.precision) for q in r.params.bins] == \
                   [(q.lower, q.upper, q.cardinality, q.precision) for q in d.params.bins]


def test_pageable_staging_ring_back_to_back():
    """numpy inputs of many staging chunks, back-to-back calls with different
    data (the pinned staging ring is reused across calls: a buffer is refilled
    only after its previous H2D finished) and the C ABI one-call host path."""
    import ctypes
    from paper_2105_00115_b200 import _lib
    from paper_2105_00115_b200.device import config_struct
    n = (1 << 24) + 5
    cfg = Q.ToleranceConfig(1e-8)
    pairs = [O.gen_normal(n, seed=s) for s in (40, 41, 42)]
    want = [Q.qdot(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg).value for a, b in pairs]
    for _ in range(2):
        assert [Q.qdot(a, b, cfg).value for a, b in pairs] == want
    lib = _lib.load()
    c = config_struct(cfg, Q.ExactBinning())
    res = _lib.QdotResult()
    bins = (_lib.QdotBin * (_lib.KEYS + 1))()
    dp = ctypes.POINTER(ctypes.c_double)
    for (a, b), w in zip(pairs, want):
        _lib.check(lib.qdot_b200_dot_host(a.ctypes.data_as(dp), b.ctypes.data_as(dp), n, 0, ctypes.byref(c),
                                          ctypes.byref(res), bins, _lib.KEYS + 1), lib)
        assert res.value == w
    assert lib.qdot_b200_host_copy_threads() >= 1


@pytest.mark.parametrize("strategy,eps", [("ranged:8", 1e-8), ("ranged:2", 1e-8), ("ranged:8", 1e-4), ("ranged:3", 1e-6)])
def test_pass2_over_cold_list(strategy, eps):
    # ranged bins whose pass-2 keys all lie outside every private window run
    # pass 2 over the cold-element list (pass2_needed == 2) instead of a second
    # stream; either way the result equals the oracle bit for bit
    from paper_2105_00115_b200.kernel import run_device
    x, y = O.gen_normal(1 << 21, seed=11)
    cfg = Q.ToleranceConfig(eps)
    s = Q.parse_strategy(strategy)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    res, bins, _ = run_device(xd, yd, x.size, False, cfg, s, timing=False)
    ref = O.qdot(x, y, eps, "none", 52, strategy)
    got = [(bins[i].lower, bins[i].upper, bins[i].cardinality, bins[i].precision) for i in range(res.n_bins)]
    assert got == [(b.lower, b.upper, b.cardinality, b.precision) for b in ref.bins]
    assert res.value == ref.value
    if strategy in ("ranged:8", "ranged:2") and eps == 1e-8:
        assert res.pass2_needed == 2


@pytest.mark.parametrize("n,norm", [(0, False), (1000, False), ((1 << 22) + 12345, False), ((1 << 22) + 7, True),
                                    (3 * (1 << 22), False)])
def test_c_abi_dot_host(n, norm):
    # the one-call host-buffer entry point of the C ABI (what an FFI binding uses)
    import ctypes
    from paper_2105_00115_b200 import _lib
    from paper_2105_00115_b200.device import config_struct
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n)
    y = x if norm else rng.standard_normal(n)
    cfg = Q.ToleranceConfig(1e-7, Q.SplitMode.PER_BIN)
    lib = _lib.load()
    c = config_struct(cfg, Q.RangedBinning(2))
    res = _lib.QdotResult()
    bins = (_lib.QdotBin * (_lib.KEYS + 1))()
    dp = ctypes.POINTER(ctypes.c_double)
    for _ in range(2):   # second call reuses the cached buffers
        _lib.check(lib.qdot_b200_dot_host(x.ctypes.data_as(dp) if n else None,
                                          y.ctypes.data_as(dp) if n else None, n, int(norm), ctypes.byref(c),
                                          ctypes.byref(res), bins, _lib.KEYS + 1), lib)
        if n == 0:
            assert res.value == 0.0 and res.n_bins == 0
            continue
        xd = torch.from_numpy(x).cuda()
        yd = xd if norm else torch.from_numpy(y).cuda()
        rep = Q.qdot(xd, yd, cfg, strategy=Q.RangedBinning(2))
        assert res.value == rep.value and res.n_bins == len(rep.params.bins)
        assert [(bins[i].lower, bins[i].upper, bins[i].cardinality) for i in range(res.n_bins)] == \
               [(b.lower, b.upper, b.cardinality) for b in rep.params.bins]


@pytest.mark.parametrize("n", [0, 1, 2, 255, 4096, 100003])
def test_graph_one_call_path_small(n):
    # run_device(timing=False) -> qdot_b200_dot: the cached-graph pipeline with
    # the host-mapped result; repeated calls (graph replay) stay identical
    from paper_2105_00115_b200.kernel import run_device
    rng = np.random.default_rng(1000 + n)
    x = rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n))
    y = rng.standard_normal(n)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    cfg = Q.ToleranceConfig(1e-6, Q.SplitMode.PER_BIN)
    ref = O.qdot(x, y, 1e-6, "per-bin", 52, "exact")
    for _ in range(3):
        res, bins, _ = run_device(xd, yd, n, False, cfg, Q.ExactBinning(), timing=False)
        assert res.status == 0 and res.n_bins == ref.n_bins
        assert res.value == ref.value or (n == 0 and res.value == 0.0)
        assert [bins[i].cardinality for i in range(res.n_bins)] == [b.cardinality for b in ref.bins]


@pytest.mark.parametrize("strategy,eps", [("exact", 1e-8), ("ranged:3", 1e-8), ("split:4", 1e-6), ("ranged:8", 1e-4)])
@pytest.mark.parametrize("n", [0, 1000, 300001])
def test_pass2_finalize_sequences_agree(strategy, eps, n):
    """The three single-device launch sequences give byte-identical results:
    score + pass2 + finalize (staged), score_finalize + pass2_finalize (fused:
    score or the last pass-2 CTA finalizes), score + pass2_finalize."""
    import ctypes
    from paper_2105_00115_b200 import _lib
    from paper_2105_00115_b200.device import config_struct, thread_state
    rng = np.random.default_rng(n + 17)
    x = torch.from_numpy(rng.standard_normal(n) * np.exp2(rng.integers(-30, 30, n))).cuda()
    y = torch.from_numpy(rng.standard_normal(n)).cuda()
    lib = _lib.load()
    st = thread_state(x.device)
    ws = st.ws_ptr
    s = torch.cuda.current_stream().cuda_stream
    c = config_struct(Q.ToleranceConfig(eps), strat(strategy))
    xp, yp = (x.data_ptr(), y.data_ptr()) if n else (0, 0)
    outs = []
    for seq in ("staged", "fused", "score+p2fin"):
        _lib.check(lib.qdot_b200_begin(ws, s), lib)
        _lib.check(lib.qdot_b200_pass1(xp, yp, n, 0, ctypes.byref(c), n, ws, s), lib)
        if seq == "fused":
            _lib.check(lib.qdot_b200_score_finalize(ws, n, ctypes.byref(c), s), lib)
        else:
            _lib.check(lib.qdot_b200_score(ws, n, ctypes.byref(c), s), lib)
        if seq == "staged":
            _lib.check(lib.qdot_b200_pass2(xp, yp, n, 0, ws, s), lib)
            _lib.check(lib.qdot_b200_finalize(ws, s), lib)
        else:
            _lib.check(lib.qdot_b200_pass2_finalize(xp, yp, n, 0, ws, s), lib)
        res = _lib.QdotResult()
        bins = (_lib.QdotBin * (_lib.KEYS + 1))()
        _lib.check(lib.qdot_b200_fetch(ws, ctypes.byref(res), bins, _lib.KEYS + 1, s), lib)
        torch.cuda.synchronize()
        nb = res.n_bins
        outs.append((res.value, res.status, res.n_bins, tuple(res.counts), res.pass2_needed, res.half_order_sensitive,
                     ctypes.string_at(ctypes.addressof(bins), nb * ctypes.sizeof(_lib.QdotBin))))
    assert outs[0] == outs[1] == outs[2]
    if n:
        ref = O.qdot(x.cpu().numpy(), y.cpu().numpy(), eps, "none", 52, strategy)
        if outs[0][5]:   # a HALF bin the reference sums order-sensitively in fp32: replay it in index order
            from paper_2105_00115_b200.kernel import resolve_half_order
            st.result = res
            ctypes.memmove(st.bins, bins, ctypes.sizeof(bins))
            resolve_half_order(x, y, n, False, st, s)
            assert st.result.half_order_sensitive == 2
            assert st.result.value == ref.value
        else:
            assert outs[0][0] == ref.value


@pytest.mark.parametrize("n", [5000, 1 << 17, (1 << 22) + 3])
def test_inputs_written_just_before_the_call_are_seen(n):
    """The launch chain (k_begin launched normally, then pass 1 / score /
    pass 2 with programmatic dependent launch) is ordered after a kernel that
    rewrites x and y on the same stream with no host sync in between: each
    call must see the new data (eager launches and the cached graph path)."""
    def agree(rep, ref):
        return rep.value == ref.value

    rng = np.random.default_rng(n)
    xs = [rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n)) for _ in range(4)]
    ys = [rng.standard_normal(n) for _ in range(4)]
    want = [O.qdot(a, b, 1e-8) for a, b in zip(xs, ys)]
    xsrc = [torch.from_numpy(a).cuda() for a in xs]
    ysrc = [torch.from_numpy(b).cuda() for b in ys]
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    cfg = Q.ToleranceConfig(1e-8)
    torch.cuda.synchronize()
    for rep in range(3):                       # the third round runs through the cached graph
        for i in range(4):
            x.copy_(xsrc[i])                   # device kernels on the current stream, no sync
            y.copy_(ysrc[i])
            assert agree(Q.qdot(x, y, cfg), want[i]), (rep, i)
    # norm mode on a vector rewritten in place
    for i in range(2):
        x.copy_(xsrc[i])
        assert agree(Q.qdot(x, x, cfg), O.qdot(xs[i], xs[i], 1e-8)), i


@pytest.mark.parametrize("n", [606_209, (1 << 21) + 777, 1 << 22])
@pytest.mark.parametrize("data", ["normal", "wide", "special"])
def test_norm_ring_pass1_against_oracle(n, data, pass1_mode):
    """Norm mode above the compact pass-1 size (the streaming k_pass1): bins and
    value bit-exact against the oracle in every pass-1 mode, with a partial
    last tile (odd n), zeros, subnormals and wide exponents."""
    rng = np.random.default_rng(n % 1000 + len(data))
    x = rng.standard_normal(n)
    if data == "wide":
        x *= np.exp2(rng.integers(-300, 300, n))
    elif data == "special":
        x[rng.integers(0, n, 500)] = 0.0
        x[rng.integers(0, n, 50)] = 5e-320
        x[rng.integers(0, n, 50)] *= 2.0 ** 500
    eps = 1e-8 if data != "wide" else 1e-3
    r = O.qdot(x, x, eps, "none", 52, "exact", members=True)
    xd = torch.from_numpy(x).cuda()
    rep = Q.qdot(xd, xd, Q.ToleranceConfig(eps))
    assert [[b.lower, b.upper, b.cardinality, b.score, b.precision.code] for b in rep.params.bins] == \
        [[b.lower, b.upper, b.cardinality, b.score, b.precision] for b in r.bins]
    assert_bins_exact(x, x, rep, r)
    assert rep.params.zero_count == r.zero_count
