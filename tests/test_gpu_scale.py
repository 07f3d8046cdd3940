"""BASELINE configs at their stated sizes and the device
input generator they use.

* generator: shards of every law concatenate to the unsharded vectors
  (any rank count sees the same data), and the laws look like their numpy
  counterparts (moments, exponent ranges, the C3 pair structure).
* C3 (configs[2]) at n = 2^28 with the reference's own ill-conditioned
  generator (oracle.gen_illcond, numpy): bins, precisions and the value equal
  the oracle's bit for bit; with the exact dot passed as `reference` the
  hypothesis reads "violated" and the error lies within abs_cap and within
  rel_bound_e * |exact| (the reference's gate, test_kernel.py:186-189).
* C5 (configs[4]) at n = 2^31 on one B200: the whole vector (32 GiB) and
  G = 2, 4, 8 contiguous shards emulated through the staged C ABI (begin /
  pass 1 per shard -> summed region A -> score -> pass 2 per shard -> summed
  region B -> finalize) give identical bins and value; histogram equals the
  oracle's, value within abs_cap of the device exact dot.
"""

import ctypes
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_00115_b200 as Q  # noqa: E402
from paper_2105_00115_b200 import _lib  # noqa: E402
from paper_2105_00115_b200.generate import device_vectors  # noqa: E402
from oracle import oracle as O  # noqa: E402


@pytest.mark.parametrize("law,param", [("normal", 0), ("illcond", 0), ("A", 40), ("B", 14)])
def test_generator_shards_concatenate(law, param):
    n = 1000003
    x, y = device_vectors(law, n, seed=5, param=param)
    cuts = [0, 1, 77, 500001, 999999, n]
    for a, b in zip(cuts[:-1], cuts[1:]):
        xs, ys = device_vectors(law, b - a, seed=5, offset=a, param=param)
        assert torch.equal(xs, x[a:b]) and torch.equal(ys, y[a:b]), (law, a, b)
    x2, _ = device_vectors(law, n, seed=6, param=param)
    assert not torch.equal(x, x2)


def test_generator_laws():
    n = 1 << 22
    x, y = device_vectors("normal", n, seed=1)
    for v in (x, y):
        assert abs(float(v.mean())) < 5e-3 and abs(float(v.var()) - 1.0) < 5e-3
    assert abs(float(torch.corrcoef(torch.stack([x, y]))[0, 1])) < 5e-3
    x, y = device_vectors("illcond", n, seed=1)
    assert torch.equal(x[0::2], x[1::2])                         # pairs share x1
    r = (y[1::2] / -y[0::2]) - 1.0                               # 1 + delta
    assert float(r.abs().max()) <= 2.0**-25 and float(r.abs().max()) > 2.0**-27
    ex = torch.frexp(x).exponent.cpu().numpy() - 1
    assert ex.max() <= 149 and ex.min() >= 149 - 300 and np.mean(ex >= 140) > 0.9
    xa, _ = device_vectors("A", n, seed=1, param=40)
    ea = torch.frexp(xa).exponent.cpu().numpy() - 1
    assert ea.min() == -21 and ea.max() == 19                    # U[.5,1) 2^U{-20..20}
    xb, _ = device_vectors("B", n, seed=1, param=14)
    eb = (torch.frexp(xb).exponent - 1).double()
    assert abs(float(eb.std()) - 7.0) < 0.1


def bins_digest(bins):
    h = hashlib.sha256()
    for b in bins:
        h.update(np.array([b[0], b[1], b[2], b[3], b[4]], dtype=np.int64).tobytes())
    return h.hexdigest()[:16]


def staged_sharded(xd, yd, n, cfg, strategy, world):
    """G emulated ranks on one device through the staged C ABI; region A and
    B 'allreduces' are sums of the G workspaces' regions."""
    from paper_2105_00115_b200.device import ThreadState, config_struct
    from paper_2105_00115_b200.dist import shard_bounds
    lib = _lib.load()
    dev = xd.device
    s = torch.cuda.current_stream().cuda_stream
    c = config_struct(cfg, strategy)
    parts = [shard_bounds(n, r, world) for r in range(world)]
    sts = [ThreadState(dev) for _ in range(world)]
    for st, (a, b) in zip(sts, parts):
        _lib.check(lib.qdot_b200_begin(st.ws_ptr, s), lib)
        _lib.check(lib.qdot_b200_pass1(xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, ctypes.byref(c), n,
                                       st.ws_ptr, s), lib)
    ra = sum(st.region_a() for st in sts)
    for st in sts:
        st.region_a().copy_(ra)
    for st, (a, b) in zip(sts, parts):
        _lib.check(lib.qdot_b200_score(st.ws_ptr, n, ctypes.byref(c), s), lib)
        _lib.check(lib.qdot_b200_pass2(xd[a:].data_ptr(), yd[a:].data_ptr(), b - a, 0, st.ws_ptr, s), lib)
    rb = sum(st.region_b() for st in sts)
    out = []
    for st in sts:
        st.region_b().copy_(rb)
        _lib.check(lib.qdot_b200_finalize(st.ws_ptr, s), lib)
        _lib.check(lib.qdot_b200_fetch(st.ws_ptr, ctypes.byref(st.result), st.bins, _lib.KEYS + 1, s), lib)
        nb = st.result.n_bins
        rows = [(st.bins[i].lower, st.bins[i].upper, st.bins[i].cardinality, st.bins[i].score,
                 st.bins[i].precision) for i in range(nb)]
        out.append((st.result.value, bins_digest(rows), tuple(st.result.counts)))
    del sts
    return out


@pytest.mark.parametrize("law,eps,strategy", [("normal", 1e-8, "exact"), ("illcond", 1e-12, "exact"),
                                              ("illcond", 1e-12, "ranged:8"), ("normal", 1e-6, "split:5")])
def test_sharded_equals_whole_device_generated(law, eps, strategy):
    n = (1 << 22) + 13
    xd, yd = device_vectors(law, n, seed=3)
    cfg = Q.ToleranceConfig(eps)
    st = Q.parse_strategy(strategy)
    whole = Q.qdot(xd, yd, cfg, strategy=st)
    ref = O.qdot(xd.cpu().numpy(), yd.cpu().numpy(), eps, "none", 52, strategy)
    assert whole.value == ref.value
    wd = bins_digest([(b.lower, b.upper, b.cardinality, b.score, b.precision.code) for b in whole.params.bins])
    for world in (2, 3, 8):
        for v, d, _ in staged_sharded(xd, yd, n, cfg, st, world):
            assert v == whole.value and d == wd, (world, v, whole.value)


@pytest.mark.slow
def test_c3_2e28_against_oracle_and_exact():
    n = 1 << 28
    x, y = O.gen_illcond(n, seed=0)
    O.set_threads(32)
    r = O.qdot(x, y, 1e-12)
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    ex = Q.reference_dot(xt, yt, plain=False)
    assert ex.value == O.exact_dot(x, y)[0]
    del x, y
    rep = Q.qdot(xt, yt, Q.ToleranceConfig(1e-12), reference=ex)
    assert [[b.lower, b.upper, b.cardinality, b.score, b.precision.code] for b in rep.params.bins] == \
        [[b.lower, b.upper, b.cardinality, b.score, b.precision] for b in r.bins]
    assert rep.value == r.value
    assert rep.rel_hypothesis == "violated"                      # cond ~1e12: e_max > flexp(exact)
    assert abs(rep.value - ex.value) <= rep.abs_cap
    assert abs(rep.value - ex.value) <= rep.rel_bound_e * abs(ex.value)
    assert rep.n == n and rep.params.n_bins > 300


@pytest.mark.slow
def test_c5_2e31_sharded_identical_for_every_world_size():
    n = 1 << 31
    xd, yd = device_vectors("normal", n, seed=0)               # 32 GiB on one B200
    cfg = Q.ToleranceConfig(1e-8)
    whole = Q.qdot(xd, yd, cfg)
    wd = bins_digest([(b.lower, b.upper, b.cardinality, b.score, b.precision.code) for b in whole.params.bins])
    # histogram of the whole vector = the oracle's (bins follow from it), in 2^27 slices on the host
    tot = np.zeros(_lib.KEYS, dtype=np.int64)
    zc = 0
    O.set_threads(32)
    step = 1 << 27
    for a in range(0, n, step):
        h, z = O.hist(xd[a:a + step].cpu().numpy(), yd[a:a + step].cpu().numpy())
        tot += h
        zc += z
    assert [(b.upper, b.cardinality) for b in whole.params.bins] == \
        [(k - _lib.KEY_OFFSET, int(c)) for k, c in enumerate(tot) if c]
    ex = Q.reference_dot(xd, yd, plain=False)
    assert abs(whole.value - ex.value) <= whole.abs_cap
    for world in (2, 4, 8):
        for v, d, cnt in staged_sharded(xd, yd, n, cfg, Q.ExactBinning(), world):
            assert v == whole.value and d == wd, (world, v, whole.value)
