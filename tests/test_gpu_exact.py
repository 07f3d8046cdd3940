"""Device exact dot (kernel.reference_dot on the GPU) against the reference.

Golden results come from running the reference's reference_dot
(tests/golden/make_exact_golden.py, exact_golden.json; plus the `exact`
field of every qdot golden case): value, flexp_e and plain must be
bit-identical, and the exception type must match."""

import math
from fractions import Fraction

import numpy as np
import pytest

import golden_util as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import json  # noqa: E402
import os  # noqa: E402

import paper_2105_00115_b200 as Q  # noqa: E402
from paper_2105_00115_b200 import exact  # noqa: E402

with open(os.path.join(G.GOLDEN, "exact_golden.json")) as f:
    EXACT = json.load(f)["cases"]


def vec(case):
    if "input" in case:
        z = G._npz()
        return z[case["input"] + "__x"], z[case["input"] + "__y"]
    return (np.array([float.fromhex(v) for v in case["x"]]), np.array([float.fromhex(v) for v in case["y"]]))


@pytest.mark.parametrize("case", EXACT, ids=lambda c: c["name"])
def test_reference_dot_golden(case):
    x, y = vec(case)
    if case["raises"]:
        with pytest.raises({"ValueError": ValueError, "OverflowError": OverflowError}[case["raises"]]):
            Q.reference_dot(x, y)
        return
    r = Q.reference_dot(x, y)
    assert r.value.hex() == case["value"]
    assert r.flexp_e == case["flexp_e"]
    assert float(r.plain).hex() == case["plain"]


@pytest.mark.parametrize("case", G.select(lambda c: "exact" in c, max_n=1 << 20), ids=lambda c: c["name"])
def test_exact_field_of_qdot_goldens(case):
    x, y = G.inputs(case)
    if case["exact"] is None:
        with pytest.raises(OverflowError):
            Q.reference_dot(x, x if case["norm"] else y, plain=False)
        return
    r = Q.reference_dot(x, x if case["norm"] else y, plain=False)
    assert r.value == G.hexf(case["exact"])
    assert r.flexp_e == case["exact_flexp"]
    assert math.isnan(r.plain) or case["n"] == 0


def fraction_dot(x, y):
    return float(sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y)))


@pytest.mark.parametrize("seed", range(6))
def test_random_wide_against_fractions(seed):
    rng = np.random.default_rng(100 + seed)
    n = 2000
    x = np.ldexp(rng.normal(size=n), rng.integers(-1070, 1000, n))
    y = np.ldexp(rng.normal(size=n), rng.integers(-60, 20, n))
    x[::17] = 0.0
    x[5::29] = rng.normal(size=len(x[5::29])) * 2.0 ** -1074 * 7   # subnormals
    try:
        want = fraction_dot(x, y)
    except OverflowError:
        with pytest.raises(OverflowError):
            Q.reference_dot(x, y)
        return
    r = Q.reference_dot(x, y)
    assert r.value == want


def test_sharded_regions_sum_to_whole():
    # emulate 4 ranks on one device: per-shard accumulators, summed, then finalize
    import ctypes
    from paper_2105_00115_b200 import _lib
    from paper_2105_00115_b200.device import stream_handle
    rng = np.random.default_rng(3)
    x = rng.standard_normal(1 << 20) * np.exp2(rng.integers(-200, 200, 1 << 20))
    y = rng.standard_normal(1 << 20)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    lib = _lib.load()
    s = stream_handle(xd.device)
    total = None
    bounds = np.linspace(0, x.size, 5).astype(int)
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        ws = exact._ExactWs(xd.device)
        _lib.check(lib.qdot_b200_exact_begin(ws.ptr, s))
        _lib.check(lib.qdot_b200_exact_accumulate(xd[lo:].data_ptr(), yd[lo:].data_ptr(), int(hi - lo), 0, ws.ptr, s))
        reg = ws.buf[:ws.region_words]
        total = reg.clone() if total is None else total + reg
    ws = exact._ExactWs(xd.device)
    _lib.check(lib.qdot_b200_exact_begin(ws.ptr, s))
    ws.buf[:ws.region_words] = total
    _lib.check(lib.qdot_b200_exact_finalize(ws.ptr, s))
    r = _lib.QdotExactResult()
    _lib.check(lib.qdot_b200_exact_fetch(ws.ptr, ctypes.byref(r), s))
    whole = Q.reference_dot(xd, yd, plain=False)
    assert r.value == whole.value and r.status == 0


def test_norm_mode_and_symmetry():
    rng = np.random.default_rng(8)
    x = rng.standard_normal(300001)
    y = rng.standard_normal(300001)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    assert Q.reference_dot(xd, xd).value == Q.reference_dot(xd, xd.clone()).value
    a, b = Q.reference_dot(xd, yd), Q.reference_dot(yd, xd)
    assert a.value == b.value and a.plain == b.plain
    assert Q.reference_dot(xd, -yd).value == -a.value
    # plain is the numpy left-to-right sum of the rounded products
    assert a.plain == float(np.add.accumulate(x * y)[-1])


@pytest.mark.slow
def test_c2_exact_bounds_qdot():
    # C2 (2^28 standard normal): the qdot value lies within abs_cap of the exact dot
    from oracle import oracle as O
    x, y = O.gen_normal(1 << 28, seed=0)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    r = Q.reference_dot(xd, yd, plain=False)
    rep = Q.qdot(xd, yd, Q.ToleranceConfig(1e-8))
    assert rep.value == -23532.7407708119
    assert abs(rep.value - r.value) <= rep.abs_cap
    del xd, yd
