"""GPU: the one-launch cluster path (qdot_b200_small, csrc/qdot_small.cuh)
against the four-launch pipeline (begin, pass 1, score, pass 2) on the same
inputs -- result header and every bin bit-identical -- and against the CPU
oracle; the hand-over cases (keys outside the 64-key table, DOUBLE overflow,
no nonzero product, early termination below input_mu 52) are checked to take
the hand-over path (A[A_SMALL] == 2) and still agree."""

import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_00115_b200 as Q  # noqa: E402
from paper_2105_00115_b200 import _lib  # noqa: E402
from paper_2105_00115_b200.device import config_struct  # noqa: E402
from oracle import oracle as O  # noqa: E402

A_SMALL = 12664          # int64 word of region A (qdot_common.cuh)
LIB = _lib.load()


def _ws():
    nb = int(LIB.qdot_b200_workspace_bytes())
    return torch.zeros(nb, dtype=torch.uint8, device="cuda")


def _fetch(ws, s):
    res = _lib.QdotResult()
    bins = (_lib.QdotBin * (_lib.KEYS + 1))()
    _lib.check(LIB.qdot_b200_fetch(ws.data_ptr(), ctypes.byref(res), bins, _lib.KEYS + 1, s), LIB)
    torch.cuda.synchronize()
    return res, [bins[i] for i in range(res.n_bins)]


def run_small(x, y, norm, c):
    ws = _ws()
    s = torch.cuda.current_stream().cuda_stream
    n = int(x.shape[0])
    yp = x.data_ptr() if norm else y.data_ptr()
    _lib.check(LIB.qdot_b200_small(x.data_ptr(), yp, n, int(norm), ctypes.byref(c), ws.data_ptr(), s), LIB)
    _lib.check(LIB.qdot_b200_score_finalize(ws.data_ptr(), n, ctypes.byref(c), s), LIB)
    _lib.check(LIB.qdot_b200_pass2_finalize(x.data_ptr(), yp, n, int(norm), ws.data_ptr(), s), LIB)
    res, bins = _fetch(ws, s)
    state = int(ws[A_SMALL * 8:A_SMALL * 8 + 8].view(torch.int64).item())
    return res, bins, state


def run_four(x, y, norm, c):
    ws = _ws()
    s = torch.cuda.current_stream().cuda_stream
    n = int(x.shape[0])
    yp = x.data_ptr() if norm else y.data_ptr()
    _lib.check(LIB.qdot_b200_begin(ws.data_ptr(), s), LIB)
    _lib.check(LIB.qdot_b200_pass1(x.data_ptr(), yp, n, int(norm), ctypes.byref(c), n, ws.data_ptr(), s), LIB)
    _lib.check(LIB.qdot_b200_score_finalize(ws.data_ptr(), n, ctypes.byref(c), s), LIB)
    _lib.check(LIB.qdot_b200_pass2_finalize(x.data_ptr(), yp, n, int(norm), ws.data_ptr(), s), LIB)
    return _fetch(ws, s)


def same(a, b):
    return a == b or (math.isnan(a) and math.isnan(b))


def bin_tuple(b):
    return (b.lower, b.upper, b.cardinality, b.score, b.precision, b.first_key, b.last_key, b.flags)


def assert_same(r1, b1, r2, b2):
    assert r1.status == r2.status
    if r1.status != _lib.QDOT_OK:
        return
    assert same(r1.value, r2.value), (r1.value, r2.value)
    for f in ("eps_eff", "n", "nnz", "zero_count", "n_bins", "e_min", "e_max", "early_terminated",
              "pass2_needed", "half_order_sensitive"):
        assert getattr(r1, f) == getattr(r2, f), f
    assert list(r1.counts) == list(r2.counts)
    assert [bin_tuple(b) for b in b1] == [bin_tuple(b) for b in b2]
    assert all(same(a.value, b.value) for a, b in zip(b1, b2))


def data(kind, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    y = rng.standard_normal(n)
    if kind == "wide":
        x *= np.exp2(rng.integers(-300, 300, n))
    elif kind == "special":
        x[rng.integers(0, n, max(1, n // 50))] = 0.0
        x[rng.integers(0, n, max(1, n // 200))] = 5e-320
    elif kind == "nonfinite":
        x[rng.integers(0, n, 1)] = np.inf
    elif kind == "overflow":
        x[rng.integers(0, n, 1)] = 1e300
        y[rng.integers(0, n, 1)] = 1e300
        x[0], y[0] = 1e300, 1e300
    elif kind == "zeros":
        x[:] = 0.0
    elif kind == "narrow":                     # early termination at loose epsilon
        x = 1.0 + rng.random(n)
        y = 1.0 + rng.random(n)
    return x, y


CASES = [
    # kind, n, norm, eps, split, mu, expected state
    ("normal", 1, False, 1e-8, 1, 52, 1),
    ("normal", 2, False, 1e-8, 1, 52, 1),
    ("normal", 777, False, 1e-8, 1, 52, 1),
    ("normal", 10_000, False, 1e-8, 1, 52, 1),
    ("normal", 10_000, True, 1e-8, 1, 52, 1),
    ("normal", 16_384, False, 1e-12, 0, 52, 1),
    ("normal", 40_001, False, 1e-8, 1, 52, 1),
    ("normal", 65_536, True, 1e-6, 1, 52, 1),
    ("normal", 65_536, False, 1e-3, 1, 23, 1),
    ("normal", 5_000, False, 1e-2, 1, 10, None),
    ("special", 20_000, False, 1e-8, 1, 52, 2),       # subnormal factors: keys far below the table
    ("wide", 3_000, False, 1e-3, 1, 52, 2),
    ("wide", 65_536, True, 1e-3, 1, 52, 2),
    ("nonfinite", 1_000, False, 1e-8, 1, 52, 1),
    ("overflow", 1_000, False, 1e-8, 1, 52, 2),
    ("zeros", 1_000, False, 1e-8, 1, 52, 2),
    ("narrow", 4_096, False, 1e-2, 1, 52, 1),
    ("narrow", 4_096, False, 1e-1, 1, 10, None),
]


@pytest.mark.parametrize("kind,n,norm,eps,split,mu,state", CASES,
                         ids=[f"{c[0]}-{c[1]}-{'norm' if c[2] else 'dot'}-{c[3]}-mu{c[5]}" for c in CASES])
def test_small_matches_four_launch_pipeline(kind, n, norm, eps, split, mu, state):
    x, y = data(kind, n, n + len(kind))
    if norm:
        y = x
    cfg = Q.ToleranceConfig(eps, split=Q.SplitMode.PER_BIN if split else Q.SplitMode.NONE, input_mu=mu)
    c = config_struct(cfg, Q.ExactBinning())
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    r1, b1, st = run_small(xd, yd, norm, c)
    r2, b2 = run_four(xd, yd, norm, c)
    assert_same(r1, b1, r2, b2)
    if state is not None:
        assert st == state, st
    if r1.status == _lib.QDOT_OK and r1.half_order_sensitive == 0:
        try:
            ref = O.qdot(x, y, eps, "per-bin" if split else "none", mu, "exact")
        except OverflowError:                  # the reference's bound terms overflow (math.ldexp)
            with pytest.raises(OverflowError):
                Q.qdot(xd, xd if norm else yd, cfg)
            return
        assert same(r1.value, ref.value), (r1.value, ref.value)
        assert [(b.lower, b.upper, b.cardinality, b.score, b.precision) for b in b1] == \
            [(w.lower, w.upper, w.cardinality, w.score, w.precision) for w in ref.bins]


def test_enqueue_uses_the_cluster_path_at_small_n():
    """qdot_b200_enqueue (what qdot() and the solvers run) takes the cluster
    path at n <= 16384 and the four-launch pipeline above it."""
    cfg = Q.ToleranceConfig(1e-8)
    c = config_struct(cfg, Q.ExactBinning())
    s = torch.cuda.current_stream().cuda_stream
    for n, want in ((5_000, 1), (16_384, 1), (16_385, 0), (100_000, 0)):
        x, y = data("normal", n, 3)
        xd = torch.from_numpy(x).cuda()
        yd = torch.from_numpy(y).cuda()
        ws = _ws()
        _lib.check(LIB.qdot_b200_enqueue(xd.data_ptr(), yd.data_ptr(), n, 0, ctypes.byref(c), ws.data_ptr(), s), LIB)
        res, bins = _fetch(ws, s)
        assert int(ws[A_SMALL * 8:A_SMALL * 8 + 8].view(torch.int64).item()) == want, n
        ref = O.qdot(x, y, 1e-8)
        assert same(res.value, ref.value)
        assert Q.qdot(xd, yd, cfg).value == ref.value
