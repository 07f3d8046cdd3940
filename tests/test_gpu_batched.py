"""GPU parity of qdot_batched (BASELINE configs[3]) against the reference's
golden rows and a per-row loop of the oracle."""

import math

import numpy as np
import pytest

import golden_util as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_00115_b200 as Q  # noqa: E402
from oracle import oracle as O  # noqa: E402

LABELS = ["perforate", "half", "single", "double"]


def check_rows(X, Y, rep, eps, split="none", strategy="exact"):
    for r in range(X.shape[0]):
        o = O.qdot(X[r], Y[r], eps, split, 52, strategy)
        assert rep.n_bins[r] == o.n_bins, r
        assert [int(v) for v in rep.counts[r]] == [o.counts[k] for k in range(4)], r
        if o.n_bins:
            assert (rep.e_min[r], rep.e_max[r]) == (o.e_min, o.e_max), r
        assert bool(rep.early_terminated[r]) == o.early_terminated
        assert rep.values[r] == o.value or (math.isnan(o.value) and math.isnan(rep.values[r])), \
            (r, rep.values[r], o.value)


def test_c4_golden_rows():
    names = ["C4_row0", "C4_row1", "C4_row2", "C4_row65535"]
    cases = {c["name"]: c for c in G.cases() if c["name"] in names}
    X = np.stack([G.inputs(cases[nm])[0] for nm in names])
    Y = np.stack([G.inputs(cases[nm])[1] for nm in names])
    rep = Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6))
    for i, nm in enumerate(names):
        c = cases[nm]
        assert rep.values[i] == G.hexf(c["value"]), nm
        assert rep.n_bins[i] == c["n_bins"]
        assert {LABELS[k]: int(rep.counts[i, k]) for k in range(4)} == c["counts"]
    assert rep.values[0] == 45.36721523563339 and rep.values[3] == 72.77242249700646
    assert len(rep.general_rows) == 0


def test_golden_mixed_rows():
    cases = [c for c in G.cases() if c["name"].startswith("batch_")]
    for c in cases:
        x, y = G.inputs(c)
        cfg = Q.ToleranceConfig(G.hexf(c["epsilon"]), Q.SplitMode(c["split"]))
        rep = Q.qdot_batched(x[None, :], y[None, :], cfg)
        assert rep.n_bins[0] == c["n_bins"], c["name"]
        assert {LABELS[k]: int(rep.counts[0, k]) for k in range(4)} == c["counts"], c["name"]
        assert rep.values[0] == G.hexf(c["value"]), c["name"]


@pytest.mark.parametrize("eps,split", [(1e-6, "none"), (1e-3, "per-bin"), (1e-10, "none"), (1e-1, "none")])
def test_random_normal_rows(eps, split):
    rng = np.random.default_rng(31)
    X = rng.standard_normal((257, 4096))
    Y = rng.standard_normal((257, 4096))
    X[7, ::13] = 0.0
    rep = Q.qdot_batched(X, Y, Q.ToleranceConfig(eps, Q.SplitMode(split)))
    check_rows(X, Y, rep, eps, split)


def test_special_rows_and_layouts():
    rng = np.random.default_rng(32)
    rows = []
    for r in range(24):
        x, y = O.gen_family("AB"[r % 2], [4, 20, 80, 200][r % 4], 1000, 900 + r)
        rows.append((x, y))
    X = np.stack([r[0] for r in rows])
    Y = np.stack([r[1] for r in rows])
    X[3, :] = 0.0                                   # all-zero row
    X[5, 10] = 5e-320                               # subnormal factor
    X[6, :] = 1.0
    Y[6, :] = 1.0                                   # early-terminated row
    Y[8, 0] = 1e300                                 # wide spread -> general path
    for eps in [1e-4, 1e-9]:
        rep = Q.qdot_batched(X, Y, Q.ToleranceConfig(eps))
        check_rows(X, Y, rep, eps)
        assert 8 in rep.general_rows.tolist()
    # odd length (scalar loads) and a row stride larger than the length
    Xt = torch.from_numpy(np.ascontiguousarray(X[:, :999])).cuda()
    Yt = torch.from_numpy(np.ascontiguousarray(Y[:, :999])).cuda()
    rep = Q.qdot_batched(Xt, Yt, Q.ToleranceConfig(1e-7))
    check_rows(X[:, :999], Y[:, :999], rep, 1e-7)
    big = torch.from_numpy(np.concatenate([X, X], axis=1)).cuda()[:, :1000]
    bigy = torch.from_numpy(np.concatenate([Y, Y], axis=1)).cuda()[:, :1000]
    rep = Q.qdot_batched(big, bigy, Q.ToleranceConfig(1e-7))
    check_rows(X, Y, rep, 1e-7)
    # norm mode
    rep = Q.qdot_batched(X, X, Q.ToleranceConfig(1e-7))
    check_rows(X, X, rep, 1e-7)


def check_bins(X, Y, rep, eps, split="none", strategy="exact"):
    """Per-row bin tables bit-equal to the oracle's (lower, upper, cardinality,
    score, precision, value)."""
    for r in range(X.shape[0]):
        o = O.qdot(X[r], Y[r], eps, split, 52, strategy)
        got = [(int(b["lower"]), int(b["upper"]), int(b["cardinality"]), int(b["score"]), int(b["precision"]),
                float(b["value"])) for b in rep.row_bins(r)]
        want = [(b.lower, b.upper, b.cardinality, b.score, b.precision, b.value) for b in o.bins]
        assert got == want, (r, strategy)


@pytest.mark.parametrize("strategy", ["ranged:1", "ranged:2", "ranged:3", "ranged:7", "ranged:40", "split:0",
                                      "split:1", "split:3", "split:6", "split:12"])
@pytest.mark.parametrize("eps,split", [(1e-4, "none"), (1e-9, "per-bin"), (1e-1, "none")])
def test_non_exact_strategies_on_device(strategy, eps, split):
    """Ranged / split rows finish in the fused kernel (no per-row host loop),
    bit-exact against the oracle, bin tables included."""
    rng = np.random.default_rng(33)
    X = rng.standard_normal((40, 700))
    Y = rng.standard_normal((40, 700))
    X[3, ::5] = 0.0
    X[4] *= np.exp2(rng.integers(-20, 20, 700))          # wider exponent spread
    X[5, :] = 1.0
    Y[5, :] = 1.0                                        # early-terminated row
    st = Q.parse_strategy(strategy)
    cfg = Q.ToleranceConfig(eps, Q.SplitMode(split))
    rep = Q.qdot_batched(X, Y, cfg, strategy=st, bins=True)
    check_rows(X, Y, rep, eps, split, strategy)
    check_bins(X, Y, rep, eps, split, strategy)
    # rerun rows: the wide row, and rows with an order-sensitive HALF bin (fp32 replay in index order)
    assert all(r == 4 or rep.half_order_sensitive[r] for r in rep.general_rows.tolist()), rep.general_rows
    repn = Q.qdot_batched(X, X, cfg, strategy=st, bins=True)
    check_rows(X, X, repn, eps, split, strategy)
    check_bins(X, X, repn, eps, split, strategy)


@pytest.mark.parametrize("strategy", ["exact", "ranged:3", "split:5"])
def test_bin_tables_golden_and_general(strategy):
    """bins=True on C4 golden rows, mixed special rows and a wide-spread row
    that reruns on the single-vector path."""
    names = ["C4_row0", "C4_row1", "C4_row2", "C4_row65535"]
    cases = {c["name"]: c for c in G.cases() if c["name"] in names}
    X = np.stack([G.inputs(cases[nm])[0] for nm in names])
    Y = np.stack([G.inputs(cases[nm])[1] for nm in names])
    X[2, 0] = 1e300                                      # spread > 64 keys: rerun row
    rep = Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6), strategy=Q.parse_strategy(strategy), bins=True)
    assert 2 in rep.general_rows.tolist()
    check_rows(X, Y, rep, 1e-6, "none", strategy)
    check_bins(X, Y, rep, 1e-6, "none", strategy)
    if strategy == "exact":
        assert rep.values[0] == 45.36721523563339 and rep.values[3] == 72.77242249700646


def test_ranged_c4_shape_no_host_loop():
    """The former per-row host cliff: 4096 rows x 4096, ranged:3 -- all rows on
    device (none rerun), values equal to the exact per-row oracle on a sample."""
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn(4096, 4096, dtype=torch.float64, device="cuda", generator=g)
    Y = torch.randn(4096, 4096, dtype=torch.float64, device="cuda", generator=g)
    rep = Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6), strategy=Q.RangedBinning(3))
    assert len(rep.general_rows) == 0
    Xh, Yh = X[:64].cpu().numpy(), Y[:64].cpu().numpy()
    sub = Q.qdot_batched(Xh, Yh, Q.ToleranceConfig(1e-6), strategy=Q.RangedBinning(3))
    assert np.array_equal(sub.values, rep.values[:64])
    check_rows(Xh, Yh, sub, 1e-6, "none", "ranged:3")


def test_errors():
    X = np.ones((3, 8))
    Y = np.ones((3, 8))
    Y[1, 2] = np.nan
    with pytest.raises(ValueError):
        Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-3))
    with pytest.raises(ValueError):
        Q.qdot_batched(np.ones(8), np.ones(8), Q.ToleranceConfig(1e-3))
    with pytest.raises(ValueError):
        Q.qdot_batched(np.ones((2, 8)), np.ones((3, 8)), Q.ToleranceConfig(1e-3))


@pytest.mark.slow
def test_c4_full_size():
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((65536, 4096))).cuda()
    Y = torch.from_numpy(rng.standard_normal((65536, 4096))).cuda()
    rep = Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6))
    assert rep.values[0] == 45.36721523563339
    assert rep.values[1] == -110.94441662421859
    assert rep.values[65535] == 72.77242249700646
    assert len(rep.general_rows) == 0
    rep2 = Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6))
    assert np.array_equal(rep.values, rep2.values)
