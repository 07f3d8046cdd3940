"""Pin the CPU oracle (oracle/qdot_oracle.c) to the reference's own outputs.

Every golden case in tests/golden/golden_cases.json was produced by running
the unmodified reference package (tests/golden/make_golden.py).  The oracle
must reproduce values, bins, scores, precisions, per-bin values, counts,
bounds and error behaviour bit for bit before any GPU result is compared
against it.
"""

import math

import numpy as np
import pytest

import golden_util as G
from oracle import oracle as O

CASES = G.cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(case):
    x, y = G.inputs(case)
    if "error" in case:
        exc = {"ValueError": ValueError, "OverflowError": OverflowError}[case["error"]]
        with pytest.raises(exc):
            O.qdot(x, y, G.hexf(case["epsilon"]), case["split"], case["input_mu"], case["strategy"])
        return
    r = O.qdot(x, y, G.hexf(case["epsilon"]), case["split"], case["input_mu"], case["strategy"], members=True)
    zero_idx = np.flatnonzero((x == 0) | (y == 0))
    assert G.members_sha(zero_idx, [b.indices for b in r.bins]) == case["members_sha"]
    got_bins = [[b.lower, b.upper, b.cardinality, b.score, b.precision] for b in r.bins]
    want_bins = [b[:5] for b in case["bins"]]
    assert got_bins == want_bins
    for b, w in zip(r.bins, case["bins"]):
        v = G.hexf(w[5])
        assert b.value == v or (math.isnan(b.value) and math.isnan(v)), (b, w)
    want = G.hexf(case["value"])
    assert r.value == want or (math.isnan(r.value) and math.isnan(want))
    assert r.n_bins == case["n_bins"]
    assert r.early_terminated == case["early_terminated"]
    assert r.eps_eff == G.hexf(case["eps_eff"])
    if case["n_bins"]:
        assert (r.e_min, r.e_max) == (case["e_min"], case["e_max"])
    assert r.zero_count == case["zero_count"]
    assert {G.PREC_LABEL[k]: v for k, v in r.counts.items()} == case["counts"]
    assert r.abs_bound == G.hexf(case["abs_bound"])
    assert r.rel_bound == G.hexf(case["rel_bound"])
    assert r.rel_guarantee == G.hexf(case["rel_guarantee"])


@pytest.mark.parametrize("case", [c for c in CASES if c.get("exact") and "error" not in c][:200],
                         ids=lambda c: c["name"])
def test_oracle_exact_dot(case):
    x, y = G.inputs(case)
    v, fe, _ = O.exact_dot(x, y)
    assert v == G.hexf(case["exact"])
    assert fe == case["exact_flexp"]


def test_round_half_known_answers():
    # test_emulate.py:22-32 tie-to-even and overflow
    assert O.round_half(1.0 + 2.0**-11) == 1.0
    assert O.round_half(1.0 + 3 * 2.0**-11) == 1.0 + 2 * 2.0**-10
    assert math.isinf(O.round_half(2.0**20))
    assert O.round_half(65504.0) == 65504.0
    assert math.isinf(O.round_half(65520.0))
    assert O.round_half(65519.9) == 65504.0


def test_round_matches_numpy_casts():
    rng = np.random.default_rng(0)
    vals = np.concatenate([np.ldexp(rng.uniform(-2, 2, 4000), rng.integers(-40, 20, 4000)),
                           np.array([65519.9, 65520.0, 6.1e-5, 5.9e-8, 2.0**-25, 2.0**-24 * 1.5,
                                     -65520.0, 0.0, 3e-38, 1e-45, 7e-46])])
    with np.errstate(over="ignore"):
        h = vals.astype(np.float16).astype(np.float64)
        s = vals.astype(np.float32).astype(np.float64)
    for v, a, b in zip(vals.tolist(), h.tolist(), s.tolist()):
        assert O.round_half(v) == a or (math.isinf(a) and math.isinf(O.round_half(v)))
        assert O.round_single(v) == b


def test_flexp_subnormal():
    # test_floatbits.py:48-52
    assert O.flexp(5e-324) == -1074
    assert O.flexp(1.0) == 0
    assert O.flexp(0.75) == -1


def test_fold_known_answer():
    # test_emulate.py:160-162
    assert O.neumaier([0.0, 0.0, 2.0**17, 2.0**50]) == 1125899906973696.0
    assert O.neumaier([1.0] + [2.0**-60] * 1000) == math.fsum([1.0] + [2.0**-60] * 1000)


def test_hist_matches_golden_counts():
    case = next(c for c in CASES if c["name"] == "C1_none")
    x, y = G.inputs(case)
    counts, z = O.hist(x, y)
    assert z == case["zero_count"]
    present = [(k - O.KEY_OFF, int(c)) for k, c in enumerate(counts) if c]
    assert [p[0] for p in present] == [b[1] for b in case["bins"]]
    assert [p[1] for p in present] == [b[2] for b in case["bins"]]
