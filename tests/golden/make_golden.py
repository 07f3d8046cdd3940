"""Generate golden vectors for the qdot hot path BY RUNNING THE REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the unmodified reference package (qdot 0.1.0 from
/root/reference/pkg/src) and records, for every case, the reference's own
`qdot` report (value, bins with lower/upper/cardinality/score/precision, the
per-bin `bin_dot` values, counts, bounds, flags) plus `reference_dot`.
Inputs are stored in golden_inputs.npz (small cases) or regenerated from a
seeded generator whose output checksum is recorded (large cases).  The GPU
box never reads /root/reference: tests consume only these committed files.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from qdot.binning import BinSplitting, ExactBinning, RangedBinning  # noqa: E402
from qdot.emulate import bin_dot  # noqa: E402
from qdot.kernel import qdot, reference_dot  # noqa: E402
from qdot.scoring import SplitMode, ToleranceConfig  # noqa: E402

from oracle.oracle import gen_family, gen_illcond, gen_normal  # noqa: E402  (generators only)

PREC = {"perforate": 0, "half": 1, "single": 2, "double": 3}


def strat_obj(s):
    head, _, arg = s.partition(":")
    if head == "exact":
        return ExactBinning()
    if head == "ranged":
        return RangedBinning(int(arg))
    return BinSplitting(int(arg))


def checksum(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:16]


def members_sha(ps) -> str:
    """Digest of the member order: zero_idx then every bin's indices, int64."""
    h = hashlib.sha256(np.ascontiguousarray(ps.zero_idx, dtype=np.int64).tobytes())
    for b in ps.bins:
        h.update(b"|")
        h.update(np.ascontiguousarray(b.indices, dtype=np.int64).tobytes())
    return h.hexdigest()[:16]


def half_seq_inputs(n: int = 1 << 18, seed: int = 21):
    """Positive products whose HALF bins' fp32 running sums leave the exact
    range of fp32 (the reference's sequential sum then rounds, order-sensitively)."""
    rng = np.random.default_rng(seed)
    return np.abs(rng.standard_normal(n)), np.abs(rng.standard_normal(n))


def run_case(name, x, y, eps, split, strategy, input_mu=52, norm=False, store=True, key=None):
    cfg = ToleranceConfig(epsilon=eps, split=SplitMode.PER_BIN if split == "per-bin" else SplitMode.NONE,
                          input_mu=input_mu)
    case = {"name": name, "n": int(x.shape[0]), "epsilon": float(eps).hex(), "split": split,
            "strategy": strategy, "input_mu": input_mu, "norm": norm,
            "x_sha": checksum(x), "y_sha": checksum(y), "stored": store,
            "input": key or name}
    xx = x
    yy = x if norm else y
    try:
        rep = qdot(xx, yy, cfg, strategy=strat_obj(strategy))
    except (ValueError, OverflowError) as exc:
        case["error"] = type(exc).__name__
        return case
    ps = rep.params
    case.update({
        "value": float(rep.value).hex(),
        "abs_bound": float(rep.abs_bound).hex(),
        "rel_bound": float(rep.rel_bound).hex(),
        "abs_cap": float(rep.abs_cap).hex(),
        "rel_guarantee": float(rep.rel_guarantee).hex(),
        "rel_hypothesis": rep.rel_hypothesis,
        "early_terminated": bool(rep.early_terminated),
        "e_min": int(ps.e_min), "e_max": int(ps.e_max),
        "n_bins": int(ps.n_bins), "eps_eff": float(ps.eps_eff).hex(),
        "zero_count": int(ps.zero_idx.size),
        "counts": {lvl.label: int(c) for lvl, c in rep.counts.items()},
        "bins": [[int(b.lower), int(b.upper), int(b.cardinality), int(b.score),
                  PREC[b.precision.label], float(bin_dot(xx, yy, b)).hex()]
                 for b in ps.bins],
        "members_sha": members_sha(ps),
    })
    try:
        ref = reference_dot(xx, yy)
        case["exact"] = float(ref.value).hex()
        case["exact_flexp"] = ref.flexp_e
    except OverflowError:
        case["exact"] = None
    # bit-exactness sanity of the per-bin values we just recorded
    return case


def main():
    cases = []
    inputs = {}

    def add(name, x, y, eps, split="none", strategy="exact", input_mu=52, norm=False, store=True,
            key=None):
        c = run_case(name, x, y, eps, split, strategy, input_mu, norm, store, key)
        cases.append(c)
        if store and (key or name) + "__x" not in inputs:
            inputs[(key or name) + "__x"] = np.asarray(x, dtype=np.float64)
            inputs[(key or name) + "__y"] = np.asarray(y, dtype=np.float64)

    # --- toy (test_kernel.py:15-17) under every strategy/split
    tx = np.array([2.0**27, 2.0**8, 2.0**-3, 2.0**20])
    ty = np.array([2.0**23, 2.0**-14, 2.0**7, 2.0**-3])
    for st in ["exact", "ranged:1", "ranged:3", "ranged:60", "split:0", "split:1", "split:2", "split:40"]:
        for sp in ["none", "per-bin"]:
            add(f"toy_{st}_{sp}", tx, ty, 2.0**-34, sp, st, key="toy")

    # --- oracle-equivalence set (test_kernel.py:125-141)
    for st in ["exact", "ranged:3", "split:3"]:
        for seed in range(40):
            rng = np.random.default_rng(seed)
            n = int(rng.integers(1, 65))
            x = np.ldexp(rng.uniform(0.5, 1, n) * rng.choice([-1, 1], n), rng.integers(-25, 25, n))
            y = np.ldexp(rng.uniform(0.5, 1, n), rng.integers(-25, 25, n))
            if seed % 5 == 0:
                x[rng.integers(0, n)] = 0.0
            eps = float(np.ldexp(1.0, -int(rng.integers(0, 50))))
            sp = "per-bin" if seed % 2 else "none"
            add(f"equiv_{st}_{seed}", x, y, eps, sp, st)

    # --- harness families A/B, mid-size, all strategies, both splits, several eps
    for k, (fam, t) in enumerate([("A", 10), ("A", 40), ("A", 100), ("B", 6), ("B", 14), ("B", 30)]):
        x, y = gen_family(fam, t, 3000, 1000 + k)
        for eps in [1e-2, 1e-5, 1e-8, 1e-12, 2.0**-52]:
            for st in ["exact", "ranged:2", "ranged:5", "split:2", "split:5"]:
                for sp in ["none", "per-bin"]:
                    add(f"fam{fam}{t}_{eps:g}_{st}_{sp}", x, y, eps, sp, st, key=f"fam{fam}{t}")

    # --- norm mode and input_mu clamps
    x, y = gen_family("B", 10, 2000, 7)
    for mu in [52, 23, 10]:
        for eps in [1e-3, 1e-6, 1e-9]:
            add(f"mu{mu}_{eps:g}", x, y, eps, "none", "exact", input_mu=mu, key="muB10")
            add(f"mu{mu}_{eps:g}_norm", x, x, eps, "per-bin", "exact", input_mu=mu, norm=True,
                key="muB10x")

    # --- edge cases
    add("empty", np.zeros(0), np.zeros(0), 2.0**-34)
    add("single", np.array([3.0]), np.array([-5.0]), 1e-6)
    add("all_zero", np.zeros(4), np.ones(4), 2.0**-34)
    add("neg_zero", np.array([-0.0, 1.0, 2.0, -0.0]), np.array([1.0, -0.0, 3.0, 4.0]), 1e-6)
    add("all_ones", np.ones(1024), np.ones(1024), 2.0**-34, norm=True)
    add("zero_component", np.array([1.0, 0.0, 4.0]), np.ones(3), 1e-3)
    sub = np.array([5e-324, -1e-310, 2.2e-308, 3.0, -4e-320, 1e-300, 7.0, 1e300])
    add("subnormal_mix", sub, sub[::-1].copy(), 1e-6)
    add("subnormal_mix_norm", sub, sub, 1e-6, norm=True)
    big = np.array([1e300, -1e300, 1.5e307, 3.0, 1e-5])
    add("near_overflow", big, np.array([1e8, 1e8, 2.0, 1.0, 1.0]), 1e-9)
    add("product_overflow", np.array([1e300, 1.0]), np.array([1e300, 1.0]), 1e-9)
    add("product_underflow", np.array([1e-200, 1e-170, 1.0]), np.array([1e-200, 1e-170, 1.0]), 1e-9)
    rng = np.random.default_rng(11)
    xs = np.ldexp(rng.uniform(0.5, 1, 500), rng.integers(-1070, -1000, 500))
    add("deep_subnormal_products", xs, np.ldexp(rng.uniform(0.5, 1, 500), rng.integers(-60, 60, 500)), 1e-4)
    add("huge_width", tx, ty, 2.0**-34, "none", "ranged:1000000")
    add("split_clamped", np.array([2.0, 4.0]), np.array([1.0, 1.0]), 1e-3, "none", "split:40")
    add("ties_split", np.ldexp(np.ones(64), np.repeat(np.arange(4), 16)), np.ones(64), 1e-3, "none", "split:3")
    add("nonfinite", np.array([1.0, np.inf]), np.ones(2), 1e-3)
    add("nan", np.array([1.0, np.nan]), np.ones(2), 1e-3)
    add("tiny_eps", tx, ty, 5e-324, "per-bin", "exact")
    add("huge_eps", tx, ty, 2.0**60, "none", "exact")
    # cancellation: hypothesis violated
    add("cancel", np.array([1e10, -1e10, 1.0]), np.ones(3), 1e-12)
    # HALF bins that would be order-sensitive in fp32 (big M, loose eps)
    rng = np.random.default_rng(12)
    hx = np.ldexp(rng.uniform(0.5, 1, 20000), rng.integers(-30, 3, 20000))
    add("many_half", hx, np.abs(hx[::-1]).copy(), 1e-1, key="many_half")
    add("many_half_ranged", hx, np.abs(hx[::-1]).copy(), 1e-1, "none", "ranged:4", key="many_half")

    # --- ill-conditioned C3 generator, small
    x, y = gen_illcond(1 << 14, seed=0)
    for st in ["exact", "ranged:8", "split:6"]:
        for sp in ["none", "per-bin"]:
            add(f"illcond14_{st}_{sp}", x, y, 1e-12, sp, st, key="illcond14")

    # --- standard normal, small stored + C1 (2^20) regenerated
    x, y = gen_normal(1 << 12, seed=3)
    for st in ["exact", "ranged:3", "split:4"]:
        for eps in [1e-3, 1e-8]:
            add(f"normal12_{st}_{eps:g}", x, y, eps, "none", st, key="normal12")
    x, y = gen_normal(1 << 20, seed=0)
    for sp in ["none", "per-bin"]:
        add(f"C1_{sp}", x, y, 1e-8, sp, "exact", store=False)
    add("C1_norm", x, x, 1e-8, "none", "exact", norm=True, store=False)
    add("C1_ranged4", x, y, 1e-8, "none", "ranged:4", store=False)
    add("C1_split5", x, y, 1e-8, "none", "split:5", store=False)
    add("C1_loose", x, y, 1e-3, "per-bin", "exact", store=False)
    # HALF bins with 2^13..2^17 positive members: the fp32 running sums round
    # (order-sensitive), so the device must replay them in index order
    x, y = half_seq_inputs()
    for st in ["exact", "ranged:4", "split:3"]:
        for sp in ["none", "per-bin"]:
            add(f"half_seq_{st}_{sp}", x, y, 2.0**10, sp, st, store=False)
    add("half_seq_norm", x, x, 2.0**8, "none", "exact", norm=True, store=False)
    x, y = gen_illcond(1 << 20, seed=0)
    add("C3_2e20", x, y, 1e-12, "none", "exact", store=False)
    add("C3_2e20_perbin", x, y, 1e-12, "per-bin", "exact", store=False)

    # --- C4 batched rows (BASELINE configs[3]): X, Y = default_rng(0) standard normal (65536, 4096)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((65536, 4096))
    Y = rng.standard_normal((65536, 4096))
    for r in [0, 1, 2, 65535]:
        add(f"C4_row{r}", X[r].copy(), Y[r].copy(), 1e-6, "none", "exact", key=f"C4_row{r}")
    del X, Y
    # --- batched parity matrix: 48 rows of mixed families, length 1024
    rng = np.random.default_rng(21)
    for r in range(48):
        fam = "AB"[r % 2]
        t = [6, 14, 30, 60][r % 4]
        x, y = gen_family(fam, t, 1024, 5000 + r)
        if r % 5 == 0:
            x[rng.integers(0, 1024, 40)] = 0.0
        eps = [1e-2, 1e-5, 1e-8, 1e-12][r % 4]
        sp = "per-bin" if r % 3 == 0 else "none"
        add(f"batch_{r}", x, y, eps, sp, "exact", key=f"batch_{r}")

    np.savez_compressed(os.path.join(HERE, "golden_inputs.npz"), **inputs)
    with open(os.path.join(HERE, "golden_cases.json"), "w") as f:
        json.dump({"reference": "qdot 0.1.0 (/root/reference/pkg/src)",
                   "generator": "tests/golden/make_golden.py", "cases": cases}, f, indent=0)
    print(f"{len(cases)} cases written")


if __name__ == "__main__":
    main()
