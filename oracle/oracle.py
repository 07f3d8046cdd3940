"""Python face of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Wraps oracle/_build/libqdot_oracle.so (oracle/qdot_oracle.c, a line-by-line
C restatement of the reference qdot path) with ctypes and rebuilds the
report fields exactly as the reference does (kernel.py:205-240: bounds with
math.fsum over per-bin terms).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker.  The product package never imports it.

Pinned against the reference's own outputs by tests/test_oracle_golden.py
(fixtures from tests/golden/make_golden.py, which imports the reference).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libqdot_oracle.so")

KEYS = 4195
KEY_OFF = 2148
PERFORATE, HALF, SINGLE, DOUBLE = 0, 1, 2, 3
MU = {PERFORATE: 0, HALF: 10, SINGLE: 23, DOUBLE: 52}
NAMES = {PERFORATE: "perforate", HALF: "half", SINGLE: "single", DOUBLE: "double"}

OR_OK, OR_ERR_NONFINITE, OR_ERR_OVERFLOW, OR_ERR_ARG, OR_ERR_EPS, OR_ERR_NOMEM = range(6)


class _Bin(ctypes.Structure):
    _fields_ = [("lower", ctypes.c_int64), ("upper", ctypes.c_int64),
                ("cardinality", ctypes.c_int64), ("score", ctypes.c_int64),
                ("precision", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("value", ctypes.c_double), ("member_start", ctypes.c_int64)]


class _Result(ctypes.Structure):
    _fields_ = [("value", ctypes.c_double), ("eps_eff", ctypes.c_double),
                ("rel_bound_plain", ctypes.c_double),
                ("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("zero_count", ctypes.c_int64),
                ("e_min", ctypes.c_int64), ("e_max", ctypes.c_int64), ("n_bins", ctypes.c_int64),
                ("early_terminated", ctypes.c_int64), ("counts", ctypes.c_int64 * 4)]


_lib = None


def build() -> None:
    """Compile the oracle (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    dp = ctypes.POINTER(ctypes.c_double)
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.or_qdot.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                            ctypes.c_int, ctypes.c_int64, ctypes.POINTER(_Result),
                            ctypes.POINTER(_Bin), ctypes.c_int64, i64p]
    lib.or_qdot.restype = ctypes.c_int
    lib.or_hist.argtypes = [dp, dp, ctypes.c_int64, i64p, i64p]
    lib.or_hist.restype = ctypes.c_int
    lib.or_exact_dot.argtypes = [dp, dp, ctypes.c_int64, dp, i64p, ctypes.POINTER(ctypes.c_int), dp]
    lib.or_exact_dot.restype = ctypes.c_int
    lib.or_round_half.argtypes = [ctypes.c_double]
    lib.or_round_half.restype = ctypes.c_double
    lib.or_round_single.argtypes = [ctypes.c_double]
    lib.or_round_single.restype = ctypes.c_double
    lib.or_flexp_export.argtypes = [ctypes.c_double]
    lib.or_flexp_export.restype = ctypes.c_int64
    lib.or_neumaier.argtypes = [dp, ctypes.c_int64]
    lib.or_neumaier.restype = ctypes.c_double
    lib.or_set_threads.argtypes = [ctypes.c_int]
    lib.or_set_threads.restype = None
    _lib = lib
    return lib


def set_threads(n: int) -> None:
    load().or_set_threads(int(n))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def parse_strategy(strategy) -> tuple:
    """'exact' | 'ranged:W' | 'split:S' | (kind, param) -> (code, param)."""
    if strategy is None:
        return 0, 0
    if isinstance(strategy, tuple):
        kind, param = strategy
    else:
        head, _, arg = str(strategy).partition(":")
        kind, param = head.strip().lower(), (int(arg) if arg else 0)
    return {"exact": 0, "ranged": 1, "split": 2}[kind], int(param)


@dataclass
class OracleBin:
    lower: int
    upper: int
    cardinality: int
    score: int
    precision: int
    value: float
    indices: Optional[np.ndarray] = None


@dataclass
class OracleReport:
    value: float
    bins: List[OracleBin]
    n: int
    nnz: int
    zero_count: int
    e_min: int
    e_max: int
    n_bins: int
    eps_eff: float
    early_terminated: bool
    counts: Dict[int, int]
    abs_bound: float
    rel_bound: float
    abs_cap: float
    rel_guarantee: float
    rel_bound_plain: float = 0.0
    extra: dict = field(default_factory=dict)


def qdot(x, y, epsilon: float, split: str = "none", input_mu: int = 52, strategy=None,
         members: bool = False) -> OracleReport:
    """Oracle restatement of kernel.qdot (kernel.py:179-240)."""
    lib = load()
    x = _f64(x)
    y = x if y is x else _f64(y)
    if x.ndim != 1 or y.ndim != 1:
        raise ValueError("inputs must be 1-D arrays")
    if x.shape[0] != y.shape[0]:
        raise ValueError(f"length mismatch: {x.shape[0]} vs {y.shape[0]}")
    n = x.shape[0]
    code, param = parse_strategy(strategy)
    res = _Result()
    max_bins = KEYS + 1
    bins = (_Bin * max_bins)()
    mem = np.empty(max(n, 1), dtype=np.int64) if members else None
    st = lib.or_qdot(_ptr(x), _ptr(y), n, float(epsilon), 1 if split == "per-bin" else 0,
                     int(input_mu), code, param, ctypes.byref(res), bins, max_bins,
                     mem.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if members else None)
    if st == OR_ERR_NONFINITE:
        raise ValueError("inputs must be finite")
    if st == OR_ERR_OVERFLOW:
        raise OverflowError("rounded bin product overflowed its format")
    if st == OR_ERR_EPS:
        raise ValueError("floor_log2 needs a positive finite value")
    if st != OR_OK:
        raise RuntimeError(f"oracle status {st}")
    out_bins = []
    for b in range(res.n_bins):
        cb = bins[b]
        ob = OracleBin(cb.lower, cb.upper, cb.cardinality, cb.score, cb.precision, cb.value)
        if members:
            ob.indices = mem[cb.member_start:cb.member_start + cb.cardinality].copy()
        out_bins.append(ob)
    e_max = res.e_max
    # kernel.py:205-206 -- fsum over M * ldexp(eps_k, u+1) and M * ldexp(eps_k, u-e_max+1)
    abs_bound = math.fsum(b.cardinality * math.ldexp(math.ldexp(1.0, -MU[b.precision]), b.upper + 1)
                          for b in out_bins)
    rel_bound = math.fsum(b.cardinality * math.ldexp(math.ldexp(1.0, -MU[b.precision]),
                                                      b.upper - e_max + 1) for b in out_bins)
    return OracleReport(
        value=res.value, bins=out_bins, n=n, nnz=res.nnz, zero_count=res.zero_count,
        e_min=res.e_min, e_max=res.e_max, n_bins=res.n_bins, eps_eff=res.eps_eff,
        early_terminated=bool(res.early_terminated),
        counts={k: int(res.counts[k]) for k in range(4)},
        abs_bound=abs_bound, rel_bound=rel_bound, abs_cap=2.0 * abs_bound,
        rel_guarantee=res.n_bins * res.eps_eff, rel_bound_plain=res.rel_bound_plain)


def hist(x, y):
    """Exponent-sum histogram over keys e+2148 and the zero-product count."""
    lib = load()
    x = _f64(x)
    y = _f64(y)
    counts = np.zeros(KEYS, dtype=np.int64)
    z = ctypes.c_int64(0)
    st = lib.or_hist(_ptr(x), _ptr(y), x.shape[0],
                     counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(z))
    if st == OR_ERR_NONFINITE:
        raise ValueError("inputs must be finite")
    return counts, int(z.value)


def exact_dot(x, y):
    """(value, flexp_e or None, plain) -- the reference_dot contract (kernel.py:98-133)."""
    lib = load()
    x = _f64(x)
    y = _f64(y)
    v = ctypes.c_double()
    fe = ctypes.c_int64()
    he = ctypes.c_int()
    pl = ctypes.c_double()
    st = lib.or_exact_dot(_ptr(x), _ptr(y), x.shape[0], ctypes.byref(v), ctypes.byref(fe),
                          ctypes.byref(he), ctypes.byref(pl))
    if st == OR_ERR_NONFINITE:
        raise ValueError("inputs must be finite")
    if st == OR_ERR_OVERFLOW:
        raise OverflowError("true dot product overflows double")
    return v.value, (fe.value if he.value else None), pl.value


def round_half(v: float) -> float:
    return load().or_round_half(float(v))


def round_single(v: float) -> float:
    return load().or_round_single(float(v))


def flexp(v: float) -> int:
    return int(load().or_flexp_export(float(v)))


def neumaier(values) -> float:
    a = _f64(values)
    return load().or_neumaier(_ptr(a), a.shape[0])


# ---------------------------------------------------------------- inputs
def gen_normal(n: int, seed: int = 0):
    """C1/C2 generator: default_rng(seed), x then y standard normal."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    y = rng.standard_normal(n)
    return x, y


def gen_illcond(n: int, seed: int = 0, mean_drop: float = 4.0, delta_bits: int = 25):
    """C3 generator (SURVEY.md §8d 'illcond2'): cond ~1e12, exponents spanning +-300."""
    rng = np.random.default_rng(seed)
    h = n // 2

    def drops():
        d = np.minimum(np.floor(rng.exponential(mean_drop, h)), 300).astype(np.int64)
        m = rng.random(h) < 1e-3
        d[m] = rng.integers(0, 301, int(m.sum()))
        return d

    a = drops()
    b = drops()
    sgn = rng.choice([-1.0, 1.0], h)
    x1 = sgn * np.ldexp(rng.uniform(0.5, 1.0, h), 150 - a)
    y1 = np.ldexp(rng.uniform(0.5, 1.0, h), 150 - b)
    delta = rng.uniform(-1.0, 1.0, h) * 2.0 ** -delta_bits
    x = np.concatenate([x1, x1])
    y = np.concatenate([y1, -y1 * (1.0 + delta)])
    perm = rng.permutation(2 * h)
    x = x[perm]
    y = y[perm]
    if n % 2:
        x = np.append(x, 1.0)
        y = np.append(y, 1.0)
    return x, y


def gen_family(family: str, t: float, n: int, seed: int):
    """Families A/B of the reference harness (harness.py:61-76), restated;
    `seed` is the final generator seed (the harness derives it per cell)."""
    rng = np.random.default_rng(seed)

    def sample():
        s = 0.5 + 0.5 * rng.random(n)
        if family == "A":
            half = int(t // 2)
            p = rng.integers(-half, half + 1, size=n)
        else:
            p = np.rint(rng.normal(0.0, 0.5 * t, size=n)).astype(np.int64)
        return np.ldexp(s, p)

    return sample(), sample()
