"""CPU-side checks of the C ABI library and the host-side mirror of the
reference interface (no GPU compute calls)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.scoring import PrecisionLevel as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "qdot_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(qdot_b200_\w+)\s*\(", src)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"binding missing for {s}"


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_workspace_layout():
    lay = _lib.layout()
    assert lay.total_bytes == _lib.load().qdot_b200_workspace_bytes()
    assert lay.a_len >= _lib.KEYS + 2 and lay.b_len >= 9 * _lib.KEYS
    assert lay.a_offset % 256 == 0 and lay.b_offset % 8 == 0
    assert lay.b_offset >= lay.a_offset + 8 * lay.a_len
    assert lay.result_offset >= lay.b_offset + 8 * lay.b_len


def _ldexp_c(v, u):
    o = ctypes.c_int(0)
    r = _lib.load().qdot_b200_ldexp_rn(v, u, ctypes.byref(o))
    return r, o.value


def test_ldexp_rn_matches_math_ldexp():
    rng = np.random.default_rng(0)
    vals = np.ldexp(rng.uniform(-2, 2, 3000), rng.integers(-60, 60, 3000))
    us = rng.integers(-1200, 1100, 3000)
    for v, u in zip(vals.tolist(), us.tolist()):
        try:
            want, wo = math.ldexp(v, u), 0
        except OverflowError:
            want, wo = math.copysign(math.inf, v), 1
        got, o = _ldexp_c(v, u)
        assert got == want and o == wo, (v, u)
    for v, u in [(1.5, -1074), (0.5, -1074), (2.5, -1075), (3.0, -1075), (1.0, 1023), (1.0, 1024), (0.0, 5000)]:
        try:
            want = math.ldexp(v, u)
        except OverflowError:
            want = math.inf
        assert _ldexp_c(v, u)[0] == want


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="only meaningful without a GPU")
def test_no_cpu_fallback():
    lib = _lib.load()
    assert lib.qdot_b200_device_info(None, None, None) == _lib.QDOT_ERR_CUDA
    with pytest.raises(RuntimeError):
        Q.qdot(np.ones(4), np.ones(4), Q.ToleranceConfig(1e-6))
    ws = ctypes.create_string_buffer(16)
    assert lib.qdot_b200_begin(ctypes.addressof(ws), None) == _lib.QDOT_ERR_CUDA


def test_config_validation_in_c():
    lib = _lib.load()
    c = _lib.QdotConfig(epsilon=0.0, split=0, input_mu=52, strategy=0, reserved=0, strategy_param=0)
    assert lib.qdot_b200_score(ctypes.c_void_p(1), 4, ctypes.byref(c), None) == _lib.QDOT_ERR_ARG
    c.epsilon = 1e-6
    c.input_mu = 17
    assert lib.qdot_b200_score(ctypes.c_void_p(1), 4, ctypes.byref(c), None) == _lib.QDOT_ERR_ARG
    c.input_mu = 52
    c.strategy = 1
    c.strategy_param = 0
    assert lib.qdot_b200_score(ctypes.c_void_p(1), 4, ctypes.byref(c), None) == _lib.QDOT_ERR_ARG


# ---- host mirror of the reference interface (scoring.py / binning.py KATs)
def test_tolerance_config_domain():
    with pytest.raises(ValueError):
        Q.ToleranceConfig(0.0)
    with pytest.raises(ValueError):
        Q.ToleranceConfig(math.inf)
    with pytest.raises(ValueError):
        Q.ToleranceConfig(2.0**61)
    with pytest.raises(ValueError):
        Q.ToleranceConfig(1e-3, input_mu=17)
    assert Q.ToleranceConfig(2**60).epsilon == 2.0**60


@pytest.mark.parametrize("score,want", [
    (35, P.DOUBLE), (2, P.HALF), (-11, P.PERFORATE), (-21, P.PERFORATE), (15, P.SINGLE), (100, P.DOUBLE),
    (0, P.HALF), (9, P.HALF), (10, P.SINGLE), (22, P.SINGLE), (23, P.DOUBLE), (52, P.DOUBLE), (-1, P.PERFORATE)])
def test_precision_of_table(score, want):
    # test_scoring.py:62-78
    assert Q.precision_of(score, 52) is want


def test_scores_and_helpers():
    eps = 2.0**-34
    assert [Q.bin_score(1, u, 50, eps) for u in (50, 17, 4, -6)] == [35, 2, -11, -21]
    assert [Q.ceil_log2(m) for m in (1, 2, 3, 4, 5, 1024, 1025)] == [0, 1, 2, 2, 3, 10, 11]
    assert Q.floor_log2(2.0**-34) == -34 and Q.floor_log2(0.5) == -1
    assert Q.precision_of(30, 23) is P.SINGLE and Q.precision_of(12, 10) is P.HALF
    assert Q.early_termination(0, 0, 52, 2.0**-34)


def test_strategy_parsing_and_labels():
    assert isinstance(Q.parse_strategy("exact"), Q.ExactBinning)
    assert Q.parse_strategy("ranged:3").width == 3
    assert Q.parse_strategy("split:2").levels == 2
    with pytest.raises(ValueError):
        Q.parse_strategy("foo")
    with pytest.raises(ValueError):
        Q.RangedBinning(0)
    with pytest.raises(ValueError):
        Q.BinSplitting(-1)
    assert Q.strategy_label(Q.RangedBinning(4)) == "ranged:4"
    from paper_2105_00115_b200.binning import strategy_code
    with pytest.raises(TypeError):
        strategy_code(object())
    assert strategy_code(None) == (_lib.STRATEGY_EXACT, 0)
    assert strategy_code(Q.BinSplitting(3)) == (_lib.STRATEGY_SPLIT, 3)


def test_precision_codes_match_c_enum():
    assert [p.code for p in (P.PERFORATE, P.HALF, P.SINGLE, P.DOUBLE)] == [0, 1, 2, 3]
    assert P.from_code(3) is P.DOUBLE and P.HALF.eps == 2.0**-10


def test_enums_interoperate_with_reference_style_enums():
    import enum

    class RefLevel(enum.Enum):          # same shape as qdot.scoring.PrecisionLevel
        PERFORATE = ("perforate", 0)
        HALF = ("half", 10)
        SINGLE = ("single", 23)
        DOUBLE = ("double", 52)

        def __init__(self, label, mantissa_bits):
            self.label = label
            self.mantissa_bits = mantissa_bits

    class RefSplit(enum.Enum):
        NONE = "none"
        PER_BIN = "per-bin"

    counts = {lvl: i for i, lvl in enumerate(P)}
    assert counts[RefLevel.DOUBLE] == counts[P.DOUBLE]
    assert P.HALF == RefLevel.HALF and P.HALF != RefLevel.SINGLE
    assert Q.SplitMode.PER_BIN == RefSplit.PER_BIN
    cfg = Q.ToleranceConfig(1e-3, split=RefSplit.PER_BIN)
    from paper_2105_00115_b200.device import config_struct
    assert config_struct(cfg, None).split == 1


def test_bound_sums_match_fsum():
    """qdot_b200_bound_sums (host code, no GPU) equals math.fsum and the plain
    left-to-right sum of the reference's bound terms (scoring.py:171-199),
    including ldexp underflow, and raises where math.ldexp overflows."""
    import ctypes
    import math
    import random

    from paper_2105_00115_b200 import _lib
    lib = _lib.load(build_if_missing=False)
    mus = [0, 10, 23, 52]
    out = (ctypes.c_double * 2)()
    rnd = random.Random(7)
    for trial in range(1500):
        nb = rnd.randint(0, 50)
        arr = (_lib.QdotBin * max(nb, 1))()
        shift = rnd.randint(-60, 60)
        terms = []
        for i in range(nb):
            b = arr[i]
            b.cardinality = rnd.choice([1, 2, 3, rnd.randint(1, 1 << 40)])
            b.precision = rnd.randint(0, 3)
            b.upper = rnd.randint(-1200, 1000) if trial % 3 == 0 else rnd.randint(-60, 60)
            try:
                terms.append(float(b.cardinality) * math.ldexp(math.ldexp(1.0, -mus[b.precision]),
                                                               b.upper - shift + 1))
            except OverflowError:
                terms = None
                break
        rc = lib.qdot_b200_bound_sums(arr, nb, shift, out)
        if terms is None:
            assert rc == _lib.QDOT_ERR_OVERFLOW
            continue
        plain = 0.0
        for t in terms:
            plain += t
        try:
            f = math.fsum(terms)
        except OverflowError:
            assert rc == _lib.QDOT_ERR_OVERFLOW
            continue
        assert rc == 0
        assert out[0] == f and out[1] == plain, (trial, out[0], f, out[1], plain)


def test_bound_sums2_equals_two_calls():
    """qdot_b200_bound_sums2 (the report's rel terms at e_max, then abs at 0, in
    one call) returns exactly what two qdot_b200_bound_sums calls return, and the
    first failing shift's status."""
    import ctypes
    import random

    from paper_2105_00115_b200 import _lib
    lib = _lib.load(build_if_missing=False)
    rnd = random.Random(11)
    for trial in range(800):
        nb = rnd.randint(0, 40)
        arr = (_lib.QdotBin * max(nb, 1))()
        for i in range(nb):
            b = arr[i]
            b.cardinality = rnd.choice([1, 5, rnd.randint(1, 1 << 40)])
            b.precision = rnd.randint(0, 3)
            b.upper = rnd.randint(-1100, 1030) if trial % 4 == 0 else rnd.randint(-60, 60)
        sa, sb = rnd.randint(-70, 70), rnd.choice([0, rnd.randint(-70, 70)])
        two = (ctypes.c_double * 4)()
        ra = lib.qdot_b200_bound_sums(arr, nb, sa, two)
        rb = lib.qdot_b200_bound_sums(arr, nb, sb, ctypes.cast(ctypes.addressof(two) + 16, ctypes.POINTER(ctypes.c_double)))
        one = (ctypes.c_double * 4)()
        r = lib.qdot_b200_bound_sums2(arr, nb, sa, sb, one)
        assert r == (ra if ra else rb)
        if r == 0:
            assert list(one) == list(two)
