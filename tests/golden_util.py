"""Loader for the committed golden vectors (tests/golden/, made by
tests/golden/make_golden.py from the reference package itself)."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PREC_LABEL = {0: "perforate", 1: "half", 2: "single", 3: "double"}


@functools.lru_cache(maxsize=1)
def cases():
    with open(os.path.join(GOLDEN, "golden_cases.json")) as f:
        return json.load(f)["cases"]


@functools.lru_cache(maxsize=1)
def _npz():
    return dict(np.load(os.path.join(GOLDEN, "golden_inputs.npz")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:16]


@functools.lru_cache(maxsize=8)
def _regen(name):
    from oracle.oracle import gen_illcond, gen_normal
    if name.startswith("C1"):
        return gen_normal(1 << 20, seed=0)
    if name.startswith("C3"):
        return gen_illcond(1 << 20, seed=0)
    if name.startswith("half_seq"):
        rng = np.random.default_rng(21)
        return np.abs(rng.standard_normal(1 << 18)), np.abs(rng.standard_normal(1 << 18))
    raise KeyError(name)


def inputs(case):
    """(x, y) for a golden case; regenerated large inputs are checksum-verified."""
    if case["stored"]:
        z = _npz()
        x = z[case["input"] + "__x"]
        y = z[case["input"] + "__y"]
    else:
        x, y = _regen(case["name"])
    if case["norm"]:
        y = x
    assert _sha(x) == case["x_sha"] and _sha(y) == case["y_sha"], "generator drift"
    return x, y


def hexf(s):
    return float.fromhex(s)


def select(pred=None, max_n=None):
    out = []
    for c in cases():
        if max_n is not None and c["n"] > max_n:
            continue
        if pred is None or pred(c):
            out.append(c)
    return out


def members_sha(zero_idx, bin_indices) -> str:
    """Digest of the member order (make_golden.members_sha): zero_idx, then
    each bin's indices, as int64."""
    h = hashlib.sha256(np.ascontiguousarray(zero_idx, dtype=np.int64).tobytes())
    for ind in bin_indices:
        h.update(b"|")
        h.update(np.ascontiguousarray(ind, dtype=np.int64).tobytes())
    return h.hexdigest()[:16]
