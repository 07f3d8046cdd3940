"""Shared helpers for the solver tests: rebuild the inputs of a golden case
(tests/golden/apps_golden.json, made by make_apps_golden.py from the reference)."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np
import scipy.sparse as sp

from paper_2105_00115_b200 import apps
from paper_2105_00115_b200.binning import BinSplitting, ExactBinning, RangedBinning
from paper_2105_00115_b200.scoring import SplitMode

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "apps_golden.json")


@functools.lru_cache(maxsize=1)
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def matrix(spec):
    kind = spec[0]
    if kind == "stencil":
        return apps.gen_stencil(*spec[1:4])
    if kind == "laplacian":
        return apps.gen_graph_laplacian(*spec[1:4]), None
    if kind == "scaled_eye":
        return apps.SparseMatrix.from_csr((spec[2] * sp.eye(spec[1])).tocsr()), None
    raise KeyError(kind)


def x0_for(spec, n):
    if spec is None:
        return None
    kind = spec[0]
    if kind == "e":
        v = np.zeros(n)
        v[spec[1]] = 1.0
        return v
    if kind == "normal":
        v = np.random.default_rng(spec[1]).standard_normal(n)
        if len(spec) > 2 and spec[2] == "unit":
            v /= np.linalg.norm(v)
        return v
    if kind == "ones":
        return np.ones(n)
    raise KeyError(kind)


def strat(s):
    head, _, arg = s.partition(":")
    return {"exact": lambda: ExactBinning(), "ranged": lambda: RangedBinning(int(arg)),
            "split": lambda: BinSplitting(int(arg))}[head]()


def kwargs(opts):
    out = {}
    for k, v in opts.items():
        if k in ("b", "x0"):
            continue
        if k == "split":
            out["split"] = SplitMode.NONE if v == "none" else SplitMode.PER_BIN
        elif k == "strategy":
            out["strategy"] = strat(v)
        elif k == "epsilon":
            out["epsilon"] = float.fromhex(v)
        else:
            out[k] = v
    return out
