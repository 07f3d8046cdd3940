"""Golden solver runs (ACG / APM) and generator checksums BY RUNNING THE REFERENCE.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_apps_golden.py

Imports the unmodified reference (qdot 0.1.0, apps.py) and records, per
case, everything the device solvers must reproduce bit for bit: iteration
count, convergence flag, final residual / eigenvalue (hex), a checksum of the
returned iterate, and every trace row (site, precision counts, residual).
Also records CSR / rhs checksums of the reference generators.  The GPU box
never reads /root/reference: the tests consume only apps_golden.json.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from qdot import apps as R  # noqa: E402
from qdot.binning import BinSplitting, ExactBinning, RangedBinning  # noqa: E402
from qdot.scoring import PrecisionLevel, SplitMode  # noqa: E402

LEVELS = [PrecisionLevel.PERFORATE, PrecisionLevel.HALF, PrecisionLevel.SINGLE, PrecisionLevel.DOUBLE]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def strat(s):
    head, _, arg = s.partition(":")
    return {"exact": lambda: ExactBinning(), "ranged": lambda: RangedBinning(int(arg)),
            "split": lambda: BinSplitting(int(arg))}[head]()


def matrix(spec):
    kind = spec[0]
    if kind == "stencil":
        a, b = R.gen_stencil(*spec[1:4])
        return a, b
    if kind == "laplacian":
        return R.gen_graph_laplacian(*spec[1:4]), None
    if kind == "scaled_eye":
        return R.SparseMatrix.from_csr((spec[2] * sp.eye(spec[1])).tocsr()), None
    raise KeyError(kind)


def trace_rows(tr):
    return [[r.iteration, r.call_site, [int(r.counts.get(lv, 0)) for lv in LEVELS], r.n,
             float(r.resid_or_lambda).hex()] for r in tr.rows]


def trace_csv_sha(tr):
    buf = io.StringIO()
    tr.write_csv(buf)
    return hashlib.sha256(buf.getvalue().encode()).hexdigest()[:16]


def x0_for(spec, n):
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


CG_CASES = [
    ("cg_stencil_8x8x1_eps1e-6", ("stencil", 8, 8, 1), dict(tau=1e-8, epsilon=1e-6)),
    ("cg_stencil_20x20x1_eps2m58", ("stencil", 20, 20, 1), dict(tau=1e-8, epsilon=2.0 ** -58)),
    ("cg_stencil_6x6x1_eps2m58", ("stencil", 6, 6, 1), dict(tau=1e-8, epsilon=2.0 ** -58)),
    ("cg_stencil_5x5x1_eps1e-4", ("stencil", 5, 5, 1), dict(tau=1e-8, epsilon=1e-4)),
    ("cg_stencil_6x6x6_eps1e-8", ("stencil", 6, 6, 6), dict(tau=1e-8, epsilon=1e-8)),
    ("cg_stencil_12x12x12_eps1e-5_none", ("stencil", 12, 12, 12),
     dict(tau=1e-9, epsilon=1e-5, split="none")),
    ("cg_stencil_10x10x4_eps1e-3_ranged2", ("stencil", 10, 10, 4), dict(tau=1e-8, epsilon=1e-3, strategy="ranged:2")),
    ("cg_stencil_10x10x4_eps1e-6_split3", ("stencil", 10, 10, 4), dict(tau=1e-8, epsilon=1e-6, strategy="split:3")),
    ("cg_identity12", ("scaled_eye", 12, 1.0), dict(tau=1e-10, epsilon=0.5, b="arange")),
    ("cg_zero_rhs", ("scaled_eye", 4, 1.0), dict(tau=1e-10, epsilon=1e-8, b="zeros")),
    ("cg_breakdown", ("scaled_eye", 5, -1.0), dict(tau=1e-10, epsilon=1e-10, b="ones")),
    ("cg_stencil_16x16x16_eps1e-7_x0", ("stencil", 16, 16, 16), dict(tau=1e-7, epsilon=1e-7, x0=("normal", 9))),
]

PM_CASES = [
    ("pm_two_identity", ("scaled_eye", 8, 2.0), ("e", 0), dict(tau=1e-6, epsilon=1.0)),
    ("pm_complete4", ("laplacian", 4, 1.0, 0), ("normal", 0), dict(tau=1e-6, epsilon=1e-7)),
    ("pm_laplacian200", ("laplacian", 200, 0.05, 3), ("normal", 4, "unit"),
     dict(tau=1e-6, epsilon=1e-7, max_iters=300)),
    ("pm_laplacian500_none", ("laplacian", 500, 0.02, 7), ("normal", 5),
     dict(tau=1e-8, epsilon=1e-5, split="none", max_iters=200)),
    ("pm_zero_iterate", ("laplacian", 4, 1.0, 0), ("ones",), dict(tau=1e-6, epsilon=1e-7)),
    ("pm_trace_sites", ("scaled_eye", 4, 2.0), ("e", 1), dict(tau=1e-9, epsilon=0.5)),
]


def kw(opts):
    out = {}
    for k, v in opts.items():
        if k in ("b", "x0"):
            continue
        if k == "split":
            out["split"] = SplitMode.NONE if v == "none" else SplitMode.PER_BIN
        elif k == "strategy":
            out["strategy"] = strat(v)
        else:
            out[k] = v
    return out


def main():
    out = {"cg": [], "pm": [], "generators": []}
    for name, mspec, opts in CG_CASES:
        a, rhs = matrix(mspec)
        bspec = opts.get("b")
        b = rhs if bspec is None else {"arange": np.arange(1.0, a.n + 1.0), "zeros": np.zeros(a.n),
                                       "ones": np.ones(a.n)}[bspec]
        x0 = x0_for(opts["x0"], a.n) if "x0" in opts else None
        case = {"name": name, "matrix": mspec, "opts": {k: v for k, v in opts.items() if k != "x0"},
                "x0": opts.get("x0"), "b_sha": sha(b)}
        if "epsilon" in case["opts"]:
            case["opts"]["epsilon"] = float(opts["epsilon"]).hex()
        try:
            res = R.acg(a, b, x0=x0, **kw(opts))
            case.update(raises=None, iterations=res.iterations, converged=res.converged,
                        residual_norm=float(res.residual_norm).hex(), x_sha=sha(res.x),
                        trace=trace_rows(res.trace), trace_csv_sha=trace_csv_sha(res.trace))
        except Exception as exc:  # noqa: BLE001 - record the reference's exception type
            case.update(raises=type(exc).__name__)
        out["cg"].append(case)
        print(name, case.get("iterations"), case.get("raises"))
    for name, mspec, xspec, opts in PM_CASES:
        a, _ = matrix(mspec)
        x0 = x0_for(xspec, a.n)
        case = {"name": name, "matrix": mspec, "x0": xspec, "opts": dict(opts), "x0_sha": sha(x0)}
        case["opts"]["epsilon"] = float(opts["epsilon"]).hex()
        try:
            res = R.apm(a, x0, **kw(opts))
            case.update(raises=None, iterations=res.iterations, converged=res.converged,
                        eigenvalue=float(res.eigenvalue).hex(), x_sha=sha(res.x), trace=trace_rows(res.trace),
                        trace_csv_sha=trace_csv_sha(res.trace))
        except Exception as exc:  # noqa: BLE001
            case.update(raises=type(exc).__name__)
        out["pm"].append(case)
        print(name, case.get("iterations"), case.get("raises"))
    for spec in [("stencil", 1, 1, 1), ("stencil", 2, 2, 1), ("stencil", 4, 3, 2), ("stencil", 7, 5, 3),
                 ("laplacian", 2, 1.0, 0), ("laplacian", 4, 0.0, 0), ("laplacian", 60, 0.1, 5),
                 ("laplacian", 200, 0.05, 3), ("laplacian", 500, 0.02, 7)]:
        a, rhs = matrix(spec)
        m = a.csr()
        g = {"spec": spec, "indptr": sha(m.indptr.astype(np.int64)), "indices": sha(m.indices.astype(np.int64)),
             "data": sha(m.data), "nnz": int(m.nnz), "n": a.n}
        if rhs is not None:
            g["rhs"] = sha(rhs)
        out["generators"].append(g)
    with open(os.path.join(HERE, "apps_golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
