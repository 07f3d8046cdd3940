"""pytest plugin: the reference's OWN test suite against the B200 hot path.

    PYTHONPATH=tests/ref_suite python -m pytest -p qdot_b200_adapter baseline/_ref_tests

The unmodified reference package (baseline/_ref, qdot 0.1.0) is imported and
its hot-path entry points -- kernel.qdot, kernel.select_parameters,
kernel.reference_dot (kernel.py:34-72, 98-133, 179-240) -- are replaced, in
every reference module that bound them (kernel, harness, apps, cli), by thin
adapters over paper_2105_00115_b200.  That is the drop-in the B200 build
claims: the reference's callers (harness.run_trial, apps.acg / apm, the CLI)
and its tests run unchanged on top of the device pipeline.

The adapters translate types only: ToleranceConfig / strategy objects in,
QdotReport / ParameterSet / Bin / ReferenceResult of the reference's own
classes out (so `b.precision is PrecisionLevel.DOUBLE` and
simulate_qdot(x, y, rep.params) work); Bin.indices come from the device
counting-sort scatter.  No arithmetic happens here.

Tests that exercise reference internals off the hot path (floatbits,
binning, emulate, scoring helpers) still run against the reference's own
code; the B200 entry points are exercised by test_kernel, test_scoring
(select_parameters), test_acceptance, test_harness, test_apps and test_cli.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (REF, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import qdot as _R                                         # noqa: E402  the reference package
from qdot import apps as RA, binning as RB, cli as RC, harness as RH, kernel as RK, scoring as RS  # noqa: E402

import paper_2105_00115_b200 as Q                          # noqa: E402  the B200 build

if not os.path.abspath(_R.__file__).startswith(REF):
    raise ImportError(f"reference package resolved to {_R.__file__}, expected {REF}")

_LEVEL = {0: RS.PrecisionLevel.PERFORATE, 1: RS.PrecisionLevel.HALF, 2: RS.PrecisionLevel.SINGLE,
          3: RS.PrecisionLevel.DOUBLE}
CALLS = {"qdot": 0, "select_parameters": 0, "reference_dot": 0}


def _cfg(cfg):
    return Q.ToleranceConfig(epsilon=cfg.epsilon, split=Q.SplitMode(cfg.split.value), input_mu=cfg.input_mu)


def _strategy(s):
    if s is None:
        return None
    if isinstance(s, (RB.ExactBinning, RB.RangedBinning, RB.BinSplitting)):
        return Q.parse_strategy(RB.strategy_label(s))
    return s                                               # unknown object: the B200 qdot raises TypeError


def _params(ps, cfg, strategy):
    bins = [RB.Bin(lower=b.lower, upper=b.upper, indices=b.indices, score=b.score,
                   precision=_LEVEL[b.precision.code]) for b in ps.bins]
    return RS.ParameterSet(bins=bins, zero_idx=ps.zero_idx, e_min=ps.e_min, e_max=ps.e_max,
                           strategy=strategy if strategy is not None else RB.ExactBinning(), tolerance=cfg,
                           early_terminated=ps.early_terminated, n=ps.n, eps_eff=ps.eps_eff, n_bins=ps.n_bins,
                           rel_bound=ps.rel_bound)


def qdot(x, y, cfg, strategy=None, reference=None):
    """kernel.qdot (kernel.py:179-240) on the B200 path, reference types out."""
    CALLS["qdot"] += 1
    yy = x if y is x else y
    rep = Q.qdot(x, yy, _cfg(cfg), strategy=_strategy(strategy), reference=reference)
    counts = {lvl: 0 for lvl in RS.PrecisionLevel}
    for lvl, c in rep.counts.items():
        counts[_LEVEL[lvl.code]] = int(c)
    return RK.QdotReport(value=rep.value, counts=counts, abs_bound=rep.abs_bound, rel_bound=rep.rel_bound,
                         abs_cap=rep.abs_cap, rel_guarantee=rep.rel_guarantee, rel_hypothesis=rep.rel_hypothesis,
                         rel_bound_e=rep.rel_bound_e, early_terminated=rep.early_terminated, n=rep.n,
                         epsilon=rep.epsilon, split=cfg.split, strategy=rep.strategy, phase_ns=dict(rep.phase_ns),
                         params=_params(rep.params, cfg, strategy))


def select_parameters(x, y, cfg, strategy=None):
    """kernel.select_parameters (kernel.py:34-72) on the B200 path."""
    CALLS["select_parameters"] += 1
    yy = x if y is x else y
    ps = Q.select_parameters(x, yy, _cfg(cfg), strategy=_strategy(strategy))
    return _params(ps, cfg, strategy)


def reference_dot(x, y):
    """kernel.reference_dot (kernel.py:98-133) on the device exact dot."""
    CALLS["reference_dot"] += 1
    r = Q.reference_dot(x, y)
    return RK.ReferenceResult(value=r.value, flexp_e=r.flexp_e, plain=r.plain)


PATCHED = []
for _mod in (RK, RH, RA, RC, _R):
    for _name, _fn in (("qdot", qdot), ("select_parameters", select_parameters), ("reference_dot", reference_dot)):
        if hasattr(_mod, _name):
            setattr(_mod, _name, _fn)
            PATCHED.append(f"{_mod.__name__}.{_name}")


def pytest_report_header(config):
    return [f"qdot_b200_adapter: reference {REF} with B200 entry points: {', '.join(PATCHED)}"]


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    terminalreporter.write_line(f"qdot_b200_adapter: B200 entry-point calls {CALLS}")
