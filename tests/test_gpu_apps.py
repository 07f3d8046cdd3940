"""GPU solvers (ACG / APM) against the reference, bit for bit.

Every golden case (tests/golden/apps_golden.json, recorded by running the
reference's apps.acg / apps.apm) must be reproduced exactly: iteration count,
convergence, final residual / eigenvalue, the returned iterate, every trace
row (precision counts, residual) and the trace CSV.  Also the reference's own
solver KATs (test_apps.py:73-158) and the SpMV against scipy."""

import io
import hashlib
import math

import numpy as np
import pytest
import scipy.sparse as sp

import apps_util as U

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2105_00115_b200 import apps  # noqa: E402
from paper_2105_00115_b200.scoring import PrecisionLevel as P  # noqa: E402

LEVELS = [P.PERFORATE, P.HALF, P.SINGLE, P.DOUBLE]


def rows(tr):
    return [[r.iteration, r.call_site, [int(r.counts.get(lv, 0)) for lv in LEVELS], r.n,
             float(r.resid_or_lambda).hex()] for r in tr.rows]


def csv_sha(tr):
    b = io.StringIO()
    tr.write_csv(b)
    return hashlib.sha256(b.getvalue().encode()).hexdigest()[:16]


@pytest.fixture(params=["eager", "graph"])
def iteration_mode(request, monkeypatch):
    # "graph": every solve, however small, runs its iterations as CUDA graphs
    if request.param == "graph":
        monkeypatch.setattr(apps, "GRAPH_MIN", 1)
    else:
        monkeypatch.setattr(apps, "GRAPH_MIN", 1 << 62)
        monkeypatch.setattr(apps, "GRAPH_REPEAT", False)
    return request.param


@pytest.mark.parametrize("case", U.golden()["cg"], ids=lambda c: c["name"])
def test_acg_golden(case, iteration_mode):
    a, rhs = U.matrix(case["matrix"])
    bspec = case["opts"].get("b")
    b = rhs if bspec is None else {"arange": np.arange(1.0, a.n + 1.0), "zeros": np.zeros(a.n),
                                   "ones": np.ones(a.n)}[bspec]
    assert U.sha(b) == case["b_sha"]
    x0 = U.x0_for(case["x0"], a.n)
    kw = U.kwargs(case["opts"])
    if case["raises"]:
        with pytest.raises(getattr(apps, case["raises"])):
            apps.acg(a, b, x0=x0, **kw)
        return
    res = apps.acg(a, b, x0=x0, **kw)
    assert res.iterations == case["iterations"] and res.converged == case["converged"]
    assert float(res.residual_norm).hex() == case["residual_norm"]
    assert rows(res.trace) == case["trace"]
    assert U.sha(res.x) == case["x_sha"]
    assert csv_sha(res.trace) == case["trace_csv_sha"]


@pytest.mark.parametrize("case", U.golden()["pm"], ids=lambda c: c["name"])
def test_apm_golden(case, iteration_mode):
    a, _ = U.matrix(case["matrix"])
    x0 = U.x0_for(case["x0"], a.n)
    assert U.sha(x0) == case["x0_sha"]
    kw = U.kwargs(case["opts"])
    if case["raises"]:
        with pytest.raises(getattr(apps, case["raises"])):
            apps.apm(a, x0, **kw)
        return
    res = apps.apm(a, x0, **kw)
    assert res.iterations == case["iterations"] and res.converged == case["converged"]
    assert float(res.eigenvalue).hex() == case["eigenvalue"]
    assert rows(res.trace) == case["trace"]
    assert U.sha(res.x) == case["x_sha"]
    assert csv_sha(res.trace) == case["trace_csv_sha"]


@pytest.mark.parametrize("shape,density,seed", [((1, 1), 1.0, 0), ((300, 300), 0.05, 1), ((5000, 5000), 0.002, 2),
                                                ((64, 64), 0.0, 3)])
def test_spmv_bitwise_scipy(shape, density, seed):
    rng = np.random.default_rng(seed)
    m = sp.random(*shape, density=density, random_state=seed, format="csr",
                  data_rvs=lambda k: rng.standard_normal(k) * np.exp2(rng.integers(-40, 40, k)))
    m.sort_indices()
    a = apps.SparseMatrix.from_csr(m, symmetric=False)
    for v in (rng.standard_normal(shape[1]), np.where(rng.random(shape[1]) < 0.3, -0.0, rng.standard_normal(shape[1]))):
        got = a.matvec(v)
        want = m @ v
        assert got.tobytes() == want.tobytes()
    # int64 column indices take the same path
    m64 = sp.csr_matrix((m.data, m.indices.astype(np.int64), m.indptr.astype(np.int64)), shape=shape)
    a64 = apps.SparseMatrix(indptr=m64.indptr, indices=m64.indices, data=m64.data, n=shape[0], symmetric=False)
    v = rng.standard_normal(shape[1])
    assert a64.matvec(v).tobytes() == (m @ v).tobytes()


def _ragged_csr(n, lens, seed):
    rng = np.random.default_rng(seed)
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    indices = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int32)
    data = rng.standard_normal(indptr[-1]) * np.exp2(rng.integers(-30, 30, indptr[-1]))
    return sp.csr_matrix((data, indices, indptr), shape=(n, n))


@pytest.mark.parametrize("kind", ["ragged", "skewed", "tail"])
def test_spmv_sliced_ell_vs_csr(kind):
    """The sliced-ELL kernel (used when padding stays under 2x) and the CSR
    kernel (the fallback) both equal scipy bit for bit on ragged rows, empty
    rows and a row count that is not a multiple of the 32-row slice."""
    rng = np.random.default_rng(11)
    n = {"ragged": 1037, "skewed": 2000, "tail": 33}[kind]
    lens = rng.integers(0, 9, n)
    if kind == "skewed":
        lens[::500] = 900                                   # padding blows past 2x -> CSR
    m = _ragged_csr(n, lens, 12)
    a = apps.SparseMatrix.from_csr(m, symmetric=False)
    assert (a.sell_arrays() is None) == (kind == "skewed")
    v = rng.standard_normal(n)
    assert a.matvec(v).tobytes() == (m @ v).tobytes()
    a._sell = False                                         # force the CSR kernel on the same matrix
    assert a.matvec(v).tobytes() == (m @ v).tobytes()


def test_vector_updates_match_numpy():
    rng = np.random.default_rng(5)
    a, b = rng.standard_normal(100001), rng.standard_normal(100001)
    s = 0.7318273645123
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out = torch.empty_like(ad)
    for op, want in ((0, a + s * b), (1, a - s * b), (2, a / s)):
        apps._update(op, ad, s, bd if op != 2 else None, out)
        assert out.cpu().numpy().tobytes() == want.tobytes()


def identity(n):
    return apps.SparseMatrix.from_csr(sp.eye(n, format="csr"))


def test_reference_solver_kats():
    res = apps.acg(identity(12), np.arange(1.0, 13.0), tau=1e-10, epsilon=0.5)
    assert res.iterations == 1 and res.converged
    a, b = apps.gen_stencil(20, 20, 1)
    ref = apps.reference_cg(a, b, tau=1e-8)
    approx = apps.acg(a, b, tau=1e-8, epsilon=2.0 ** -58)
    assert approx.iterations == ref.iterations and approx.converged and ref.converged
    assert np.allclose(approx.x, np.ones(a.n), atol=1e-6)
    a, b = apps.gen_stencil(8, 8, 1)
    res = apps.acg(a, b, tau=1e-8, epsilon=1e-6)
    assert {r.call_site for r in res.trace.rows} == {"rtr", "pAp"}
    for row in res.trace.rows:
        assert sum(row.pct(lv) for lv in P) == pytest.approx(100.0)
    with pytest.raises(ValueError):
        apps.acg(apps.SparseMatrix.from_csr(sp.eye(3, format="csr"), symmetric=False), np.ones(3))
    lap = apps.gen_graph_laplacian(200, 0.05, seed=3)
    x0 = np.random.default_rng(4).standard_normal(200)
    x0 /= np.linalg.norm(x0)
    approx = apps.apm(lap, x0, tau=1e-6, epsilon=1e-7, max_iters=300)
    plain = apps.reference_pm(lap, x0, tau=1e-6, max_iters=300)
    assert abs(approx.eigenvalue - plain.eigenvalue) <= 1e-6
    with pytest.raises(apps.ZeroIterateError):
        apps.apm(identity(3), np.zeros(3))
    lap4 = apps.gen_graph_laplacian(4, 1.0)
    res = apps.apm(lap4, np.random.default_rng(0).standard_normal(4), tau=1e-6, epsilon=1e-7)
    assert abs(res.eigenvalue - 4.0) <= 1e-6 and res.converged


def test_large_stencil_runs_on_device():
    # a 64^3 stencil (262,144 unknowns): converges to the all-ones solution
    a, b = apps.gen_stencil(64, 64, 64)
    res = apps.acg(a, b, tau=1e-6, epsilon=1e-8)
    assert res.converged and math.isfinite(res.residual_norm)
    assert np.abs(res.x - 1.0).max() < 1e-6


def _same_cg(r1, r2):
    return (r1.iterations == r2.iterations and r1.x.tobytes() == r2.x.tobytes()
            and float(r1.residual_norm).hex() == float(r2.residual_norm).hex() and rows(r1.trace) == rows(r2.trace))


def test_repeated_solves_replay_the_cached_graph():
    """A second solve on the same matrix replays the captured iteration graph
    with new b / x0 (and new start vectors for APM): every result equals a
    solve on a fresh matrix object, also with two threads solving at once."""
    import threading
    a, b = apps.gen_stencil(16, 16, 12)                   # n = 3072 >= GRAPH_MIN
    rng = np.random.default_rng(9)
    rhs = [b, rng.standard_normal(a.n), rng.standard_normal(a.n)]
    x0s = [None, None, rng.standard_normal(a.n)]
    fresh = [apps.acg(apps.SparseMatrix.from_csr(a.csr()), bb, x0=xx, tau=1e-8, epsilon=1e-8)
             for bb, xx in zip(rhs, x0s)]
    for _ in range(2):
        for bb, xx, want in zip(rhs, x0s, fresh):
            assert _same_cg(apps.acg(a, bb, x0=xx, tau=1e-8, epsilon=1e-8), want)
    out = [None, None]

    def solve(i):
        out[i] = apps.acg(a, rhs[i + 1], x0=x0s[i + 1], tau=1e-8, epsilon=1e-8)
    ts = [threading.Thread(target=solve, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert _same_cg(out[0], fresh[1]) and _same_cg(out[1], fresh[2])

    small, sb = apps.gen_stencil(8, 8, 8)                   # n = 512 < GRAPH_MIN: eager, then a graph
    sfresh = apps.acg(apps.SparseMatrix.from_csr(small.csr()), sb, tau=1e-8, epsilon=1e-8)
    for _ in range(3):
        assert _same_cg(apps.acg(small, sb, tau=1e-8, epsilon=1e-8), sfresh)

    lap = apps.gen_graph_laplacian(3000, 0.003, seed=5)
    starts = [rng.standard_normal(lap.n) for _ in range(3)]
    pf = [apps.apm(apps.SparseMatrix.from_csr(lap.csr()), s0, tau=1e-6, epsilon=1e-7, max_iters=60) for s0 in starts]
    for _ in range(2):
        for s0, want in zip(starts, pf):
            got = apps.apm(lap, s0, tau=1e-6, epsilon=1e-7, max_iters=60)
            assert got.iterations == want.iterations and got.x.tobytes() == want.x.tobytes()
            assert float(got.eigenvalue).hex() == float(want.eigenvalue).hex()
            assert rows(got.trace) == rows(want.trace)
