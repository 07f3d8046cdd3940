"""Solver callers, host side (no GPU): the matrix generators reproduce the
reference's CSR matrices exactly (checksums recorded from the reference by
tests/golden/make_apps_golden.py) and the reference's generator / trace KATs
(test_apps.py:15-70, 161-175)."""

import io

import numpy as np
import pytest

import apps_util as U
from paper_2105_00115_b200 import apps
from paper_2105_00115_b200.scoring import PrecisionLevel as P


@pytest.mark.parametrize("g", U.golden()["generators"], ids=lambda g: "-".join(map(str, g["spec"])))
def test_generator_matches_reference(g):
    a, rhs = U.matrix(g["spec"])
    m = a.csr()
    assert a.n == g["n"] and m.nnz == g["nnz"]
    assert U.sha(m.indptr.astype(np.int64)) == g["indptr"]
    assert U.sha(m.indices.astype(np.int64)) == g["indices"]
    assert U.sha(m.data) == g["data"]
    if "rhs" in g:
        assert U.sha(rhs) == g["rhs"]


def test_stencil_kats():
    a, rhs = apps.gen_stencil(1, 1, 1)
    assert a.csr().toarray().tolist() == [[27.0]] and rhs.tolist() == [27.0]
    a, rhs = apps.gen_stencil(2, 2, 1)
    dense = a.csr().toarray()
    assert np.all(np.diag(dense) == 27.0) and np.all((dense == -1).sum(axis=1) == 3)
    assert rhs.tolist() == [24.0] * 4
    center = apps.gen_stencil(3, 3, 1)[0].csr().toarray()[4]
    assert (center == -1).sum() == 8 and center[4] == 27.0
    assert np.linalg.eigvalsh(apps.gen_stencil(3, 3, 1)[0].csr().toarray()).min() > 0
    with pytest.raises(ValueError):
        apps.gen_stencil(0, 1, 1)


def test_laplacian_kats():
    assert apps.gen_graph_laplacian(2, 1.0).csr().toarray().tolist() == [[1.0, -1.0], [-1.0, 1.0]]
    assert apps.gen_graph_laplacian(4, 0.0).csr().nnz == 0
    eigs = sorted(np.linalg.eigvalsh(apps.gen_graph_laplacian(4, 1.0).csr().toarray()).round(9).tolist())
    assert eigs == [0.0, 4.0, 4.0, 4.0]
    a, b = apps.gen_graph_laplacian(60, 0.1, seed=5), apps.gen_graph_laplacian(60, 0.1, seed=5)
    assert (a.csr() != b.csr()).nnz == 0
    assert np.array_equal(apps.gen_graph_laplacian(50, 0.2, seed=1).csr() @ np.ones(50), np.zeros(50))
    with pytest.raises(ValueError):
        apps.gen_graph_laplacian(4, 1.5)
    with pytest.raises(ValueError):
        apps.gen_graph_laplacian(0, 0.5)


def test_trace_csv_schema():
    tr = apps.SolveTrace()

    class Rep:
        counts = {P.PERFORATE: 1, P.HALF: 0, P.SINGLE: 2, P.DOUBLE: 5}
        n = 8
    tr.record(0, "rtr", Rep(), 0.5)
    tr.record(1, "pAp", Rep(), 0.25)
    bufs = []
    for _ in range(2):
        b = io.StringIO()
        tr.write_csv(b)
        bufs.append(b.getvalue())
    assert bufs[0] == bufs[1]
    lines = bufs[0].splitlines()
    assert lines[0] == apps.TRACE_HEADER and len(lines) == 3
    assert lines[1] == "0,rtr,12.5,0.0,25.0,62.5,0.5"
    assert tr.rows[0].pct(P.DOUBLE) == 62.5


@pytest.mark.parametrize("kind", ["stencil", "ragged", "tail", "skewed", "empty_rows"])
def test_sell_layout_keeps_csr_row_order(kind):
    """The sliced-ELL copy the SpMV kernel reads (apps.sell_layout, run here on
    CPU tensors): every CSR entry lands at slice_off[r//32] + 32 j + r%32, and a
    sequential per-row sum over that layout (what k_sell_spmv does) equals
    scipy's csr_matvec byte for byte."""
    import scipy.sparse as sp
    import torch
    rng = np.random.default_rng(3)
    if kind == "stencil":
        m = apps.gen_stencil(6, 5, 4)[0].csr()
    else:
        n = {"ragged": 517, "tail": 33, "skewed": 700, "empty_rows": 96}[kind]
        lens = rng.integers(0, 9, n)
        if kind == "skewed":
            lens[::350] = 600
        if kind == "empty_rows":
            lens = rng.integers(6, 9, n)
            lens[::3] = 0
        indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        indices = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int32)
        data = rng.standard_normal(indptr[-1]) * np.exp2(rng.integers(-30, 30, indptr[-1]))
        m = sp.csr_matrix((data, indices, indptr), shape=(n, n))
    n = m.shape[0]
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt))  # noqa: E731
    out = apps.sell_layout(torch, t(m.indptr, np.int64), t(m.indices, np.int32), t(m.data, np.float64), n)
    lens = np.diff(m.indptr)
    ns = (n + 31) // 32
    width = np.pad(lens, (0, ns * 32 - n)).reshape(ns, 32).max(axis=1)
    too_padded = 32 * int(width.sum()) > 2 * m.nnz + 32 * ns
    if kind in ("skewed", "ragged", "stencil"):
        assert too_padded == (kind == "skewed")
    if too_padded:
        assert out is None                                   # padding > 2x: the CSR kernel serves it
        return
    so, rl, cols, vals = (o.numpy() for o in out)
    assert (rl == np.diff(m.indptr)).all()
    v = rng.standard_normal(n)
    y = np.empty(n)
    for r in range(n):
        base = so[r // 32] + (r % 32)
        s = 0.0
        for j in range(rl[r]):
            k = base + 32 * j
            assert cols[k] == m.indices[m.indptr[r] + j] and vals[k] == m.data[m.indptr[r] + j]
            s = s + vals[k] * v[cols[k]]
        y[r] = s
    assert y.tobytes() == (m @ v).tobytes()
