"""Iterative-solver callers of qdot, on the device: approximate CG (acg) and
the approximate power method (apm).

Mirrors the reference's apps.py (apps.py:1-359): same names, signatures,
result types, trace schema and exceptions.  Underneath, every vector lives in
HBM and every operation runs in this package's sm_100a kernels:

    A.matvec(p)         qdot_b200_csr_spmv   (bit-identical to scipy csr_matvec)
    x + alpha*p, ...    qdot_b200_vec_update (bit-identical to the numpy expression)
    r.r, p.Ap, ...      the qdot device pipeline (bit-identical to kernel.qdot)

so iterates, iteration counts, residuals and precision traces equal the
reference's bit for bit.  Host work per iteration is the scalar recurrence
(alpha = c/d, beta, sqrt) in Python floats, exactly as the reference does it.

The generators (gen_stencil, gen_graph_laplacian) build the same CSR matrices
as the reference on the host; they are input preparation, not the hot path.
reference_cg / reference_pm are the plain-double baselines (torch on the
device), kept for iteration-count comparisons like the reference's.

Solves with at least GRAPH_MIN unknowns run their iterations on the device:
one CUDA graph whose WHILE-conditional node repeats a captured iteration
(SpMV, both qdot pipelines, fused kernels for the scalar recurrence -- alpha,
beta, sqrt, lambda with IEEE division / square root / product, i.e. the
Python float values -- and the vector updates) and ends with a check kernel
that records the iteration (both qdot result headers and the scalars) and
stops the loop where the host loop would; the host parses the records once
per solve, raises the same errors and builds the same trace.
"""

from __future__ import annotations

import csv
import ctypes
import math
import threading
from dataclasses import dataclass, field
from typing import IO, List, Optional, Tuple, Union

import numpy as np
import scipy.sparse as sp

from . import _lib
from .binning import ExactBinning, Strategy, strategy_label
from .device import config_struct, require_cuda, stream_handle, thread_state
from .kernel import _raise_status, run_device
from .scoring import LEVELS_ASC, PrecisionLevel, SplitMode, ToleranceConfig

__all__ = ["TRACE_HEADER", "BreakdownError", "ZeroIterateError", "SparseMatrix", "gen_stencil",
           "gen_graph_laplacian", "TraceRow", "SolveTrace", "CGResult", "PMResult", "acg", "apm",
           "reference_cg", "reference_pm"]

TRACE_HEADER = "iter,call_site,pct_perforate,pct_half,pct_single,pct_double,resid_or_lambda"   # apps.py:22

_ADD, _SUB, _DIV = 0, 1, 2


class BreakdownError(RuntimeError):
    """CG direction lost positive curvature (p.Ap <= 0 or non-finite)."""


class ZeroIterateError(RuntimeError):
    """Power-method iterate collapsed to the zero vector."""


# --------------------------------------------------------------------------- device helpers
def _dev():
    torch = require_cuda()
    return torch, torch.device("cuda", torch.cuda.current_device())


def _to_device(v, n: Optional[int] = None):
    torch, device = _dev()
    if isinstance(v, torch.Tensor):
        t = v.to(device=device, dtype=torch.float64).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(device)
    if t.dim() != 1 or (n is not None and t.shape[0] != n):
        raise ValueError(f"expected a 1-D vector of length {n}")
    return t


def _update(op: int, a, s: float, b, out) -> None:
    """out = a + s*b | a - s*b | a / s on the device (numpy rounding)."""
    lib = _lib.load()
    _lib.check(lib.qdot_b200_vec_update(a.shape[0], op, a.data_ptr(), float(s),
                                        b.data_ptr() if b is not None else None, out.data_ptr(),
                                        stream_handle(a.device)), lib)


class _Dots:
    """qdot calls of one solver run: the device pipeline with a reused
    workspace, returning what the solvers and their traces consume."""

    def __init__(self, cfg: ToleranceConfig, strategy):
        self.cfg, self.strategy = cfg, strategy

    def __call__(self, xd, yd, norm: bool):
        n = int(xd.shape[0])
        res, _, _ = run_device(xd, xd if norm else yd, n, norm, self.cfg, self.strategy, timing=False)
        _raise_status(res)
        counts = {level: int(res.counts[i]) for i, level in enumerate(LEVELS_ASC)}
        return _DotReport(float(res.value), counts, n, int(res.zero_count))


@dataclass
class _DotReport:
    """The QdotReport fields a solver trace reads (value, counts, n)."""

    value: float
    counts: dict
    n: int
    zero_count: int


# --------------------------------------------------------------------------- matrices
def sell_layout(torch, indptr, indices, data, n):
    """CSR -> sliced ELL on the tensors' device: slices of 32 rows, entry j of
    row r at slice_off[r // 32] + 32 j + r % 32 (a warp's 32 rows read one
    coalesced line per j).  Returns (slice_off int64[ns], row_len int32[n],
    cols int32[total], vals f64[total]) or None (no rows or entries, n >= 2^31,
    or padding above 2x).  The order of a row's entries is kept, so a
    sequential per-row sum equals scipy's csr_matvec."""
    nnz = int(indptr[-1]) if n else 0
    if n == 0 or nnz == 0 or n > (1 << 31) - 1:
        return None
    device = indptr.device
    row_len = (indptr[1:] - indptr[:-1]).to(torch.int32)
    ns = (n + 31) // 32
    padded = torch.zeros(ns * 32, dtype=torch.int32, device=device)
    padded[:n] = row_len
    width = padded.view(ns, 32).max(dim=1).values.to(torch.int64)
    slice_off = torch.zeros(ns + 1, dtype=torch.int64, device=device)
    slice_off[1:] = torch.cumsum(width * 32, 0)
    total = int(slice_off[-1])
    if total > 2 * nnz + 32 * ns:
        return None
    rows = torch.repeat_interleave(torch.arange(n, device=device), row_len.to(torch.int64))
    j = torch.arange(rows.numel(), device=device) - indptr[rows]
    dest = slice_off[rows // 32] + 32 * j + rows % 32
    cols = torch.zeros(total, dtype=torch.int32, device=device)
    vals = torch.zeros(total, dtype=torch.float64, device=device)
    cols[dest] = indices.to(torch.int32)
    vals[dest] = data
    return slice_off[:-1].contiguous(), row_len.contiguous(), cols, vals


@dataclass
class SparseMatrix:
    """CSR storage plus the symmetry promise the solvers rely on (apps.py:33-58);
    a device copy (int64 indptr, int32/int64 indices, fp64 data) is made on
    first use."""

    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    n: int
    symmetric: bool = True
    _csr: Optional[sp.csr_matrix] = field(default=None, repr=False, compare=False)
    _device: Optional[tuple] = field(default=None, repr=False, compare=False)
    _sell: Optional[object] = field(default=None, repr=False, compare=False)
    # captured solver-iteration graphs and the device vectors they read, per
    # solver configuration (see _graph_entry)
    _graphs: dict = field(default_factory=dict, repr=False, compare=False)

    @classmethod
    def from_csr(cls, m: sp.csr_matrix, symmetric: bool = True) -> "SparseMatrix":
        m = m.tocsr()
        m.sort_indices()
        return cls(indptr=m.indptr, indices=m.indices, data=m.data, n=m.shape[0], symmetric=symmetric, _csr=m)

    def csr(self) -> sp.csr_matrix:
        if self._csr is None:
            self._csr = sp.csr_matrix((self.data, self.indices, self.indptr), shape=(self.n, self.n))
        return self._csr

    def device_arrays(self):
        if self._device is None:
            torch, device = _dev()
            indptr = torch.from_numpy(np.ascontiguousarray(self.indptr, dtype=np.int64)).to(device)
            idx = np.ascontiguousarray(self.indices)
            if idx.dtype not in (np.int32, np.int64):
                idx = idx.astype(np.int64)
            indices = torch.from_numpy(idx).to(device)
            data = torch.from_numpy(np.ascontiguousarray(self.data, dtype=np.float64)).to(device)
            self._device = (indptr, indices, int(idx.dtype.itemsize), data)
        return self._device

    def sell_arrays(self):
        """Sliced-ELL copy (slices of 32 rows, column-major inside a slice),
        built on the device from the CSR arrays; None when a column index does
        not fit int32 or the padding would more than double the storage."""
        if self._sell is None:
            torch, _ = _dev()
            indptr, indices, _, data = self.device_arrays()
            self._sell = sell_layout(torch, indptr, indices, data, self.n) or False
        return self._sell or None

    def matvec_device(self, xd, out=None):
        """y = A x with device vectors: sliced-ELL kernel when available, else
        the CSR kernel (both sum each row like scipy's csr_matvec)."""
        torch, _ = _dev()
        if out is None:
            out = torch.empty(self.n, dtype=torch.float64, device=xd.device)
        lib = _lib.load()
        sell = self.sell_arrays()
        if sell is not None:
            so, rl, cols, vals = sell
            _lib.check(lib.qdot_b200_sell_spmv(self.n, so.data_ptr(), rl.data_ptr(), cols.data_ptr(),
                                               vals.data_ptr(), xd.data_ptr(), out.data_ptr(),
                                               stream_handle(xd.device)), lib)
            return out
        indptr, indices, ib, data = self.device_arrays()
        _lib.check(lib.qdot_b200_csr_spmv(self.n, indptr.data_ptr(), indices.data_ptr(), ib, data.data_ptr(),
                                          xd.data_ptr(), out.data_ptr(), stream_handle(xd.device)), lib)
        return out

    def clear_graphs(self) -> None:
        """Drop the cached solver-iteration graphs and their device buffers
        (entries a running solve holds are kept)."""
        with _graphs_lock:
            for k in list(self._graphs):
                e = self._graphs[k]
                if e.lock.acquire(blocking=False):
                    del self._graphs[k]
                    e.lock.release()

    def matvec(self, v):
        """A v on the device; numpy in -> numpy out, tensor in -> tensor out."""
        torch, _ = _dev()
        out = self.matvec_device(_to_device(v, self.n))
        return out if isinstance(v, torch.Tensor) else out.cpu().numpy()


def gen_stencil(nx: int, ny: int, nz: int) -> Tuple[SparseMatrix, np.ndarray]:
    """27-point stencil on an nx*ny*nz grid (apps.py:61-91): diagonal 27,
    in-grid neighbours -1; rhs = row sums, so the exact solution is all ones."""
    if nx < 1 or ny < 1 or nz < 1:
        raise ValueError("grid dimensions must be >= 1")
    n = nx * ny * nz
    gx, gy, gz = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"))
    point = (gx * ny + gy) * nz + gz
    r_parts, c_parts, v_parts = [], [], []
    for off in np.ndindex(3, 3, 3):
        d = np.array(off) - 1
        hx, hy, hz = gx + d[0], gy + d[1], gz + d[2]
        inside = (hx >= 0) & (hx < nx) & (hy >= 0) & (hy < ny) & (hz >= 0) & (hz < nz)
        r_parts.append(point[inside])
        c_parts.append(((hx * ny + hy) * nz + hz)[inside])
        v_parts.append(np.full(int(inside.sum()), 27.0 if not d.any() else -1.0))
    m = sp.coo_matrix((np.concatenate(v_parts), (np.concatenate(r_parts), np.concatenate(c_parts))),
                      shape=(n, n)).tocsr()
    a = SparseMatrix.from_csr(m, symmetric=True)
    rhs = a.csr() @ np.ones(n)           # host-side input preparation, as apps.py:90
    return a, rhs


def gen_graph_laplacian(n: int, edge_prob: float, seed: int = 0) -> SparseMatrix:
    """Laplacian D - A of an Erdos-Renyi G(n, edge_prob) graph (apps.py:94-118):
    the upper-triangle edges of row i are the draws rng.random(n-i-1) < p."""
    if not (0.0 <= edge_prob <= 1.0):
        raise ValueError("edge_prob must lie in [0, 1]")
    if n < 1:
        raise ValueError("n must be positive")
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for i in range(n - 1):
        j = i + 1 + np.flatnonzero(rng.random(n - i - 1) < edge_prob)
        src.append(np.full(j.size, i, dtype=np.int64))
        dst.append(j)
    r = np.concatenate(src) if src else np.empty(0, dtype=np.int64)
    c = np.concatenate(dst) if dst else np.empty(0, dtype=np.int64)
    adj = sp.coo_matrix((np.ones(r.size), (r, c)), shape=(n, n))
    adj = adj + adj.T
    deg = np.asarray(adj.sum(axis=1)).ravel()
    return SparseMatrix.from_csr((sp.diags(deg) - adj).tocsr(), symmetric=True)


# --------------------------------------------------------------------------- traces
@dataclass
class TraceRow:
    iteration: int
    call_site: str
    counts: dict
    n: int
    resid_or_lambda: float

    def pct(self, level: PrecisionLevel) -> float:
        return 100.0 * self.counts.get(level, 0) / self.n if self.n else 0.0


@dataclass
class SolveTrace:
    """Per-call precision mix of a solve (apps.py:134-159)."""

    rows: List[TraceRow] = field(default_factory=list)

    def record(self, iteration: int, call_site: str, report, resid_or_lambda: float) -> None:
        self.rows.append(TraceRow(iteration, call_site, dict(report.counts), report.n, resid_or_lambda))

    def write_csv(self, out: Union[str, IO[str]]) -> None:
        own = isinstance(out, str)
        fh = open(out, "w", newline="") if own else out
        try:
            fh.write(TRACE_HEADER + "\n")
            w = csv.writer(fh, lineterminator="\n")
            for r in self.rows:
                w.writerow([r.iteration, r.call_site, repr(r.pct(PrecisionLevel.PERFORATE)),
                            repr(r.pct(PrecisionLevel.HALF)), repr(r.pct(PrecisionLevel.SINGLE)),
                            repr(r.pct(PrecisionLevel.DOUBLE)), repr(r.resid_or_lambda)])
        finally:
            if own:
                fh.close()


@dataclass
class CGResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_norm: float
    trace: SolveTrace


@dataclass
class PMResult:
    eigenvalue: float
    x: np.ndarray
    iterations: int
    converged: bool
    trace: SolveTrace


# --------------------------------------------------------------------------- graph iterations
GRAPH_MIN = 2048          # solves of at least this many unknowns run their iterations in the device loop
GRAPH_REPEAT = True       # smaller ones too from their second solve on the same matrix and configuration
                          # (a capture costs ~2-3 ms: worth it once the graph is replayed by later solves)


class _GraphEntry:
    """A solver's captured iteration graph(s) and the device vectors they
    read, kept on the matrix so a repeated solve replays instead of
    re-capturing (a capture costs ~2-3 ms).  One solve at a time holds it."""

    def __init__(self):
        self.lock = threading.Lock()
        self.solves = 0
        self.G = None
        self.graphs = None
        self.bufs = None


def _cfg_key(cfg: ToleranceConfig):
    return (float(cfg.epsilon), cfg.split.value, int(cfg.input_mu))


GRAPH_CACHE_MAX = 4       # captured configurations kept per matrix (each holds two ~67 MB qdot workspaces)
_graphs_lock = threading.Lock()


def _graph_entry(a: "SparseMatrix", key) -> Optional[_GraphEntry]:
    """The entry for `key`, locked for this solve, or None when another solve
    holds it (that solve then uses fresh buffers and its own capture).  The
    per-matrix cache is an LRU of GRAPH_CACHE_MAX entries: the least recently
    used entry that no solve holds is dropped (with its workspaces) first."""
    with _graphs_lock:
        e = a._graphs.pop(key, None) or _GraphEntry()
        a._graphs[key] = e                                    # most recently used last
        if len(a._graphs) > GRAPH_CACHE_MAX:
            for k in list(a._graphs):
                if len(a._graphs) <= GRAPH_CACHE_MAX:
                    break
                old = a._graphs[k]
                if k != key and old.lock.acquire(blocking=False):
                    del a._graphs[k]
                    old.lock.release()
    return e if e.lock.acquire(blocking=False) else None


class _IterGraph:
    """Device resources of a solver's device-resident iteration loop: two qdot
    workspaces (one per dot product of an iteration), the scalar state st[8],
    the loop graph (a WHILE-conditional node around one captured iteration)
    and its per-iteration record buffer (two 256-byte result headers and st)."""

    def __init__(self, device):
        torch, _ = _dev()
        lib = _lib.load()
        nb = int(lib.qdot_b200_workspace_bytes())
        self.lib = lib
        self.ws = [torch.empty(nb, dtype=torch.uint8, device=device) for _ in range(2)]
        self.st = torch.zeros(8, dtype=torch.float64, device=device)

    def qdot_nodes(self, k: int, xd, yd, norm: bool, c, stream: int, zeroed: bool = False) -> None:
        """The qdot pipeline into workspace k (stream-ordered, no host sync);
        zeroed: the workspace's exchange regions were cleared by an earlier node."""
        lib, ws, n = self.lib, self.ws[k].data_ptr(), int(xd.shape[0])
        xp = xd.data_ptr()
        yp = xp if norm else yd.data_ptr()
        # begin / pass 1 / score / pass 2, or the one-launch cluster path at small n
        fn = lib.qdot_b200_enqueue_zeroed if zeroed else lib.qdot_b200_enqueue
        _lib.check(fn(xp, yp, n, int(norm), ctypes.byref(c), ws, stream), lib)

    def clear_all(self, stream: int) -> None:
        """Zero both workspaces' exchange regions (before a loop whose body
        clears them itself for the next iteration)."""
        for w in self.ws:
            _lib.check(self.lib.qdot_b200_begin(w.data_ptr(), stream), self.lib)

    # ---- device-resident loop: a WHILE-conditional graph whose body is one
    # iteration ending with a check kernel (qdot_b200_cg_p_check for ACG,
    # qdot_b200_pm_check for APM: records the iteration, sets the loop
    # condition); one launch and one host wake-up per solve
    LOOP_CAP = 4096                                           # iterations per launch (record buffer)

    def pm_div(self, z, xn, stream: int) -> None:
        _lib.check(self.lib.qdot_b200_pm_div(z.shape[0], self.ws[0].data_ptr(), self.st.data_ptr(), z.data_ptr(),
                                             xn.data_ptr(), stream), self.lib)

    def pm_check(self, xn, x, handle: int, stream: int) -> None:
        _lib.check(self.lib.qdot_b200_pm_check(x.shape[0], self.ws[0].data_ptr(), self.ws[1].data_ptr(),
                                               self.st.data_ptr(), xn.data_ptr(), x.data_ptr(), self.rec.data_ptr(),
                                               self.ctr.data_ptr(), handle, stream), self.lib)

    def cg_xr(self, x, p, r, q, stream: int) -> None:
        """... and zero workspace 1 for the r.r qdot that follows."""
        _lib.check(self.lib.qdot_b200_cg_xr(x.shape[0], self.ws[0].data_ptr(), self.st.data_ptr(), x.data_ptr(),
                                            p.data_ptr(), r.data_ptr(), q.data_ptr(), self.ws[1].data_ptr(), stream),
                   self.lib)

    def cg_p_check(self, r, p, handle: int, stream: int) -> None:
        """... and zero workspace 0 for the next iteration's p.Ap qdot."""
        _lib.check(self.lib.qdot_b200_cg_p_check(r.shape[0], self.ws[0].data_ptr(), self.ws[1].data_ptr(),
                                                 self.st.data_ptr(), r.data_ptr(), p.data_ptr(), self.rec.data_ptr(),
                                                 self.ctr.data_ptr(), handle, self.ws[0].data_ptr(), stream),
                   self.lib)

    def capture_loop(self, body):
        """Build the loop graph: `body(stream, handle)` is captured as the
        WHILE node's body on a side stream (nothing runs yet)."""
        torch, device = _dev()
        self.ctr = torch.zeros(3, dtype=torch.int64, device=self.st.device)    # k, cap, CTA ticket
        self.ctr_host = torch.zeros(3, dtype=torch.int64).pin_memory()
        self.st_host = torch.zeros(8, dtype=torch.float64).pin_memory()
        self.rec = torch.empty(self.LOOP_CAP * 576, dtype=torch.uint8, device=self.st.device)
        # read back after a launch: the counter and the first REC_HEAD records in one
        # copy + sync, the rest only for longer runs
        self.back = torch.empty(64 + self.REC_HEAD * 576, dtype=torch.uint8).pin_memory()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        loop = ctypes.c_void_p()
        handle = ctypes.c_ulonglong()
        _lib.check(self.lib.qdot_b200_loop_create(side.cuda_stream, ctypes.byref(loop), ctypes.byref(handle)),
                   self.lib)
        self.loop = loop
        try:
            with torch.cuda.stream(side):
                body(side.cuda_stream, handle.value)
        finally:
            _lib.check(self.lib.qdot_b200_loop_finish(loop, side.cuda_stream), self.lib)
        torch.cuda.current_stream().wait_stream(side)

    REC_DTYPE = np.dtype({"names": ["a", "b", "st"], "formats": [_lib.RESULT_DTYPE, _lib.RESULT_DTYPE, ("<f8", (8,))],
                          "offsets": [0, 256, 512], "itemsize": 576})

    REC_HEAD = 64                                             # records read back with the counter

    def run_loop(self, cap: int, tau: float, st0=None):
        """Run up to `cap` iterations on the device; st0: {index: value} of the
        scalar state to set first (with st[7] = tau, one host->device copy).
        Returns the recorded iterations as a numpy record array (fields a / b:
        the two dots' result headers, st: the scalar state)."""
        torch, _ = _dev()
        stream = torch.cuda.current_stream()
        if st0 is not None:
            for i, v in st0.items():
                self.st_host[i] = v
            self.st_host[7] = tau
            self.st.copy_(self.st_host, non_blocking=True)
        else:
            self.st[7] = tau
        self.ctr_host[0] = 0
        self.ctr_host[1] = cap
        self.ctr_host[2] = 0
        self.ctr.copy_(self.ctr_host, non_blocking=True)
        _lib.check(self.lib.qdot_b200_loop_launch(self.loop, stream.cuda_stream), self.lib)
        back = self.back
        back[:24].copy_(self.ctr.view(torch.uint8), non_blocking=True)
        back[64:].copy_(self.rec[:self.REC_HEAD * 576], non_blocking=True)
        stream.synchronize()                                  # waits for the loop
        k = int(back[:8].view(torch.int64)[0])
        if k <= self.REC_HEAD:
            raw = back[64:64 + k * 576].numpy().tobytes()
        else:
            raw = back[64:].numpy().tobytes() + self.rec[self.REC_HEAD * 576:k * 576].cpu().numpy().tobytes()
        return np.frombuffer(raw, dtype=self.REC_DTYPE, count=k)

    def header(self, rec, field: str, i: int):
        """Record i's result header `field` as a QdotResult (error paths)."""
        raw = rec[field][i:i + 1].tobytes()
        return _lib.QdotResult.from_buffer_copy(raw + bytes(ctypes.sizeof(_lib.QdotResult) - len(raw)))

    def __del__(self):
        loop = getattr(self, "loop", None)
        if loop is not None and loop.value:
            try:
                self.lib.qdot_b200_loop_destroy(loop)
            except Exception:
                pass


def _dot_report(res) -> "_DotReport":
    _raise_status(res)
    counts = {level: int(res.counts[i]) for i, level in enumerate(LEVELS_ASC)}
    return _DotReport(float(res.value), counts, int(res.n), int(res.zero_count))


# --------------------------------------------------------------------------- solvers
def _norm_dot(dots: _Dots, v):
    rep = dots(v, v, True)
    if not (rep.value >= 0.0):                              # apps.py:171-175
        raise AssertionError("norm computed by qdot must be nonnegative")
    return rep


def acg(a: SparseMatrix, b, x0=None, tau: float = 1e-8, epsilon: float = 1e-8,
        split: SplitMode = SplitMode.PER_BIN, max_iters: int = 10_000, strategy: Strategy = None) -> CGResult:
    """Conjugate gradient with r.r and p.Ap computed by qdot (apps.py:178-229)."""
    if strategy is None:
        strategy = ExactBinning()
    if not a.symmetric:
        raise ValueError("CG needs a symmetric positive definite matrix")
    cfg = ToleranceConfig(epsilon=epsilon, split=split)
    torch, device = _dev()
    n = a.n
    entry = _graph_entry(a, ("acg", _cfg_key(cfg), strategy_label(strategy), str(device))) if max_iters > 0 else None
    use_graph = max_iters > 0 and (n >= GRAPH_MIN or (GRAPH_REPEAT and entry is not None and entry.solves > 0))
    try:
        return _acg(a, b, x0, tau, max_iters, cfg, strategy, torch, device, n, use_graph, entry)
    finally:
        if entry is not None:
            entry.solves += 1
            entry.lock.release()


def _acg(a, b, x0, tau, max_iters, cfg, strategy, torch, device, n, use_graph, entry) -> CGResult:
    dots = _Dots(cfg, strategy)
    cached = entry is not None and entry.G is not None
    if cached:                                                # the captured graph reads these buffers
        x, r, p, q = entry.bufs
        if x0 is None:
            x.zero_()
        else:
            x.copy_(_to_device(x0, n))
    else:
        x = torch.zeros(n, dtype=torch.float64, device=device) if x0 is None else _to_device(x0, n).clone()
        q = torch.empty(n, dtype=torch.float64, device=device)
        r = torch.empty(n, dtype=torch.float64, device=device)
        p = torch.empty(n, dtype=torch.float64, device=device)
    bd = _to_device(b, n)
    trace = SolveTrace()

    a.matvec_device(x, out=q)
    _update(_SUB, bd, 1.0, q, r)                              # r = b - A x (1.0 * q is exact)
    p.copy_(r)
    c_rep = _norm_dot(dots, r)
    c = c_rep.value
    resid = math.sqrt(c)
    trace.record(0, "rtr", c_rep, resid)

    k = 0
    if use_graph and resid > tau:
        # the iterations run on the device: one CUDA graph whose WHILE node
        # repeats SpMV, p.Ap, alpha, x and r updates, r.r, beta, p update and
        # the check node (records the iteration, decides whether to go on);
        # one launch and one host wake-up per solve (or per LOOP_CAP iterations)
        if cached:
            G = entry.G
        else:
            G = _IterGraph(device)
            cst = config_struct(cfg, strategy)

            def body(stream, handle):
                # the workspaces are cleared by the kernel before each qdot (cg_p_check
                # for the next p.Ap, cg_xr for r.r): no begin launches in the loop
                a.matvec_device(p, out=q)
                G.qdot_nodes(0, p, q, False, cst, stream, zeroed=True)
                G.cg_xr(x, p, r, q, stream)                     # alpha = c / d; x += alpha p; r -= alpha q
                G.qdot_nodes(1, r, r, True, cst, stream, zeroed=True)
                G.cg_p_check(r, p, handle, stream)              # beta = c_new / c; p = r + beta p; c = c_new; check

            a.device_arrays()                                   # host->device copies cannot be captured
            a.sell_arrays()
            G.capture_loop(body)
            if entry is not None:
                entry.G, entry.graphs, entry.bufs = G, None, (x, r, p, q)
        G.clear_all(stream_handle(device))                       # workspace 0 for the first p.Ap
        first = True
        while resid > tau and k < max_iters:
            # st[0] = c on the first launch (later chunks continue from the device's c)
            rec = G.run_loop(min(max_iters - k, G.LOOP_CAP), tau, st0={0: c} if first else None)
            first = False
            # the host loop's checks and trace rows, from the parsed records in bulk
            a, b = rec["a"], rec["b"]
            sa, va, ca, na = a["status"].tolist(), a["value"].tolist(), a["counts"].tolist(), a["n"].tolist()
            sb, vb, cb, nb_ = b["status"].tolist(), b["value"].tolist(), b["counts"].tolist(), b["n"].tolist()
            rows = trace.rows
            for i in range(len(sa)):
                if sa[i] != _lib.QDOT_OK:
                    _dot_report(G.header(rec, "a", i))                # raises the call's error
                d = va[i]
                if not math.isfinite(d) or d <= 0.0:
                    raise BreakdownError(f"p.Ap = {d!r} at iteration {k}")
                if sb[i] != _lib.QDOT_OK:
                    _dot_report(G.header(rec, "b", i))
                c = vb[i]
                if not (c >= 0.0):                                    # apps.py:171-175
                    raise AssertionError("norm computed by qdot must be nonnegative")
                resid = math.sqrt(c)
                k += 1
                rows.append(TraceRow(k, "pAp", dict(zip(LEVELS_ASC, ca[i])), na[i], resid))
                rows.append(TraceRow(k, "rtr", dict(zip(LEVELS_ASC, cb[i])), nb_[i], resid))
    while resid > tau and k < max_iters:
        a.matvec_device(p, out=q)
        d_rep = dots(p, q, False)
        d = d_rep.value
        if not math.isfinite(d) or d <= 0.0:
            raise BreakdownError(f"p.Ap = {d!r} at iteration {k}")
        alpha = c / d
        _update(_ADD, x, alpha, p, x)                         # x = x + alpha * p
        _update(_SUB, r, alpha, q, r)                         # r = r - alpha * q
        c_rep = _norm_dot(dots, r)
        c_new = c_rep.value
        beta = c_new / c
        _update(_ADD, r, beta, p, p)                          # p = r + beta * p
        c = c_new
        resid = math.sqrt(c)
        k += 1
        trace.record(k, "pAp", d_rep, resid)
        trace.record(k, "rtr", c_rep, resid)
    return CGResult(x=x.cpu().numpy(), iterations=k, converged=resid <= tau, residual_norm=resid, trace=trace)


def apm(a: SparseMatrix, x0, tau: float = 1e-6, epsilon: float = 1e-7, split: SplitMode = SplitMode.PER_BIN,
        max_iters: int = 300, strategy: Strategy = None) -> PMResult:
    """Power method with z.z and the Rayleigh quotient computed by qdot (apps.py:275-325)."""
    if strategy is None:
        strategy = ExactBinning()
    cfg = ToleranceConfig(epsilon=epsilon, split=split)
    x_h = np.array(x0, dtype=np.float64)
    nrm = float(np.linalg.norm(x_h))                          # host, as apps.py:292
    if nrm == 0.0:
        raise ZeroIterateError("x0 is the zero vector")
    torch, device = _dev()
    entry = _graph_entry(a, ("apm", _cfg_key(cfg), strategy_label(strategy), str(device))) if max_iters > 0 else None
    use_graph = max_iters > 0 and (a.n >= GRAPH_MIN or (GRAPH_REPEAT and entry is not None and entry.solves > 0))
    try:
        return _apm(a, x_h, nrm, tau, max_iters, cfg, strategy, torch, device, use_graph, entry)
    finally:
        if entry is not None:
            entry.solves += 1
            entry.lock.release()


def _apm(a, x_h, nrm, tau, max_iters, cfg, strategy, torch, device, use_graph, entry) -> PMResult:
    cached = entry is not None and entry.G is not None
    if cached:                                                # the captured graphs read these buffers
        x, x_next, z = entry.bufs
        x.copy_(_to_device(x_h / nrm, a.n))
    else:
        x = _to_device(x_h / nrm, a.n).clone()
        z = torch.empty_like(x)
        x_next = torch.empty_like(x)
    dots = _Dots(cfg, strategy)
    trace = SolveTrace()

    lam_prev = None
    lam = 0.0
    k = 0
    converged = False
    if use_graph:
        # the iterations run on the device: one CUDA graph whose WHILE node
        # repeats SpMV (z = A x), z.z, x_next = z / sqrt(z.z), x.x_next and the
        # check node (x = x_next, lam, record, convergence); one launch and one
        # host wake-up per solve (or per LOOP_CAP iterations)
        if cached:
            G = entry.G
        else:
            G = _IterGraph(device)
            cst = config_struct(cfg, strategy)

            def body(stream, handle):
                a.matvec_device(x, out=z)
                G.qdot_nodes(0, z, z, True, cst, stream)
                G.pm_div(z, x_next, stream)                     # x_next = z / sqrt(z.z)
                G.qdot_nodes(1, x, x_next, False, cst, stream)
                G.pm_check(x_next, x, handle, stream)           # x = x_next; lam; record; go on?

            a.device_arrays()                                   # host->device copies cannot be captured
            a.sell_arrays()
            G.capture_loop(body)
            if entry is not None:
                entry.G, entry.graphs, entry.bufs = G, None, (x, x_next, z)
        while k < max_iters and not converged:
            rec = G.run_loop(min(max_iters - k, G.LOOP_CAP), tau,
                             st0={5: 0.0 if lam_prev is None else lam_prev, 6: 0.0 if lam_prev is None else 1.0})
            ra, rb = rec["a"], rec["b"]
            sa, va, ca, na, za = (ra["status"].tolist(), ra["value"].tolist(), ra["counts"].tolist(),
                                  ra["n"].tolist(), ra["zero_count"].tolist())
            sb, vb, cb, nb_ = rb["status"].tolist(), rb["value"].tolist(), rb["counts"].tolist(), rb["n"].tolist()
            rows = trace.rows
            for i in range(len(sa)):
                if sa[i] != _lib.QDOT_OK:
                    _dot_report(G.header(rec, "a", i))                # raises the call's error
                if za[i] == na[i]:
                    raise ZeroIterateError(f"A x vanished at iteration {k}")
                if not (va[i] >= 0.0):                                # apps.py:171-175
                    raise AssertionError("norm computed by qdot must be nonnegative")
                s_ = math.sqrt(va[i])
                if sb[i] != _lib.QDOT_OK:
                    _dot_report(G.header(rec, "b", i))
                lam = vb[i] * s_
                k += 1
                rows.append(TraceRow(k, "norm", dict(zip(LEVELS_ASC, ca[i])), na[i], lam))
                rows.append(TraceRow(k, "lambda", dict(zip(LEVELS_ASC, cb[i])), nb_[i], lam))
                if lam_prev is not None and abs(lam - lam_prev) <= tau:
                    converged = True
                    break
                lam_prev = lam
        return PMResult(eigenvalue=lam, x=x.cpu().numpy(), iterations=k, converged=converged, trace=trace)
    while k < max_iters:
        a.matvec_device(x, out=z)
        # np.any(z) (apps.py:305) from the same qdot call: z.z has a zero
        # product exactly where z_i == 0 (NaN makes qdot raise ValueError, as
        # the reference's qdot would right after its np.any)
        c_rep = _norm_dot(dots, z)
        if c_rep.zero_count == c_rep.n:
            raise ZeroIterateError(f"A x vanished at iteration {k}")
        c = c_rep.value
        s = math.sqrt(c)
        _update(_DIV, z, s, None, x_next)                     # x_next = z / s
        lam_rep = dots(x, x_next, False)
        lam = lam_rep.value * s
        k += 1
        trace.record(k, "norm", c_rep, lam)
        trace.record(k, "lambda", lam_rep, lam)
        x, x_next = x_next, x
        if lam_prev is not None and abs(lam - lam_prev) <= tau:
            converged = True
            break
        lam_prev = lam
    return PMResult(eigenvalue=lam, x=x.cpu().numpy(), iterations=k, converged=converged, trace=trace)


def reference_cg(a: SparseMatrix, b, x0=None, tau: float = 1e-8, max_iters: int = 10_000) -> CGResult:
    """Plain double CG with the identical stopping rule (apps.py:232-263), on
    the device with torch dots (a baseline, not bit-identical to numpy's)."""
    torch, device = _dev()
    n = a.n
    x = torch.zeros(n, dtype=torch.float64, device=device) if x0 is None else _to_device(x0, n).clone()
    r = _to_device(b, n) - a.matvec_device(x)
    p = r.clone()
    c = float(torch.dot(r, r))
    resid = math.sqrt(c)
    k = 0
    while resid > tau and k < max_iters:
        q = a.matvec_device(p)
        d = float(torch.dot(p, q))
        if not math.isfinite(d) or d <= 0.0:
            raise BreakdownError(f"p.Ap = {d!r} at iteration {k}")
        alpha = c / d
        x = x + alpha * p
        r = r - alpha * q
        c_new = float(torch.dot(r, r))
        beta = c_new / c
        p = r + beta * p
        c = c_new
        resid = math.sqrt(c)
        k += 1
    return CGResult(x=x.cpu().numpy(), iterations=k, converged=resid <= tau, residual_norm=resid,
                    trace=SolveTrace())


def reference_pm(a: SparseMatrix, x0, tau: float = 1e-6, max_iters: int = 300) -> PMResult:
    """Plain double power method with the identical stopping rule (apps.py:328-359)."""
    torch, _ = _dev()
    x_h = np.array(x0, dtype=np.float64)
    nrm = float(np.linalg.norm(x_h))
    if nrm == 0.0:
        raise ZeroIterateError("x0 is the zero vector")
    x = _to_device(x_h / nrm, a.n)
    lam_prev = None
    lam = 0.0
    k = 0
    converged = False
    while k < max_iters:
        z = a.matvec_device(x)
        if not bool(torch.any(z != 0)):
            raise ZeroIterateError(f"A x vanished at iteration {k}")
        c = float(torch.dot(z, z))
        s = math.sqrt(c)
        x_next = z / s
        lam = float(torch.dot(x, x_next)) * s
        k += 1
        x = x_next
        if lam_prev is not None and abs(lam - lam_prev) <= tau:
            converged = True
            break
        lam_prev = lam
    return PMResult(eigenvalue=lam, x=x.cpu().numpy(), iterations=k, converged=converged, trace=SolveTrace())
