// qdot_apps.cu -- device kernels for the solver callers of qdot (apps.py):
// CSR matrix-vector product and the vector updates of ACG / APM, each
// bit-identical to the reference's numpy / scipy operation it replaces, so
// the solvers' iterates, iteration counts and traces match the reference.
//
//   csr_spmv   scipy csr_matvec (apps.py:57-58): y[i] = ((0 + a_0 x_j0) + a_1 x_j1) + ...
//              in CSR order, every product and sum rounded separately (no FMA).
//   vec_update numpy elementwise forms of apps.py:216-220, 306-308:
//              a + s*b, a - s*b (the product rounded first), a / s.
//
// Everything is memory bound (a few bytes per flop); grids are sized in
// multiples of the SM count and loops are grid-stride.

#include <cuda_runtime.h>

#include <cstdint>

#include "qdot_common.cuh"

namespace qd {
int report_cuda_error(cudaError_t e, const char* where);
}

namespace {

constexpr int T = 256;

int grid_for(int64_t n, int per_thread) {
    const int sms = qd::device_sm_count();
    int64_t g = (n + (int64_t)T * per_thread - 1) / ((int64_t)T * per_thread);
    int64_t cap = (int64_t)sms * 8;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

// one thread per row; the row's products are summed sequentially from +0.0
// exactly like scipy's csr_matvec (sum = Yx[i] = 0; sum += Ax[jj] * Xx[Aj[jj]])
template <typename IDX>
__global__ void __launch_bounds__(T) k_csr_spmv(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                const IDX* __restrict__ indices, const double* __restrict__ data,
                                                const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * T) {
        const int64_t b = __ldg(indptr + i), e = __ldg(indptr + i + 1);
        double s = 0.0;
        for (int64_t jj = b; jj < e; ++jj) s = __dadd_rn(s, __dmul_rn(__ldg(data + jj), __ldg(x + __ldg(indices + jj))));
        y[i] = s;
    }
}

// sliced ELL (slices of 32 rows; entry j of row r at slice_off[r/32] + 32 j + r%32):
// the 32 threads of a warp read consecutive values and column indices for
// the same j -- coalesced -- while every row keeps scipy's sequential
// left-to-right sum (padding is never read: each row stops at its length)
__global__ void __launch_bounds__(T) k_sell_spmv(int64_t n_rows, const int64_t* __restrict__ slice_off,
                                                 const int32_t* __restrict__ row_len,
                                                 const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                                 const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * T) {
        const int64_t base = __ldg(slice_off + (i >> 5)) + (i & 31);
        const int len = __ldg(row_len + i);
        double s = 0.0;
        for (int j = 0; j < len; ++j) {
            const int64_t k = base + 32 * (int64_t)j;
            s = __dadd_rn(s, __dmul_rn(__ldg(vals + k), __ldg(x + __ldg(cols + k))));
        }
        y[i] = s;
    }
}

// op 0: out = a + s*b; 1: out = a - s*b; 2: out = a / s.  out may alias a or b
// (each element is read and written by the same thread), so no __restrict__.
template <int OP>
__global__ void __launch_bounds__(T) k_vec_update(int64_t n, const double* a, double s, const double* b,
                                                  double* out) {
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T) {
        const double av = a[i];
        double r;
        if (OP == 0) r = __dadd_rn(av, __dmul_rn(s, b[i]));
        else if (OP == 1) r = __dsub_rn(av, __dmul_rn(s, b[i]));
        else r = __ddiv_rn(av, s);
        out[i] = r;
    }
}

// streaming-read probe: the HBM read ceiling for pass 1's access pattern
// (grid-stride 128-bit evict-first loads, one sum per thread to keep the loads live)
__global__ void __launch_bounds__(T) k_read_probe(const double2* __restrict__ x, int64_t n2,
                                                  double* __restrict__ out) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * T;
    int64_t i = (int64_t)blockIdx.x * T + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        const double2 a = __ldcs(x + i), b = __ldcs(x + i + stride);
        const double2 c = __ldcs(x + i + 2 * stride), d = __ldcs(x + i + 3 * stride);
        acc += (a.x + a.y) + (b.x + b.y) + (c.x + c.y) + (d.x + d.y);
    }
    for (; i < n2; i += stride) {
        const double2 a = __ldcs(x + i);
        acc += a.x + a.y;
    }
    if (acc == 1.2345e-300) *out = acc;     // never true for real data; keeps the loads
}

// ---- device-side scalar recurrences of the solvers (for CUDA-graph iterations)
// st: [0] c (r.r, or z.z for the power method), [1] alpha, [2] beta, [3] sqrt(c),
//     [4] d (p.Ap), [5..7] unused
__device__ __forceinline__ double result_value(const void* ws) {
    return reinterpret_cast<const qdot_result*>(static_cast<const char*>(ws) + qd::OFF_RESULT)->value;
}

// alpha = c / d with d = value of the qdot in ws_pq (apps.py:212-216)
__global__ void k_cg_alpha(const void* ws_pq, double* st) {
    const double d = result_value(ws_pq);
    st[4] = d;
    st[1] = __ddiv_rn(st[0], d);
}

// c_new = value of the qdot in ws_rr; beta = c_new / c; c = c_new; sqrt (apps.py:217-223)
__global__ void k_cg_beta(const void* ws_rr, double* st) {
    const double c_new = result_value(ws_rr);
    st[2] = __ddiv_rn(c_new, st[0]);
    st[0] = c_new;
    st[3] = __dsqrt_rn(c_new);
}

// c = value of the qdot in ws; s = sqrt(c) (apps.py:307-309)
__global__ void k_norm_sqrt(const void* ws, double* st) {
    const double c = result_value(ws);
    st[0] = c;
    st[3] = __dsqrt_rn(c);
}

// out = a + s*b | a - s*b | a / s with s read from device memory
template <int OP>
__global__ void __launch_bounds__(T) k_vec_update_dev(int64_t n, const double* a, const double* __restrict__ sp,
                                                      const double* b, double* out) {
    const double s = *sp;
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T) {
        const double av = a[i];
        double r;
        if (OP == 0) r = __dadd_rn(av, __dmul_rn(s, b[i]));
        else if (OP == 1) r = __dsub_rn(av, __dmul_rn(s, b[i]));
        else r = __ddiv_rn(av, s);
        out[i] = r;
    }
}

// copy the result headers of two qdot workspaces and the scalar state into
// host memory (pinned, device-visible), then bump the sequence word
__global__ void k_publish_iter(const void* ws_a, const void* ws_b, const double* st, unsigned char* host,
                               uint32_t* dev_seq) {
    const int t = threadIdx.x;
    const uint32_t* ra = reinterpret_cast<const uint32_t*>(static_cast<const char*>(ws_a) + qd::OFF_RESULT);
    const uint32_t* rb = reinterpret_cast<const uint32_t*>(static_cast<const char*>(ws_b) + qd::OFF_RESULT);
    uint32_t* h = reinterpret_cast<uint32_t*>(host);
    if (t < 64) h[t] = ra[t];                       // 256 B header of ws_a
    else if (t < 128) h[t] = rb[t - 64];            // 256 B header of ws_b
    else if (t < 144) h[t] = reinterpret_cast<const uint32_t*>(st)[t - 128];   // 64 B state
    __threadfence_system();
    __syncthreads();
    if (t == 0) {
        const uint32_t sq = *dev_seq + 1;
        *dev_seq = sq;
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(host + 576) = sq;
    }
}

// ---- device-resident solver loop: the check node of a WHILE-conditional graph
// body.  Records iteration k (the two result headers and st, the block
// k_publish_iter publishes) into rec[k] and keeps looping while the host
// loop of apps.py:178-229 would: both dots OK, p.Ap finite and > 0, r.r >= 0,
// sqrt(r.r) > tau (IEEE sqrt = math.sqrt), k + 1 < cap.  counter = {k, cap}
// and tau = st[7] are set by the host before each launch (the graph is reused
// across solves and chunks).
constexpr int REC_BYTES = 576;
__global__ void k_acg_check(const void* ws_a, const void* ws_b, const double* st, unsigned char* rec,
                            long long* counter, cudaGraphConditionalHandle handle) {
    const int t = threadIdx.x;
    const long long k = counter[0], cap = counter[1];
    const double tau = st[7];
    const uint32_t* ra = reinterpret_cast<const uint32_t*>(static_cast<const char*>(ws_a) + qd::OFF_RESULT);
    const uint32_t* rb = reinterpret_cast<const uint32_t*>(static_cast<const char*>(ws_b) + qd::OFF_RESULT);
    uint32_t* h = reinterpret_cast<uint32_t*>(rec + k * REC_BYTES);
    if (t < 64) h[t] = ra[t];
    else if (t < 128) h[t] = rb[t - 64];
    else if (t < 144) h[t] = reinterpret_cast<const uint32_t*>(st)[t - 128];
    if (t == 0) {
        const qdot_result* r0 = reinterpret_cast<const qdot_result*>(ra);
        const qdot_result* r1 = reinterpret_cast<const qdot_result*>(rb);
        const double d = r0->value, c = r1->value;
        const bool go = r0->status == QDOT_OK && r1->status == QDOT_OK && (d - d == 0.0) && d > 0.0 && c >= 0.0 &&
                        __dsqrt_rn(c) > tau && k + 1 < cap;
        *counter = k + 1;
        cudaGraphSetConditional(handle, go ? 1u : 0u);
    }
}

// zero the exchange regions (A, B, rank-local counters) of the qdot workspace
// `ws`, grid-stride -- what qdot_b200_begin does, folded into a kernel that runs
// anyway once the workspace's previous call has been consumed
__device__ __forceinline__ void clear_ws(void* ws) {
    if (!ws) return;
    ulonglong2* z = reinterpret_cast<ulonglong2*>(static_cast<char*>(ws) + qd::OFF_A);
    const int64_t n16 = (qd::BYTES_A + qd::BYTES_B + qd::BYTES_LOCAL) / 16;
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n16; i += (int64_t)gridDim.x * T)
        z[i] = make_ulonglong2(0ull, 0ull);
}

// ---- fused ACG iteration kernels for the device loop (apps.py:212-223):
// x = x + alpha p and r = r - alpha q with alpha = c / d computed per thread
// (c = st[0], d = the p.Ap dot in ws_pq); the products rounded first like the
// numpy expressions.  Block 0 records alpha and d in st.
__global__ void __launch_bounds__(T) k_cg_xr(int64_t n, const void* ws_pq, double* st, double* x,
                                             const double* __restrict__ p, double* r, const double* __restrict__ q,
                                             void* ws_clear) {
    clear_ws(ws_clear);                          // the r.r workspace, for the qdot that follows
    const double d = result_value(ws_pq);
    const double alpha = __ddiv_rn(st[0], d);
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T) {
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
        r[i] = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { st[1] = alpha; st[4] = d; }
}

// p = r + beta p with beta = c_new / c (c_new = the r.r dot in ws_rr); the last
// CTA to finish (ticket counter[2]) then runs the check of k_acg_check and
// advances the recurrence: st[0] = c_new, st[2] = beta, st[3] = sqrt(c_new).
__global__ void __launch_bounds__(T) k_cg_p_check(int64_t n, const void* ws_pq, const void* ws_rr, double* st,
                                                  const double* __restrict__ r, double* p, unsigned char* rec,
                                                  long long* counter, cudaGraphConditionalHandle handle,
                                                  void* ws_clear) {
    clear_ws(ws_clear);                          // the p.Ap workspace (its result header is outside the regions)
    const double c_new = result_value(ws_rr);
    const double beta = __ddiv_rn(c_new, st[0]);
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T)
        p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
    __threadfence();
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0)
        last = atomicAdd(reinterpret_cast<unsigned long long*>(counter + 2), 1ull) == (unsigned long long)gridDim.x - 1ull;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int t = threadIdx.x;
    const long long k = counter[0], cap = counter[1];
    const qdot_result* r0 = reinterpret_cast<const qdot_result*>(static_cast<const char*>(ws_pq) + qd::OFF_RESULT);
    const qdot_result* r1 = reinterpret_cast<const qdot_result*>(static_cast<const char*>(ws_rr) + qd::OFF_RESULT);
    __shared__ bool go;
    if (t == 0) {
        const double d = r0->value;
        const double sq = __dsqrt_rn(c_new);
        go = r0->status == QDOT_OK && r1->status == QDOT_OK && (d - d == 0.0) && d > 0.0 && c_new >= 0.0 &&
             sq > st[7] && k + 1 < cap;
        st[0] = c_new;
        st[2] = beta;
        st[3] = sq;
    }
    __syncthreads();
    const uint32_t* ra = reinterpret_cast<const uint32_t*>(r0);
    const uint32_t* rb = reinterpret_cast<const uint32_t*>(r1);
    uint32_t* h = reinterpret_cast<uint32_t*>(rec + k * REC_BYTES);
    if (t < 64) h[t] = ra[t];
    else if (t < 128) h[t] = rb[t - 64];
    else if (t < 144) h[t] = reinterpret_cast<const uint32_t*>(st)[t - 128];
    if (t == 0) {
        counter[0] = k + 1;
        counter[2] = 0;
        cudaGraphSetConditional(handle, go ? 1u : 0u);
    }
}

// ---- fused power-method iteration kernels for the device loop (apps.py:302-315)
// x_next = z / s with s = sqrt(c), c = the z.z result in ws_zz (numpy z / s);
// block 0 records c and s in st[0], st[3]
__global__ void __launch_bounds__(T) k_pm_div(int64_t n, const void* ws_zz, double* st, const double* __restrict__ z,
                                              double* __restrict__ xn) {
    const double c = result_value(ws_zz);
    const double sq = __dsqrt_rn(c);
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T)
        xn[i] = __ddiv_rn(z[i], sq);
    if (blockIdx.x == 0 && threadIdx.x == 0) { st[0] = c; st[3] = sq; }
}

// x = x_next (the iterate for the next iteration); the last CTA computes
// lam = (x . x_next) * s (the host's lam_rep.value * s_), records the iteration
// and keeps looping while the host loop would: both dots OK, z not all zero,
// z.z >= 0, not (a previous lam and |lam - lam_prev| <= tau), k + 1 < cap.
// st: [0] c, [3] s, [4] lam, [5] lam_prev, [6] 1 when lam_prev exists, [7] tau.
__global__ void __launch_bounds__(T) k_pm_check(int64_t n, const void* ws_zz, const void* ws_lam, double* st,
                                                const double* __restrict__ xn, double* __restrict__ x,
                                                unsigned char* rec, long long* counter,
                                                cudaGraphConditionalHandle handle) {
    for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T) x[i] = xn[i];
    __threadfence();
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0)
        last = atomicAdd(reinterpret_cast<unsigned long long*>(counter + 2), 1ull) == (unsigned long long)gridDim.x - 1ull;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int t = threadIdx.x;
    const long long k = counter[0], cap = counter[1];
    const qdot_result* r0 = reinterpret_cast<const qdot_result*>(static_cast<const char*>(ws_zz) + qd::OFF_RESULT);
    const qdot_result* r1 = reinterpret_cast<const qdot_result*>(static_cast<const char*>(ws_lam) + qd::OFF_RESULT);
    __shared__ bool go;
    if (t == 0) {
        const double lam = __dmul_rn(r1->value, st[3]);
        const bool conv = st[6] != 0.0 && fabs(__dsub_rn(lam, st[5])) <= st[7];
        go = r0->status == QDOT_OK && r0->zero_count != r0->n && r0->value >= 0.0 && r1->status == QDOT_OK &&
             !conv && k + 1 < cap;
        st[4] = lam;
        st[5] = lam;
        st[6] = 1.0;
    }
    __syncthreads();
    const uint32_t* ra = reinterpret_cast<const uint32_t*>(r0);
    const uint32_t* rb = reinterpret_cast<const uint32_t*>(r1);
    uint32_t* h = reinterpret_cast<uint32_t*>(rec + k * REC_BYTES);
    if (t < 64) h[t] = ra[t];
    else if (t < 128) h[t] = rb[t - 64];
    else if (t < 144) h[t] = reinterpret_cast<const uint32_t*>(st)[t - 128];
    if (t == 0) {
        counter[0] = k + 1;
        counter[2] = 0;
        cudaGraphSetConditional(handle, go ? 1u : 0u);
    }
}

struct SolverLoop {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle handle = 0;
};

}  // namespace

extern "C" {

// A graph with one WHILE node (condition initially 1); the caller's stream
// then captures the loop body into it until qdot_b200_loop_finish.
int qdot_b200_loop_create(void* stream, void** loop, unsigned long long* handle) {
    if (!loop || !handle) return QDOT_ERR_ARG;
    SolverLoop* L = new SolverLoop();
    cudaError_t e = cudaGraphCreate(&L->graph, 0);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&L->handle, L->graph, 1u, cudaGraphCondAssignDefault);
    cudaGraph_t body = nullptr;
    if (e == cudaSuccess) {
        cudaGraphNodeParams p = {};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = L->handle;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        e = cudaGraphAddNode(&node, L->graph, nullptr, 0, &p);
        body = p.conditional.phGraph_out ? p.conditional.phGraph_out[0] : nullptr;
    }
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(static_cast<cudaStream_t>(stream), body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        if (L->graph) cudaGraphDestroy(L->graph);
        delete L;
        return qd::report_cuda_error(e, "loop_create");
    }
    *loop = L;
    *handle = (unsigned long long)L->handle;
    return QDOT_OK;
}

int qdot_b200_loop_finish(void* loop, void* stream) {
    if (!loop) return QDOT_ERR_ARG;
    SolverLoop* L = static_cast<SolverLoop*>(loop);
    cudaGraph_t body = nullptr;
    cudaError_t e = cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &body);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&L->exec, L->graph, 0);
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "loop_finish");
}

int qdot_b200_loop_launch(void* loop, void* stream) {
    if (!loop || !static_cast<SolverLoop*>(loop)->exec) return QDOT_ERR_ARG;
    cudaError_t e = cudaGraphLaunch(static_cast<SolverLoop*>(loop)->exec, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "loop_launch");
}

void qdot_b200_loop_destroy(void* loop) {
    if (!loop) return;
    SolverLoop* L = static_cast<SolverLoop*>(loop);
    if (L->exec) cudaGraphExecDestroy(L->exec);
    if (L->graph) cudaGraphDestroy(L->graph);
    delete L;
}

int qdot_b200_cg_xr(int64_t n, const void* ws_pq, double* st, double* x, const double* p, double* r,
                    const double* q, void* ws_clear, void* stream) {
    if (n < 0 || !ws_pq || !st || (n > 0 && (!x || !p || !r || !q))) return QDOT_ERR_ARG;
    const int g = grid_for(n > 0 ? n : 1, 4);
    k_cg_xr<<<g, T, 0, static_cast<cudaStream_t>(stream)>>>(n, ws_pq, st, x, p, r, q, ws_clear);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "cg_xr");
}

int qdot_b200_cg_p_check(int64_t n, const void* ws_pq, const void* ws_rr, double* st, const double* r, double* p,
                         void* rec, long long* counter, unsigned long long handle, void* ws_clear, void* stream) {
    if (n < 0 || !ws_pq || !ws_rr || !st || !rec || !counter || (n > 0 && (!r || !p))) return QDOT_ERR_ARG;
    const int g = grid_for(n > 0 ? n : 1, 4);
    k_cg_p_check<<<g, T, 0, static_cast<cudaStream_t>(stream)>>>(n, ws_pq, ws_rr, st, r, p,
                                                                  static_cast<unsigned char*>(rec), counter,
                                                                  (cudaGraphConditionalHandle)handle, ws_clear);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "cg_p_check");
}

int qdot_b200_pm_div(int64_t n, const void* ws_zz, double* st, const double* z, double* xn, void* stream) {
    if (n < 0 || !ws_zz || !st || (n > 0 && (!z || !xn))) return QDOT_ERR_ARG;
    const int g = grid_for(n > 0 ? n : 1, 4);
    k_pm_div<<<g, T, 0, static_cast<cudaStream_t>(stream)>>>(n, ws_zz, st, z, xn);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "pm_div");
}

int qdot_b200_pm_check(int64_t n, const void* ws_zz, const void* ws_lam, double* st, const double* xn, double* x,
                       void* rec, long long* counter, unsigned long long handle, void* stream) {
    if (n < 0 || !ws_zz || !ws_lam || !st || !rec || !counter || (n > 0 && (!xn || !x))) return QDOT_ERR_ARG;
    const int g = grid_for(n > 0 ? n : 1, 4);
    k_pm_check<<<g, T, 0, static_cast<cudaStream_t>(stream)>>>(n, ws_zz, ws_lam, st, xn, x,
                                                                static_cast<unsigned char*>(rec), counter,
                                                                (cudaGraphConditionalHandle)handle);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "pm_check");
}

int qdot_b200_acg_check(const void* ws_a, const void* ws_b, const double* st, void* rec, long long* counter,
                        unsigned long long handle, void* stream) {
    if (!ws_a || !ws_b || !st || !rec || !counter) return QDOT_ERR_ARG;
    k_acg_check<<<1, 160, 0, static_cast<cudaStream_t>(stream)>>>(ws_a, ws_b, st, static_cast<unsigned char*>(rec),
                                                                   counter, (cudaGraphConditionalHandle)handle);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "acg_check");
}

int qdot_b200_vec_update_dev(int64_t n, int op, const double* a, const double* s_dev, const double* b, double* out,
                             void* stream) {
    if (n < 0 || op < 0 || op > 2 || !s_dev) return QDOT_ERR_ARG;
    if (n == 0) return QDOT_OK;
    if (!a || !out || (op != 2 && !b)) return QDOT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int g = grid_for(n, 4);
    if (op == 0) k_vec_update_dev<0><<<g, T, 0, st>>>(n, a, s_dev, b, out);
    else if (op == 1) k_vec_update_dev<1><<<g, T, 0, st>>>(n, a, s_dev, b, out);
    else k_vec_update_dev<2><<<g, T, 0, st>>>(n, a, s_dev, b, out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "vec_update_dev");
}

int qdot_b200_solver_scalar(int which, const void* ws, double* st, void* stream) {
    if (!ws || !st || which < 0 || which > 2) return QDOT_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (which == 0) k_cg_alpha<<<1, 1, 0, s>>>(ws, st);
    else if (which == 1) k_cg_beta<<<1, 1, 0, s>>>(ws, st);
    else k_norm_sqrt<<<1, 1, 0, s>>>(ws, st);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "solver_scalar");
}

int qdot_b200_publish_iter(const void* ws_a, const void* ws_b, const double* st, void* host, uint32_t* dev_seq,
                           void* stream) {
    if (!ws_a || !ws_b || !st || !host || !dev_seq) return QDOT_ERR_ARG;
    k_publish_iter<<<1, 160, 0, static_cast<cudaStream_t>(stream)>>>(ws_a, ws_b, st,
                                                                      static_cast<unsigned char*>(host), dev_seq);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "publish_iter");
}

int qdot_b200_read_probe(const double* x, int64_t n, double* out, void* stream) {
    if (n < 0 || (n > 0 && (!x || !out)) || (reinterpret_cast<uintptr_t>(x) & 15u)) return QDOT_ERR_ARG;
    if (n < 2) return QDOT_OK;
    const int sms = qd::device_sm_count();
    k_read_probe<<<sms * 8, T, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const double2*>(x), n / 2, out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "read_probe");
}

int qdot_b200_csr_spmv(int64_t n_rows, const int64_t* indptr, const void* indices, int index_bytes,
                       const double* data, const double* x, double* y, void* stream) {
    if (n_rows < 0 || (index_bytes != 4 && index_bytes != 8)) return QDOT_ERR_ARG;
    if (n_rows == 0) return QDOT_OK;
    if (!indptr || !y) return QDOT_ERR_ARG;   // indices / data / x may be NULL when nnz == 0
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int g = grid_for(n_rows, 1);
    if (index_bytes == 4)
        k_csr_spmv<int32_t><<<g, T, 0, st>>>(n_rows, indptr, static_cast<const int32_t*>(indices), data, x, y);
    else
        k_csr_spmv<int64_t><<<g, T, 0, st>>>(n_rows, indptr, static_cast<const int64_t*>(indices), data, x, y);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "csr_spmv");
}

int qdot_b200_sell_spmv(int64_t n_rows, const int64_t* slice_off, const int32_t* row_len, const int32_t* cols,
                        const double* vals, const double* x, double* y, void* stream) {
    if (n_rows < 0) return QDOT_ERR_ARG;
    if (n_rows == 0) return QDOT_OK;
    if (!slice_off || !row_len || !y) return QDOT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_sell_spmv<<<grid_for(n_rows, 1), T, 0, st>>>(n_rows, slice_off, row_len, cols, vals, x, y);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "sell_spmv");
}

int qdot_b200_vec_update(int64_t n, int op, const double* a, double s, const double* b, double* out,
                         void* stream) {
    if (n < 0 || op < 0 || op > 2) return QDOT_ERR_ARG;
    if (n == 0) return QDOT_OK;
    if (!a || !out || (op != 2 && !b)) return QDOT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int g = grid_for(n, 4);
    if (op == 0) k_vec_update<0><<<g, T, 0, st>>>(n, a, s, b, out);
    else if (op == 1) k_vec_update<1><<<g, T, 0, st>>>(n, a, s, b, out);
    else k_vec_update<2><<<g, T, 0, st>>>(n, a, s, b, out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : qd::report_cuda_error(e, "vec_update");
}

}  // extern "C"
