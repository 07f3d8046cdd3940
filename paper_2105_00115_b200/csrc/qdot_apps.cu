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

#include "../../include/qdot_b200.h"

namespace qd {
int report_cuda_error(cudaError_t e, const char* where);
}

namespace {

constexpr int T = 256;

int grid_for(int64_t n, int per_thread) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (!sms) sms = 148;
    }
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

}  // namespace

extern "C" {

int qdot_b200_read_probe(const double* x, int64_t n, double* out, void* stream) {
    if (n < 0 || (n > 0 && (!x || !out)) || (reinterpret_cast<uintptr_t>(x) & 15u)) return QDOT_ERR_ARG;
    if (n < 2) return QDOT_OK;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
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
