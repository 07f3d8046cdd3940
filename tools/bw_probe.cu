// Read-bandwidth ceiling probe: stream two 2^28-element fp64 vectors with the
// same grid/tiling as pass 1 and a trivial reduction (no shared memory work).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int V, int T>
__global__ void __launch_bounds__(T) probe(const double* __restrict__ x, const double* __restrict__ y, long n,
                                           unsigned long long* out) {
    const long TILE = (long)T * 2 * V;
    long ntiles = n / TILE;
    unsigned long long acc = 0;
    for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const double2* x2 = reinterpret_cast<const double2*>(x + t * TILE);
        const double2* y2 = reinterpret_cast<const double2*>(y + t * TILE);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            double2 a = __ldcs(x2 + v * T + threadIdx.x);
            double2 b = __ldcs(y2 + v * T + threadIdx.x);
            acc += __double_as_longlong(a.x * b.x) ^ __double_as_longlong(a.y * b.y);
        }
    }
    if (acc == 0x12345) out[0] = acc;
}
template <int V, int T>
float run(const double* x, const double* y, long n, unsigned long long* o, int grid) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) probe<V, T><<<grid, T>>>(x, y, n, o);
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) probe<V, T><<<grid, T>>>(x, y, n, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 20;
}
int main() {
    long n = 1L << 28;
    double *x, *y; unsigned long long* o;
    cudaMalloc(&x, n * 8); cudaMalloc(&y, n * 8); cudaMalloc(&o, 8);
    cudaMemset(x, 0x3f, n * 8); cudaMemset(y, 0x3f, n * 8);
    int grids[] = {148, 296, 444, 592, 888, 1184, 2368};
    for (int g : grids) {
        float m2 = run<2, 256>(x, y, n, o, g), m4 = run<4, 256>(x, y, n, o, g), m8 = run<8, 256>(x, y, n, o, g);
        printf("{\"grid\": %d, \"V2_ms\": %.4f, \"V2_GBps\": %.1f, \"V4_ms\": %.4f, \"V4_GBps\": %.1f, \"V8_ms\": %.4f, \"V8_GBps\": %.1f}\n",
               g, m2, n * 16 / m2 / 1e6, m4, n * 16 / m4 / 1e6, m8, n * 16 / m8 / 1e6);
    }
    return 0;
}
