// Phase clocks of the score(+finalize) CTA on a C2-like input (standard
// normal, n from argv[1]), averaged over repetitions.  Build and run:
//   bash scripts/score_prof.sh
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>
#include "qdot_b200.h"
extern "C" int qdot_b200_score_prof(long long* out);

int main(int argc, char** argv) {
    long long n = argc > 1 ? atoll(argv[1]) : 1000000;
    double eps = argc > 2 ? atof(argv[2]) : 1e-8;
    int strategy = argc > 3 ? atoi(argv[3]) : 0, param = argc > 4 ? atoi(argv[4]) : 0;
    const int twice = argc > 5 ? atoi(argv[5]) : 0;   // 1: time a second, warm-cache score launch
    std::vector<double> hx(n), hy(n);
    std::mt19937_64 g(0);
    std::normal_distribution<double> nd;
    for (long long i = 0; i < n; ++i) { hx[i] = nd(g); hy[i] = nd(g); }
    double *x, *y; void* ws;
    cudaMalloc(&x, n * 8); cudaMalloc(&y, n * 8); cudaMalloc(&ws, qdot_b200_workspace_bytes());
    cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(y, hy.data(), n * 8, cudaMemcpyHostToDevice);
    qdot_config c{};
    c.epsilon = eps; c.split = 0; c.input_mu = 52; c.strategy = strategy; c.strategy_param = param;
    const int R = 50;
    double acc[16] = {0};   // [13..15]: cached path: bin 0 setup, bin_value, rest of the per-bin phase
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int r = 0; r < R + 5; ++r) {
        qdot_b200_begin(ws, 0);
        qdot_b200_pass1(x, y, n, 0, &c, n, ws, 0);
        qdot_b200_score_finalize(ws, n, &c, 0);
        if (twice) qdot_b200_score_finalize(ws, n, &c, 0);
        cudaDeviceSynchronize();
        long long p[16];
        qdot_b200_score_prof(p);
        if (r >= 5) for (int i = 1; i <= 12; ++i) acc[i] += (double)(p[i] - p[i - 1]);
        if (r >= 5) { acc[13] += (double)(p[9] - p[4]); acc[14] += (double)(p[10] - p[9]); acc[15] += (double)(p[5] - p[10]); }
    }
    const char* nm[] = {"", "load+minmax", "scan+init+tid0", "partition", "eps", "per-bin", "lut", "lut-reduce+meta",
                        "fin:init", "fin:bins", "fin:neumaier", "fin:counts", "fin:result"};
    double tot = 0;
    for (int i = 1; i <= 12; ++i) tot += acc[i] / R;
    printf("%s n=%lld strategy=%d clock %d kHz; total %.0f cycles\n", twice ? "warm" : "cold", n, strategy, clk, tot);
    for (int i = 1; i <= 12; ++i) printf("  %-18s %8.0f cycles\n", nm[i], acc[i] / R);
    printf("  per-bin split (cached path, bin 0): setup %.0f, bin_value %.0f, rest %.0f\n", acc[13] / R, acc[14] / R,
           acc[15] / R);
    return 0;
}
