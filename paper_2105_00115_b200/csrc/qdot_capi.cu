// qdot_capi.cu -- extern "C" entry points declared in include/qdot_b200.h.
//
// Host-side orchestration only: validation, launch order, result transfer.
// All arithmetic on the data happens in the sm_100a kernels (qdot_kernels.cu).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "qdot_common.cuh"
#include "qdot_kernels.h"

using namespace qd;

namespace {

thread_local char g_err[256] = "";

int cuda_fail(cudaError_t e, const char* where) {
    std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return QDOT_ERR_CUDA;
}

#define QD_CHECK(call, where)                       \
    do {                                            \
        cudaError_t e_ = (call);                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

int validate(const qdot_config* c) {
    if (!c) return QDOT_ERR_ARG;
    // ToleranceConfig.__post_init__ (scoring.py:72-79)
    if (!std::isfinite(c->epsilon) || !(c->epsilon > 0.0) || c->epsilon > std::ldexp(1.0, 60)) return QDOT_ERR_ARG;
    if (c->input_mu != 10 && c->input_mu != 23 && c->input_mu != 52) return QDOT_ERR_ARG;
    if (c->split != 0 && c->split != 1) return QDOT_ERR_ARG;
    if (c->strategy == QDOT_STRATEGY_RANGED) {
        if (c->strategy_param < 1 || c->strategy_param > (1ll << 60)) return QDOT_ERR_ARG;   // binning.py:131
    } else if (c->strategy == QDOT_STRATEGY_SPLIT) {
        if (c->strategy_param < 0) return QDOT_ERR_ARG;                                       // binning.py:142
    } else if (c->strategy != QDOT_STRATEGY_EXACT) {
        return QDOT_ERR_ARG;                                                                   // binning.py:284
    }
    return QDOT_OK;
}

struct Staging {   // pinned host staging for the result block (per host thread)
    unsigned char* p = nullptr;
    ~Staging() { if (p) cudaFreeHost(p); }
};
thread_local Staging g_stage;

constexpr size_t RESULT_BLOCK = 256 + sizeof(qdot_bin) * (KEYS + 1);
constexpr int FIRST_BINS = 64;

}  // namespace

namespace qd {
// error reporting for the other translation units of the library
int report_cuda_error(cudaError_t e, const char* where) { return cuda_fail(e, where); }
}  // namespace qd

extern "C" {

int qdot_b200_version(void) { return QDOT_B200_VERSION; }

const char* qdot_b200_last_error(void) { return g_err; }

const char* qdot_b200_status_string(int s) {
    switch (s) {
        case QDOT_OK: return "ok";
        case QDOT_ERR_NONFINITE: return "inputs must be finite";
        case QDOT_ERR_OVERFLOW: return "rounded bin product overflowed its format";
        case QDOT_ERR_ARG: return "invalid argument";
        case QDOT_ERR_CUDA: return "CUDA error";
        case QDOT_ERR_EPS: return "floor_log2 needs a positive finite value";
        default: return "unknown status";
    }
}

size_t qdot_b200_workspace_bytes(void) { return (size_t)WS_BYTES; }

int qdot_b200_workspace_layout(qdot_ws_layout* o) {
    if (!o) return QDOT_ERR_ARG;
    o->total_bytes = WS_BYTES;
    o->a_offset = OFF_A;
    o->a_len = A_LEN;
    o->b_offset = OFF_B;
    o->b_len = B_LEN;
    o->result_offset = OFF_RESULT;
    o->result_bytes = (int64_t)RESULT_BLOCK;
    return QDOT_OK;
}

int qdot_b200_device_info(int* sm_count, int* cc_major, int* cc_minor) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        std::snprintf(g_err, sizeof(g_err), "no CUDA device");
        return QDOT_ERR_CUDA;
    }
    int dev = 0;
    QD_CHECK(cudaGetDevice(&dev), "cudaGetDevice");
    if (sm_count) QD_CHECK(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev), "attr");
    if (cc_major) QD_CHECK(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev), "attr");
    if (cc_minor) QD_CHECK(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev), "attr");
    return QDOT_OK;
}

int qdot_b200_begin(void* ws, void* stream) {
    if (!ws) return QDOT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // regions A and B are contiguous
    QD_CHECK(cudaMemsetAsync(static_cast<char*>(ws) + OFF_A, 0, (size_t)(BYTES_A + BYTES_B), st), "memset");
    return QDOT_OK;
}

int qdot_b200_pass1(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg,
                    int64_t n_total, void* ws, void* stream) {
    if (!ws || n < 0 || (n > 0 && (!x || (!norm && !y)))) return QDOT_ERR_ARG;
    P1Params prm;
    prm.epsilon = 1.0;
    prm.input_mu = 52;
    prm.mode = 1;   // no config: lean
    prm.n_total = n_total > n ? n_total : n;
    if (cfg) {
        int v = validate(cfg);
        if (v) return v;
        prm.epsilon = cfg->epsilon;
        prm.input_mu = cfg->input_mu;
        prm.mode = cfg->reserved;   // bits 0-1: 0 auto, 1 lean, 2 full; bits 2-3: queue 0 auto, 4 on, 8 off
        if (prm.mode < 0 || (prm.mode & 3) > 2 || (prm.mode >> 2) > 2) return QDOT_ERR_ARG;
    }
    WsPtrs w = ws_ptrs(ws);
    QD_CHECK(launch_pass1(x, norm ? x : y, n, norm != 0, w.a, w.b, prm, static_cast<cudaStream_t>(stream)), "pass1");
    return QDOT_OK;
}

int qdot_b200_score(void* ws, int64_t n_total, const qdot_config* cfg, void* stream) {
    if (!ws || n_total < 0) return QDOT_ERR_ARG;
    int v = validate(cfg);
    if (v) return v;
    WsPtrs w = ws_ptrs(ws);
    QD_CHECK(launch_score(w.a, w.lut_bin, w.lut_p2, w.meta, w.result, w.bins, n_total, *cfg,
                          static_cast<cudaStream_t>(stream)), "score");
    return QDOT_OK;
}

int qdot_b200_pass2(const double* x, const double* y, int64_t n, int norm, void* ws, void* stream) {
    if (!ws || n < 0 || (n > 0 && (!x || (!norm && !y)))) return QDOT_ERR_ARG;
    WsPtrs w = ws_ptrs(ws);
    QD_CHECK(launch_pass2(x, norm ? x : y, n, norm != 0, w.lut_p2, w.meta, w.b, static_cast<cudaStream_t>(stream)),
             "pass2");
    return QDOT_OK;
}

int qdot_b200_finalize(void* ws, void* stream) {
    if (!ws) return QDOT_ERR_ARG;
    WsPtrs w = ws_ptrs(ws);
    QD_CHECK(launch_finalize(w.a, w.b, w.lut_p2, w.meta, w.result, w.bins, static_cast<cudaStream_t>(stream)),
             "finalize");
    return QDOT_OK;
}

int qdot_b200_fetch(const void* ws, qdot_result* out, qdot_bin* bins, int32_t max_bins, void* stream) {
    if (!ws || !out) return QDOT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!g_stage.p) QD_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&g_stage.p), RESULT_BLOCK, cudaHostAllocDefault),
                             "cudaHostAlloc");
    const char* src = static_cast<const char*>(ws) + OFF_RESULT;
    int first = max_bins < FIRST_BINS ? (max_bins > 0 ? max_bins : 0) : FIRST_BINS;
    QD_CHECK(cudaMemcpyAsync(g_stage.p, src, 256 + sizeof(qdot_bin) * first, cudaMemcpyDeviceToHost, st), "D2H");
    QD_CHECK(cudaStreamSynchronize(st), "sync");
    std::memcpy(out, g_stage.p, sizeof(qdot_result));
    int nb = out->n_bins;
    int want = nb < max_bins ? nb : max_bins;
    if (want > first) {
        QD_CHECK(cudaMemcpyAsync(g_stage.p + 256 + sizeof(qdot_bin) * first, src + 256 + sizeof(qdot_bin) * first,
                                 sizeof(qdot_bin) * (want - first), cudaMemcpyDeviceToHost, st), "D2H bins");
        QD_CHECK(cudaStreamSynchronize(st), "sync");
    }
    if (bins && want > 0) std::memcpy(bins, g_stage.p + 256, sizeof(qdot_bin) * want);
    return QDOT_OK;
}

int qdot_b200_dot(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                  qdot_result* out, qdot_bin* bins, int32_t max_bins, void* stream) {
    int v = validate(cfg);
    if (v) return v;
    int r;
    if ((r = qdot_b200_begin(ws, stream))) return r;
    if ((r = qdot_b200_pass1(x, y, n, norm, cfg, n, ws, stream))) return r;
    if ((r = qdot_b200_score(ws, n, cfg, stream))) return r;
    if ((r = qdot_b200_pass2(x, y, n, norm, ws, stream))) return r;
    if ((r = qdot_b200_finalize(ws, stream))) return r;
    return qdot_b200_fetch(ws, out, bins, max_bins, stream);
}

int qdot_b200_dot_host(const double* hx, const double* hy, int64_t n, int norm, const qdot_config* cfg,
                       qdot_result* out, qdot_bin* bins, int32_t max_bins) {
    int v = validate(cfg);
    if (v) return v;
    if (n < 0 || (n > 0 && (!hx || (!norm && !hy)))) return QDOT_ERR_ARG;
    int sm = 0;
    if ((v = qdot_b200_device_info(&sm, nullptr, nullptr))) return v;
    double *dx = nullptr, *dy = nullptr;
    void* ws = nullptr;
    cudaStream_t cs = nullptr, ks = nullptr;
    std::vector<cudaEvent_t> evs;
    int rc = QDOT_OK;
    const int64_t nb = n > 0 ? n : 1;
    const int64_t CH = 1ll << 22;   // elements per overlapped chunk
    auto fail = [&](cudaError_t e, const char* w) { rc = cuda_fail(e, w); };
    cudaError_t e;
    if ((e = cudaMalloc(&dx, sizeof(double) * nb)) != cudaSuccess) { fail(e, "malloc x"); goto out_; }
    if (!norm && (e = cudaMalloc(&dy, sizeof(double) * nb)) != cudaSuccess) { fail(e, "malloc y"); goto out_; }
    if ((e = cudaMalloc(&ws, WS_BYTES)) != cudaSuccess) { fail(e, "malloc ws"); goto out_; }
    if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) { fail(e, "stream"); goto out_; }
    if ((e = cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking)) != cudaSuccess) { fail(e, "stream"); goto out_; }
    if ((rc = qdot_b200_begin(ws, ks))) goto out_;
    // copy chunk c on the copy stream while pass 1 consumes chunk c-1
    for (int64_t off = 0; off < n; off += CH) {
        int64_t len = n - off < CH ? n - off : CH;
        cudaEvent_t ev;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) { fail(e, "event"); goto out_; }
        evs.push_back(ev);
        if ((e = cudaMemcpyAsync(dx + off, hx + off, sizeof(double) * len, cudaMemcpyHostToDevice, cs)) != cudaSuccess) {
            fail(e, "H2D x"); goto out_;
        }
        if (!norm && (e = cudaMemcpyAsync(dy + off, hy + off, sizeof(double) * len, cudaMemcpyHostToDevice, cs)) !=
                         cudaSuccess) {
            fail(e, "H2D y"); goto out_;
        }
        cudaEventRecord(ev, cs);
        cudaStreamWaitEvent(ks, ev, 0);
        if ((rc = qdot_b200_pass1(dx + off, norm ? nullptr : dy + off, len, norm, cfg, n, ws, ks))) goto out_;
    }
    if ((rc = qdot_b200_score(ws, n, cfg, ks))) goto out_;
    if ((rc = qdot_b200_pass2(dx, norm ? nullptr : dy, n, norm, ws, ks))) goto out_;
    if ((rc = qdot_b200_finalize(ws, ks))) goto out_;
    rc = qdot_b200_fetch(ws, out, bins, max_bins, ks);
out_:
    if (ks) cudaStreamSynchronize(ks);
    if (cs) cudaStreamSynchronize(cs);
    for (auto ev : evs) cudaEventDestroy(ev);
    if (cs) cudaStreamDestroy(cs);
    if (ks) cudaStreamDestroy(ks);
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(ws);
    return rc;
}

int qdot_b200_bin_ids(const double* x, const double* y, int64_t n, int norm, const int32_t* lut_bin,
                      int32_t* bin_ids, void* stream) {
    if (!lut_bin || !bin_ids || n < 0) return QDOT_ERR_ARG;
    QD_CHECK(launch_bin_ids(x, norm ? x : y, n, norm != 0, lut_bin, bin_ids, static_cast<cudaStream_t>(stream)),
             "bin_ids");
    return QDOT_OK;
}

int qdot_b200_batched(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld, int norm,
                      const qdot_config* cfg, double* values, int64_t* counts, int32_t* info, void* stream) {
    int v = validate(cfg);
    if (v) return v;
    if (rows < 0 || len < 0 || ld < len || (rows > 0 && (!X || (!norm && !Y) || !values || !counts || !info)))
        return QDOT_ERR_ARG;
    QD_CHECK(launch_batched(X, Y, rows, len, ld, norm != 0, *cfg, values, counts, info,
                            static_cast<cudaStream_t>(stream)), "batched");
    return QDOT_OK;
}

double qdot_b200_ldexp_rn(double acc, int64_t u, int* overflow) {
    int o = 0;
    double r = ldexp_rn(acc, u, &o);
    if (overflow) *overflow = o;
    return r;
}

}  // extern "C"
