// qdot_capi.cu -- extern "C" entry points declared in include/qdot_b200.h.
//
// Host-side orchestration only: validation, launch order, result transfer.
// All arithmetic on the data happens in the sm_100a kernels (qdot_kernels.cu).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
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
    static_assert((BYTES_A + BYTES_B + BYTES_LOCAL) % 16 == 0 && OFF_A % 16 == 0, "begin zeroes 16-byte words");
    QD_CHECK(launch_begin(static_cast<char*>(ws) + OFF_A, (size_t)(BYTES_A + BYTES_B + BYTES_LOCAL), st), "begin");
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
    {
        WsPtrs w0 = ws_ptrs(ws);
        prm.list = w0.list;
        prm.list_fill = w0.list_fill;
        prm.collect = 0;
        prm.per_bin = 0;
    }
    if (cfg) {
        int v = validate(cfg);
        if (v) return v;
        prm.epsilon = cfg->epsilon;
        prm.input_mu = cfg->input_mu;
        prm.collect = cfg->strategy != QDOT_STRATEGY_EXACT;
        prm.per_bin = cfg->split == 1 && cfg->strategy == QDOT_STRATEGY_EXACT;
        // bits 0-1: 0 auto, 1 lean, 2 full; bits 2-3: queue 0 auto, 4 on, 8 off; bit 4: wide lean window;
        // bit 5: norm mode without the exponent-indexed lean loop (A/B); bits 6-7: its L2 prefetch
        // distance, bits 8-9 its cache policy
        prm.mode = cfg->reserved;
        if (prm.mode < 0 || (prm.mode & 3) > 2 || ((prm.mode >> 2) & 3) > 2 || ((prm.mode >> 8) & 3) > 2 ||
            (prm.mode >> 10))
            return QDOT_ERR_ARG;
    }
    WsPtrs w = ws_ptrs(ws);
    QD_CHECK(launch_pass1(x, norm ? x : y, n, norm != 0, w.a, w.b, prm, static_cast<cudaStream_t>(stream)), "pass1");
    return QDOT_OK;
}

// the one-launch cluster path (qdot_small.cuh): single device, exact strategy,
// auto pass-1 mode, 1 <= n <= SMALL_AUTO (where it measured faster than the
// four-launch pipeline: 12.7 vs 17.8 us per call at n = 1e4, APM n = 2000 61 vs
// 67 us per iteration; at n = 32768 the ACG iteration was faster without it);
// QDOT_B200_NO_SMALL=1 turns it off, QDOT_B200_SMALL_AUTO=m moves the limit (experiments)
constexpr int64_t SMALL_AUTO = 16384;
static bool small_ok(int64_t n, const qdot_config* cfg) {
    static int off = -1;
    static int64_t lim = 0;
    if (off < 0) {
        const char* e = std::getenv("QDOT_B200_NO_SMALL");
        off = (e && e[0] && e[0] != '0') ? 1 : 0;
        const char* m = std::getenv("QDOT_B200_SMALL_AUTO");
        lim = m ? std::atoll(m) : SMALL_AUTO;
        if (lim > small_max()) lim = small_max();
    }
    return !off && cfg && cfg->strategy == QDOT_STRATEGY_EXACT && cfg->reserved == 0 && n >= 1 && n <= lim;
}

int64_t qdot_b200_small_max(void) { return small_max(); }

int qdot_b200_small(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                    void* stream) {
    int v = validate(cfg);
    if (v) return v;
    if (!ws || n < 1 || n > small_max() || !x || (!norm && !y) || cfg->strategy != QDOT_STRATEGY_EXACT)
        return QDOT_ERR_ARG;
    WsPtrs w = ws_ptrs(ws);
    QD_CHECK(launch_small(x, norm ? x : y, n, norm != 0, w.a, w.b, w.lut_bin, w.lut_p2, w.meta, w.result, w.bins, *cfg,
                          static_cast<cudaStream_t>(stream)), "small");
    return QDOT_OK;
}

static int enqueue_impl(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                        void* stream, bool begin) {
    int r;
    if (small_ok(n, cfg)) {
        if ((r = qdot_b200_small(x, y, n, norm, cfg, ws, stream))) return r;
    } else {
        if (begin && (r = qdot_b200_begin(ws, stream))) return r;
        if ((r = qdot_b200_pass1(x, y, n, norm, cfg, n, ws, stream))) return r;
    }
    if ((r = qdot_b200_score_finalize(ws, n, cfg, stream))) return r;
    return qdot_b200_pass2_finalize(x, y, n, norm, ws, stream);
}

int qdot_b200_enqueue(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                      void* stream) {
    return enqueue_impl(x, y, n, norm, cfg, ws, stream, true);
}

int qdot_b200_enqueue_zeroed(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                             void* stream) {
    return enqueue_impl(x, y, n, norm, cfg, ws, stream, false);
}

static int score_impl(void* ws, int64_t n_total, const qdot_config* cfg, bool fuse, void* stream) {
    if (!ws || n_total < 0) return QDOT_ERR_ARG;
    int v = validate(cfg);
    if (v) return v;
    WsPtrs w = ws_ptrs(ws);
    QD_CHECK(launch_score(w.a, w.b, w.lut_bin, w.lut_p2, w.meta, w.result, w.bins, n_total, *cfg, fuse,
                          static_cast<cudaStream_t>(stream)), "score");
    return QDOT_OK;
}

int qdot_b200_score(void* ws, int64_t n_total, const qdot_config* cfg, void* stream) {
    return score_impl(ws, n_total, cfg, false, stream);
}

int qdot_b200_score_finalize(void* ws, int64_t n_total, const qdot_config* cfg, void* stream) {
    return score_impl(ws, n_total, cfg, true, stream);
}

static int pass2_impl(const double* x, const double* y, int64_t n, int norm, void* ws, bool fin, void* stream) {
    if (!ws || n < 0 || (n > 0 && (!x || (!norm && !y)))) return QDOT_ERR_ARG;
    WsPtrs w = ws_ptrs(ws);
    P2Fin f;
    if (fin) { f.A = w.a; f.res = w.result; f.bins = w.bins; }
    QD_CHECK(launch_pass2(x, norm ? x : y, n, norm != 0, w.lut_p2, w.meta, w.b, w.list, w.list_fill, f,
                          static_cast<cudaStream_t>(stream)),
             "pass2");
    return QDOT_OK;
}

int qdot_b200_pass2(const double* x, const double* y, int64_t n, int norm, void* ws, void* stream) {
    return pass2_impl(x, y, n, norm, ws, false, stream);
}

int qdot_b200_pass2_finalize(const double* x, const double* y, int64_t n, int norm, void* ws, void* stream) {
    return pass2_impl(x, y, n, norm, ws, true, stream);
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

// ---- one-call path: a CUDA graph per (x, y, n, norm, cfg, ws, device), cached per
// host thread, whose last node publishes the result block into host-mapped
// memory; the host spins on its sequence word instead of a memcpy + sync.
namespace {

constexpr int PUBLISH_BYTES = 256 + (int)sizeof(qdot_bin) * FIRST_BINS;   // header + first bins
constexpr int GRAPH_CACHE = 16;

struct GraphKey {
    const double* x;
    const double* y;
    int64_t n;
    int norm;
    int dev;
    void* ws;
    qdot_config cfg;
    bool operator==(const GraphKey& o) const {
        return x == o.x && y == o.y && n == o.n && norm == o.norm && dev == o.dev && ws == o.ws &&
               std::memcmp(&cfg, &o.cfg, sizeof(cfg)) == 0;
    }
};

struct FastState {
    int dev = -1;
    unsigned char* host = nullptr;      // mapped: [0, PUBLISH_BYTES) block, then the sequence word
    unsigned char* host_dev = nullptr;
    uint32_t* dev_seq = nullptr;
    uint32_t expected = 0;
    cudaStream_t cap = nullptr;
    struct Entry { GraphKey k; cudaGraphExec_t exec; uint64_t use; };
    std::vector<Entry> cache;
    std::vector<GraphKey> seen;   // keys met once: a graph is captured on the second call only
    uint64_t tick = 0;
    void clear() {
        for (auto& e : cache) cudaGraphExecDestroy(e.exec);
        cache.clear();
        seen.clear();
        if (cap) cudaStreamDestroy(cap);
        if (dev_seq) cudaFree(dev_seq);
        if (host) cudaFreeHost(host);
        cap = nullptr; dev_seq = nullptr; host = nullptr; host_dev = nullptr; expected = 0;
    }
    ~FastState() { clear(); }
};
thread_local FastState g_fast;

int fast_init(int dev) {
    FastState& F = g_fast;
    if (F.dev == dev && F.host) return QDOT_OK;
    F.clear();
    F.dev = dev;
    QD_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&F.host), PUBLISH_BYTES + 64, cudaHostAllocMapped), "hostalloc");
    std::memset(F.host, 0, PUBLISH_BYTES + 64);
    QD_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&F.host_dev), F.host, 0), "mapped ptr");
    QD_CHECK(cudaMalloc(reinterpret_cast<void**>(&F.dev_seq), sizeof(uint32_t)), "seq");
    QD_CHECK(cudaMemset(F.dev_seq, 0, sizeof(uint32_t)), "seq");
    QD_CHECK(cudaStreamCreateWithFlags(&F.cap, cudaStreamNonBlocking), "capture stream");
    return QDOT_OK;
}

int enqueue_dot(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                cudaStream_t st) {
    int r;
    void* s = static_cast<void*>(st);
    if ((r = qdot_b200_enqueue(x, y, n, norm, cfg, ws, s))) return r;
    FastState& F = g_fast;
    QD_CHECK(launch_publish(static_cast<const char*>(ws) + OFF_RESULT, PUBLISH_BYTES, F.host_dev, F.dev_seq,
                            reinterpret_cast<uint32_t*>(F.host_dev + PUBLISH_BYTES), st), "publish");
    return QDOT_OK;
}

cudaGraphExec_t graph_for(const GraphKey& k, const qdot_config* cfg) {
    FastState& F = g_fast;
    for (auto& e : F.cache)
        if (e.k == k) { e.use = ++F.tick; return e.exec; }
    // a capture costs more than a few eager launches: only repeated calls get one
    bool repeat = false;
    for (auto& sk : F.seen)
        if (sk == k) { repeat = true; break; }
    if (!repeat) {
        if (F.seen.size() >= 64) F.seen.erase(F.seen.begin());
        F.seen.push_back(k);
        return nullptr;
    }
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(F.cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return nullptr;
    int r = enqueue_dot(k.x, k.y, k.n, k.norm, cfg, k.ws, F.cap);
    cudaError_t e = cudaStreamEndCapture(F.cap, &g);
    if (r != QDOT_OK || e != cudaSuccess || !g) { cudaGetLastError(); if (g) cudaGraphDestroy(g); return nullptr; }
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { cudaGetLastError(); return nullptr; }
    if ((int)F.cache.size() >= GRAPH_CACHE) {
        size_t old = 0;
        for (size_t i = 1; i < F.cache.size(); ++i) if (F.cache[i].use < F.cache[old].use) old = i;
        cudaGraphExecDestroy(F.cache[old].exec);
        F.cache.erase(F.cache.begin() + old);
    }
    for (size_t i = 0; i < F.seen.size(); ++i)
        if (F.seen[i] == k) { F.seen.erase(F.seen.begin() + i); break; }
    F.cache.push_back({k, exec, ++F.tick});
    return exec;
}

// wait for the published block (spinning on the mapped sequence word), then copy out
int collect(cudaStream_t st, const void* ws, qdot_result* out, qdot_bin* bins, int32_t max_bins) {
    FastState& F = g_fast;
    const uint32_t want = ++F.expected;
    volatile uint32_t* seq = reinterpret_cast<volatile uint32_t*>(F.host + PUBLISH_BYTES);
    for (uint64_t it = 1; *seq != want; ++it) {
        if ((it & 1023) == 0) {
            cudaError_t e = cudaStreamQuery(st);
            if (e == cudaSuccess && *seq != want) {          // stream idle but nothing published
                F.expected = *seq;
                std::snprintf(g_err, sizeof(g_err), "result not published");
                return QDOT_ERR_CUDA;
            }
            if (e != cudaSuccess && e != cudaErrorNotReady) { F.expected = *seq; return cuda_fail(e, "qdot graph"); }
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    std::memcpy(out, F.host, sizeof(qdot_result));
    const int nb = out->n_bins;
    const int want_bins = nb < max_bins ? nb : max_bins;
    const int first = want_bins < FIRST_BINS ? want_bins : FIRST_BINS;
    if (bins && first > 0) std::memcpy(bins, F.host + 256, sizeof(qdot_bin) * first);
    if (bins && want_bins > first) {   // rare: many bins -> one more D2H for the rest
        QD_CHECK(cudaMemcpyAsync(bins + first, static_cast<const char*>(ws) + OFF_BINS + sizeof(qdot_bin) * first,
                                 sizeof(qdot_bin) * (want_bins - first), cudaMemcpyDeviceToHost, st), "D2H bins");
        QD_CHECK(cudaStreamSynchronize(st), "sync");
    }
    return QDOT_OK;
}

}  // namespace

int qdot_b200_dot(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                  qdot_result* out, qdot_bin* bins, int32_t max_bins, void* stream) {
    int v = validate(cfg);
    if (v) return v;
    if (!ws || !out || n < 0 || (n > 0 && (!x || (!norm && !y)))) return QDOT_ERR_ARG;
    int dev = 0;
    QD_CHECK(cudaGetDevice(&dev), "cudaGetDevice");
    if ((v = fast_init(dev))) return v;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    GraphKey k{x, norm ? x : y, n, norm, dev, ws, *cfg};
    cudaGraphExec_t exec = graph_for(k, cfg);
    if (exec) {
        QD_CHECK(cudaGraphLaunch(exec, st), "graph launch");
    } else if ((v = enqueue_dot(x, norm ? x : y, n, norm, cfg, ws, st))) {   // first call / no capture: eagerly
        return v;
    }
    return collect(st, ws, out, bins, max_bins);
}

// per-host-thread device buffers, workspace, streams and chunk events of the
// host-input path (grow-only; released at thread exit)
namespace {
struct HostPath {
    int dev = -1;
    double* dx = nullptr;
    double* dy = nullptr;
    int64_t cap = 0;
    void* ws = nullptr;
    cudaStream_t ks = nullptr;
    void release() {
        if (ks) cudaStreamDestroy(ks);
        cudaFree(dx); cudaFree(dy); cudaFree(ws);
        dx = dy = nullptr; ws = nullptr; ks = nullptr; cap = 0;
    }
    ~HostPath() { release(); }
};
thread_local HostPath g_host;
}  // namespace

int qdot_b200_dot_host(const double* hx, const double* hy, int64_t n, int norm, const qdot_config* cfg,
                       qdot_result* out, qdot_bin* bins, int32_t max_bins) {
    int v = validate(cfg);
    if (v) return v;
    if (n < 0 || (n > 0 && (!hx || (!norm && !hy)))) return QDOT_ERR_ARG;
    int sm = 0;
    if ((v = qdot_b200_device_info(&sm, nullptr, nullptr))) return v;
    int dev = 0;
    QD_CHECK(cudaGetDevice(&dev), "cudaGetDevice");
    HostPath& H = g_host;
    if (H.dev != dev) { H.release(); H.dev = dev; }
    const int64_t nb = n > 0 ? n : 1;
    if (nb > H.cap) {
        cudaFree(H.dx); cudaFree(H.dy);
        H.dx = H.dy = nullptr; H.cap = 0;
        QD_CHECK(cudaMalloc(&H.dx, sizeof(double) * nb), "malloc x");
        QD_CHECK(cudaMalloc(&H.dy, sizeof(double) * nb), "malloc y");
        H.cap = nb;
    }
    if (!H.ws) QD_CHECK(cudaMalloc(&H.ws, WS_BYTES), "malloc ws");
    if (!H.ks) QD_CHECK(cudaStreamCreateWithFlags(&H.ks, cudaStreamNonBlocking), "stream");
    double *dx = H.dx, *dy = H.dy;
    void* ws = H.ws;
    cudaStream_t ks = H.ks;
    int rc = QDOT_OK;
    if ((rc = qdot_b200_begin(ws, ks))) return rc;
    // chunked H2D (pageable inputs through the library's pinned staging ring)
    // overlapped with pass 1 (qdot_host.cu)
    rc = qdot_b200_pass1_host(hx, hy, n, norm, cfg, n, ws, dx, dy, ks);
    if (!rc) rc = qdot_b200_score_finalize(ws, n, cfg, ks);
    if (!rc) rc = qdot_b200_pass2_finalize(dx, norm ? nullptr : dy, n, norm, ws, ks);
    if (!rc) rc = qdot_b200_fetch(ws, out, bins, max_bins, ks);
    cudaStreamSynchronize(ks);
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
    QD_CHECK(launch_batched(X, Y, rows, len, ld, norm != 0, *cfg, values, counts, info, nullptr,
                            static_cast<cudaStream_t>(stream)), "batched");
    return QDOT_OK;
}

int qdot_b200_batched_bins(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld, int norm,
                           const qdot_config* cfg, double* values, int64_t* counts, int32_t* info, qdot_bin* bins,
                           void* stream) {
    int v = validate(cfg);
    if (v) return v;
    if (rows < 0 || len < 0 || ld < len ||
        (rows > 0 && (!X || (!norm && !Y) || !values || !counts || !info || !bins)))
        return QDOT_ERR_ARG;
    QD_CHECK(launch_batched(X, Y, rows, len, ld, norm != 0, *cfg, values, counts, info, bins,
                            static_cast<cudaStream_t>(stream)), "batched_bins");
    return QDOT_OK;
}

// host: the report's error-bound sums over a fetched bin table
// (scoring.py:171-199, kernel.py:205-222): term_b = M_b * ldexp(eps(p_b),
// u_b - shift + 1); out[0] = fsum(terms) (correctly rounded: exact big-integer
// sum, one rounding), out[1] = left-to-right sum from 0.0.  An ldexp that
// overflows, or an fsum of finite terms that does, is QDOT_ERR_OVERFLOW
// (the reference raises OverflowError).
int qdot_b200_bound_sums(const qdot_bin* bins, int32_t n_bins, int64_t shift, double* out) {
    if (!out || n_bins < 0 || (n_bins > 0 && !bins)) return QDOT_ERR_ARG;
    static const int kMu[4] = {0, 10, 23, 52};    // PrecisionLevel mantissa bits: eps = 2^-mu
    BigSum<72> acc;
    acc.init(-1074, 72);
    double plain = 0.0;
    bool inf = false;
    for (int32_t i = 0; i < n_bins; ++i) {
        const int p = bins[i].precision;
        if (p < 0 || p > 3) return QDOT_ERR_ARG;
        const int64_t k = bins[i].upper - shift + 1 - kMu[p];
        if (k > 1023) return QDOT_ERR_OVERFLOW;                       // math.ldexp overflow
        const double pw = k < -1100 ? 0.0 : std::ldexp(1.0, (int)k);   // exact, or rounded below 2^-1074
        const double t = (double)bins[i].cardinality * pw;
        plain += t;
        if (std::isinf(t)) { inf = true; continue; }
        if (t == 0.0) continue;
        uint64_t b;
        std::memcpy(&b, &t, 8);
        const int e = (int)((b >> 52) & 0x7FF);
        uint64_t m = b & ((1ull << 52) - 1);
        int ex = -1074;
        if (e) { m |= 1ull << 52; ex = e - 1075; }
        acc.add((__int128)m, ex);                                     // terms are >= 0
    }
    if (inf) {
        out[0] = INFINITY;
    } else {
        int ovf = 0;
        out[0] = acc.round(52, -1022, 1023, &ovf);
        if (ovf) return QDOT_ERR_OVERFLOW;                            // fsum intermediate overflow
    }
    out[1] = plain;
    return QDOT_OK;
}

// two shifts in one call (the report's rel terms at e_max, then abs at 0):
// out[0..1] for shift_a, out[2..3] for shift_b; the first failure is returned
int qdot_b200_bound_sums2(const qdot_bin* bins, int32_t n_bins, int64_t shift_a, int64_t shift_b, double* out) {
    if (!out) return QDOT_ERR_ARG;
    const int r = qdot_b200_bound_sums(bins, n_bins, shift_a, out);
    return r ? r : qdot_b200_bound_sums(bins, n_bins, shift_b, out + 2);
}

double qdot_b200_ldexp_rn(double acc, int64_t u, int* overflow) {
    int o = 0;
    double r = ldexp_rn(acc, u, &o);
    if (overflow) *overflow = o;
    return r;
}

}  // extern "C"
