// qdot_host.cu -- host-side runtime of the host-input path: pageable host
// vectors -> device, overlapped with pass 1.
//
// The reference's callers hand qdot() numpy arrays, i.e. pageable host memory
// (kernel.py:195-196).  A cudaMemcpyAsync from pageable memory is staged by
// the driver through its own small pinned buffers, synchronously, at ~10 GB/s.
// Here the library stages itself:
//   * a ring of STAGE_BUFS pinned buffers per host thread (x and y halves of
//     STAGE_CHUNK elements each);
//   * a process-wide pool of host threads that fills a buffer with parallel
//     memcpys (several memory channels in flight) while the DMA engine drains
//     the previous buffer to the device and pass 1 consumes the chunk before;
//   * per-buffer events: a buffer is refilled only after its H2D completed.
// Pinned (page-locked / registered) inputs skip the staging and are copied
// chunk by chunk directly.  The call returns once the caller's host memory
// has been read and every copy and pass-1 launch is enqueued.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "qdot_common.cuh"

namespace qd {
int report_cuda_error(cudaError_t e, const char* where);
}

extern "C" int qdot_b200_pass1(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg,
                               int64_t n_total, void* ws, void* stream);

namespace {

constexpr int64_t STAGE_CHUNK = 1ll << 22;   // elements per array per staged chunk (32 MiB)
constexpr int STAGE_BUFS = 3;

// parallel memcpy: the caller's thread copies part 0, the workers the rest
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool p;
        return p;
    }
    int threads() const { return nthreads_; }

    void copy(void* dst, const void* src, size_t bytes) {
        std::lock_guard<std::mutex> one(busy_);              // one parallel copy at a time
        if (nthreads_ <= 1 || bytes < (1u << 20)) {
            std::memcpy(dst, src, bytes);
            return;
        }
        {
            std::lock_guard<std::mutex> l(m_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            pending_ = nthreads_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0);
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [&] { return pending_ == 0; });
    }

private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        nthreads_ = (int)std::max(1u, std::min(8u, hw / 2));   // 8: measured best on the B200 host
        if (const char* e = std::getenv("QDOT_B200_COPY_THREADS")) nthreads_ = std::max(1, std::min(64, std::atoi(e)));
        for (int i = 1; i < nthreads_; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> l(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    void part(int i) {
        const size_t per = (bytes_ / nthreads_ + 63) & ~size_t(63);
        const size_t lo = std::min(bytes_, per * (size_t)i), hi = std::min(bytes_, lo + per);
        if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> l(m_);
            cv_.wait(l, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            l.unlock();
            part(i);
            l.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    int nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex busy_, m_;
    std::condition_variable cv_, done_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
};

struct Stager {          // per host thread and device
    int dev = -1;
    double* buf[STAGE_BUFS] = {};
    cudaEvent_t freed[STAGE_BUFS] = {};
    std::vector<cudaEvent_t> landed;
    cudaStream_t copy = nullptr;
    cudaEvent_t start = nullptr;
    void release() {
        for (int b = 0; b < STAGE_BUFS; ++b) {
            if (freed[b]) cudaEventDestroy(freed[b]);
            if (buf[b]) cudaFreeHost(buf[b]);
            buf[b] = nullptr;
            freed[b] = nullptr;
        }
        for (auto e : landed) cudaEventDestroy(e);
        landed.clear();
        if (copy) cudaStreamDestroy(copy);
        if (start) cudaEventDestroy(start);
        copy = nullptr;
        start = nullptr;
    }
    ~Stager() { release(); }
};
thread_local Stager g_stager;

int fail(cudaError_t e, const char* where) { return qd::report_cuda_error(e, where); }

#define QH_CHECK(call, where)                          \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return fail(e_, where); \
    } while (0)

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int stager_init(Stager& S, int dev, int64_t nchunks) {
    if (S.dev != dev) {
        S.release();
        S.dev = dev;
    }
    if (!S.copy) QH_CHECK(cudaStreamCreateWithFlags(&S.copy, cudaStreamNonBlocking), "stage stream");
    if (!S.start) QH_CHECK(cudaEventCreateWithFlags(&S.start, cudaEventDisableTiming), "stage event");
    for (int b = 0; b < STAGE_BUFS; ++b) {
        if (!S.buf[b])
            QH_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&S.buf[b]), 2 * STAGE_CHUNK * sizeof(double),
                                   cudaHostAllocPortable), "stage buffer");
        if (!S.freed[b]) QH_CHECK(cudaEventCreateWithFlags(&S.freed[b], cudaEventDisableTiming), "stage event");
    }
    while ((int64_t)S.landed.size() < nchunks) {
        cudaEvent_t e;
        QH_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "stage event");
        S.landed.push_back(e);
    }
    return QDOT_OK;
}

}  // namespace

extern "C" {

int qdot_b200_pass1_host(const double* hx, const double* hy, int64_t n, int norm, const qdot_config* cfg,
                         int64_t n_total, void* ws, double* dx, double* dy, void* stream) {
    if (!ws || n < 0 || (n > 0 && (!hx || !dx || (!norm && (!hy || !dy))))) return QDOT_ERR_ARG;
    if (n == 0) return QDOT_OK;
    int dev = 0;
    QH_CHECK(cudaGetDevice(&dev), "cudaGetDevice");
    Stager& S = g_stager;
    const int64_t nchunks = (n + STAGE_CHUNK - 1) / STAGE_CHUNK;
    int rc = stager_init(S, dev, nchunks);
    if (rc) return rc;
    cudaStream_t ks = static_cast<cudaStream_t>(stream);
    // the device buffers may still be read by earlier work on the caller's stream
    QH_CHECK(cudaEventRecord(S.start, ks), "event");
    QH_CHECK(cudaStreamWaitEvent(S.copy, S.start, 0), "wait");
    const bool pinned = is_pinned(hx) && (norm || is_pinned(hy));
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t off = c * STAGE_CHUNK;
        const int64_t len = std::min<int64_t>(STAGE_CHUNK, n - off);
        const size_t bytes = (size_t)len * sizeof(double);
        if (pinned) {
            QH_CHECK(cudaMemcpyAsync(dx + off, hx + off, bytes, cudaMemcpyHostToDevice, S.copy), "H2D x");
            if (!norm) QH_CHECK(cudaMemcpyAsync(dy + off, hy + off, bytes, cudaMemcpyHostToDevice, S.copy), "H2D y");
        } else {
            const int b = (int)(c % STAGE_BUFS);
            QH_CHECK(cudaEventSynchronize(S.freed[b]), "stage wait");   // its last H2D (this or an earlier call) done
            double* sx = S.buf[b];
            double* sy = S.buf[b] + STAGE_CHUNK;
            CopyPool::get().copy(sx, hx + off, bytes);
            if (!norm) CopyPool::get().copy(sy, hy + off, bytes);
            QH_CHECK(cudaMemcpyAsync(dx + off, sx, bytes, cudaMemcpyHostToDevice, S.copy), "H2D x");
            if (!norm) QH_CHECK(cudaMemcpyAsync(dy + off, sy, bytes, cudaMemcpyHostToDevice, S.copy), "H2D y");
            QH_CHECK(cudaEventRecord(S.freed[b], S.copy), "event");
        }
        QH_CHECK(cudaEventRecord(S.landed[c], S.copy), "event");
        QH_CHECK(cudaStreamWaitEvent(ks, S.landed[c], 0), "wait");
        if ((rc = qdot_b200_pass1(dx + off, norm ? dx + off : dy + off, len, norm, cfg, n_total, ws, stream)))
            return rc;
    }
    return QDOT_OK;
}

int qdot_b200_host_copy_threads(void) { return CopyPool::get().threads(); }

}  // extern "C"
