// qdot_exact.cu -- exact (correctly rounded) dot product on the device: the
// verification oracle kernel.reference_dot (kernel.py:98-133) without the
// host round trip, for checking qdot at sizes the CPU cannot hold.
//
// Every product of two finite doubles is exact as an integer:
//     x = mx 2^qx, y = my 2^qy  (mx, my < 2^53, subnormals included)
//     x*y = P 2^q,  P = mx*my < 2^106,  q = qx + qy in [-2148, 1942]
// Pass `k_exact` streams x, y once and accumulates P per key q + 2148 exactly:
//   * a 16-key private window (chosen per CTA from its first tile) in
//     per-thread 128-bit slots in shared memory (plain LDS/STS),
//   * everything else straight into the global per-key accumulators,
// flushing the slots every <= 511 elements per thread (|slot| < 2^115) into
// global int64 accumulators of four 32-bit limbs per key (each limb sum stays
// below 2^63 for any n < 2^53).  Integer sums: order independent, bit-exact
// for any grid and any number of ranks (the accumulator region is what a
// multi-GPU run SUM-allreduces).
// `k_exact_finalize` (one CTA) folds the per-key limbs into one big integer
// and rounds it once to double (round-half-even, gradual underflow, overflow
// flagged) -- the value math.fsum / float(Fraction) give in the reference.
// `k_exact_plain` reproduces ReferenceResult.plain, the left-to-right double
// sum of the rounded products (kernel.py:122,127-129): inherently serial, one
// thread, chained across calls through the workspace.

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "qdot_common.cuh"

namespace qd {
int report_cuda_error(cudaError_t e, const char* where);
}

namespace {

using namespace qd;

constexpr int XT = 256;                 // threads per CTA
constexpr int XW = 16;                  // private window keys
constexpr int XV = 4;                   // double2 per thread per tile
constexpr int XTILE = XT * 2 * XV;      // elements per tile
constexpr int XKEYS = 4096;             // key = q + 2148 in [0, 4090]
constexpr int XFLUSH = 511 / (2 * XV);  // tiles between slot flushes
// private-window keys: exponent-field sums in [1150, 3066], where no element
// can send the reference to its Fraction path (see ref_fallback)
constexpr int X_SAFE_LO = 1150 - 2;
constexpr int X_SAFE_HI = 3066 - 2 - XW + 1;

// workspace (int64 words): the exchange region first, then local state
constexpr int64_t X_ACC = 0;                       // [XKEYS][4] limbs
constexpr int64_t X_NONFINITE = XKEYS * 4;         // non-finite element count
constexpr int64_t X_FALLBACK = X_NONFINITE + 1;    // elements that send the reference to its Fraction path
constexpr int64_t X_REGION = X_NONFINITE + 8;      // words exchanged between ranks
constexpr int64_t X_PLAIN = X_REGION;              // running plain sum (double bits) + started flag
constexpr int64_t X_PLAIN_STARTED = X_REGION + 1;
constexpr int64_t X_RESULT = X_REGION + 8;         // qdot_exact_result (64 bytes)
constexpr int64_t X_WORDS = X_RESULT + 16;

constexpr int XCW = 128;                // cold window keys (per-CTA limb table)

struct __align__(16) XShared {
    ulonglong2 priv[XW * XT];      // 128-bit signed slot (lo, hi) per (key, thread)
    // cold window: P = sum l_i 2^(14 i), l_0..l_6 unsigned 14-bit, l_7 signed,
    // summed with native 32-bit shared atomics (< 2^17 adds between flushes)
    uint32_t cold[8][XCW];
    double2 q[XT / 32][32];        // per-warp queue of cold elements (queue mode)
    int base;
    int cbase;
    int queue;
};

__device__ __forceinline__ void split_dbl(uint64_t b, uint64_t& m, int& f) {
    f = (int)((b >> 52) & 0x7FF);
    m = b & ((1ull << 52) - 1);
    if (f) m |= 1ull << 52; else f = 1;
}

// signed 128-bit product of two doubles' integer mantissas
__device__ __forceinline__ void prod128(uint64_t mx, uint64_t my, bool neg, uint64_t& lo, uint64_t& hi) {
    lo = mx * my;
    hi = __umul64hi(mx, my);
    if (neg) {
        lo = ~lo + 1;
        hi = ~hi + (lo == 0 ? 1 : 0);
    }
}

__device__ __forceinline__ void push_limbs(int64_t* __restrict__ acc, int key, uint64_t lo, uint64_t hi) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(acc + X_ACC + 4 * (int64_t)key);
    const uint64_t l0 = lo & 0xFFFFFFFFull, l1 = lo >> 32, l2 = hi & 0xFFFFFFFFull;
    const int64_t l3 = (int64_t)hi >> 32;                  // signed top limb
    if (l0) atomicAdd(a + 0, (unsigned long long)l0);
    if (l1) atomicAdd(a + 1, (unsigned long long)l1);
    if (l2) atomicAdd(a + 2, (unsigned long long)l2);
    if (l3) atomicAdd(a + 3, (unsigned long long)l3);
}

// the reference leaves its fast path (Dekker + fsum) for exact rationals when
// a rounded product or its Dekker error term is non-finite or a product is
// nonzero below 2^-900 (kernel.py:117-121); only `plain`'s start value
// depends on it.  Elements that can trigger it never sit in the private window.
__device__ __noinline__ bool ref_fallback(double x, double y) {
    const double h = __dmul_rn(x, y);
    if (!(fabs(h) <= 1.79769313486231570815e308)) return true;
    if (h != 0.0 && fabs(h) < 0x1p-900) return true;
    const double c = 134217729.0;
    const double px = __dmul_rn(c, x), py = __dmul_rn(c, y);
    const double xh = __dsub_rn(px, __dsub_rn(px, x)), yh = __dsub_rn(py, __dsub_rn(py, y));
    const double xl = __dsub_rn(x, xh), yl = __dsub_rn(y, yh);
    const double e = __dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(xh, yh), h), __dmul_rn(xh, yl)),
                                         __dmul_rn(xl, yh)), __dmul_rn(xl, yl));
    return !(fabs(e) <= 1.79769313486231570815e308);
}

// elements outside the window: zero, non-finite, cold keys, extreme magnitudes
// returns 1 for a non-finite element, 2 when the element sends the reference
// to its Fraction path (see ref_fallback), else 0
__device__ __noinline__ uint32_t x_cold(XShared& S, int64_t* __restrict__ acc, uint64_t bx, uint64_t by) {
    if (((bx >> 52) & 0x7FF) == 0x7FF || ((by >> 52) & 0x7FF) == 0x7FF) return 1u;
    uint64_t mx, my;
    int fx, fy;
    split_dbl(bx, mx, fx);
    split_dbl(by, my, fy);
    if (!mx || !my) return 0u;                              // zero product contributes nothing
    uint32_t r = 0u;
    // |x| or |y| >= 2^995, or the product near overflow / below 2^-899
    if (fx > 2017 || fy > 2017 || fx + fy > 3066 || fx + fy < 1150)
        if (ref_fallback(bitsd(bx), bitsd(by))) r = 2u;
    uint64_t lo, hi;
    prod128(mx, my, (bx ^ by) >> 63, lo, hi);
    const int c = fx + fy - 2 - S.cbase;
    if ((unsigned)c < (unsigned)XCW) {
        const unsigned __int128 P = ((unsigned __int128)hi << 64) | lo;
#pragma unroll
        for (int i = 0; i < 7; ++i) atomicAdd(&S.cold[i][c], (uint32_t)(P >> (14 * i)) & 0x3FFFu);
        atomicAdd(&S.cold[7][c], (uint32_t)(int32_t)((int64_t)hi >> 34));     // signed top: P >> 98
    } else {
        push_limbs(acc, fx + fy - 2, lo, hi);
    }
    return r;
}

// QUEUE: elements outside the private window are only flagged (returned
// true) for the warp queue; otherwise they take x_cold here
template <bool QUEUE>
__device__ __forceinline__ bool x_elem(XShared& S, ulonglong2* __restrict__ my_slots, int base, int64_t* acc,
                                       double xv, double yv, uint32_t& nf, uint32_t& fb) {
    const uint64_t bx = dbits(xv), by = dbits(yv);
    const uint32_t fx = (uint32_t)(bx >> 52) & 0x7FFu, fy = (uint32_t)(by >> 52) & 0x7FFu;
    const int rel = (int)(fx + fy) - 2 - base;
    // window keys lie in [X_SAFE_LO, X_SAFE_HI]; fx, fy in [1, 2017] (normal, below 2^995)
    if (((unsigned)rel < (unsigned)XW) & (max(fx - 1u, fy - 1u) < 2017u)) {
        uint64_t lo, hi;
        prod128((bx & 0xFFFFFFFFFFFFFull) | (1ull << 52), (by & 0xFFFFFFFFFFFFFull) | (1ull << 52),
                (bx ^ by) >> 63, lo, hi);
        ulonglong2* slot = my_slots + rel * XT;
        ulonglong2 v = *slot;
        const uint64_t nl = v.x + lo;
        v.y += hi + (nl < lo ? 1 : 0);
        v.x = nl;
        *slot = v;
        return false;
    }
    if (QUEUE) return true;
    const uint32_t r = x_cold(S, acc, bx, by);
    nf += r & 1u;
    fb += r >> 1;
    return false;
}

// drain the warp's queue, one element per lane (warp-collective)
__device__ __forceinline__ void x_drain(XShared& S, int64_t* acc, int warp, int lane, uint32_t& qn, uint32_t& nf,
                                        uint32_t& fb) {
    __syncwarp();
    if ((uint32_t)lane < qn) {
        const double2 e = S.q[warp][lane];
        const uint32_t r = x_cold(S, acc, dbits(e.x), dbits(e.y));
        nf += r & 1u;
        fb += r >> 1;
    }
    qn = 0;
    __syncwarp();
}

__device__ __forceinline__ void x_enqueue(XShared& S, int64_t* acc, int warp, int lane, uint32_t& qn, bool c,
                                          double xv, double yv, uint32_t& nf, uint32_t& fb) {
    const unsigned m = __ballot_sync(0xffffffffu, c);
    if (m) {
        const uint32_t k = __popc(m);
        if (qn + k > 32) x_drain(S, acc, warp, lane, qn, nf, fb);
        if (c) S.q[warp][qn + __popc(m & ((1u << lane) - 1u))] = make_double2(xv, yv);
        qn += k;
    }
}

struct XTileRegs {
    double x[2 * XV], y[2 * XV];
};

template <bool NORM>
__device__ __forceinline__ void x_load(XTileRegs& T, const double* __restrict__ x, const double* __restrict__ y,
                                       int64_t t, int tid) {
    const double2* x2 = reinterpret_cast<const double2*>(x + t * XTILE);
    const double2* y2 = reinterpret_cast<const double2*>(y + t * XTILE);
#pragma unroll
    for (int v = 0; v < XV; ++v) {
        const double2 a = __ldcs(x2 + v * XT + tid);
        T.x[2 * v] = a.x; T.x[2 * v + 1] = a.y;
        if (!NORM) {
            const double2 b = __ldcs(y2 + v * XT + tid);
            T.y[2 * v] = b.x; T.y[2 * v + 1] = b.y;
        } else {
            T.y[2 * v] = a.x; T.y[2 * v + 1] = a.y;
        }
    }
}

// CTA reduction of the private slots (one warp per key) -> global limbs
__device__ void x_flush(XShared& S, int64_t* __restrict__ acc, int tid) {
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = warp; r < XW; r += XT / 32) {
        uint64_t lo = 0, hi = 0;
        for (int i = lane; i < XT; i += 32) {
            const ulonglong2 v = S.priv[r * XT + i];
            S.priv[r * XT + i] = make_ulonglong2(0ull, 0ull);
            const uint64_t nl = lo + v.x;
            hi += v.y + (nl < lo ? 1 : 0);
            lo = nl;
        }
        for (int o = 16; o; o >>= 1) {
            const uint64_t ol = __shfl_xor_sync(0xffffffffu, lo, o), oh = __shfl_xor_sync(0xffffffffu, hi, o);
            const uint64_t nl = lo + ol;
            hi += oh + (nl < lo ? 1 : 0);
            lo = nl;
        }
        if (lane == 0 && (lo | hi)) push_limbs(acc, S.base + r, lo, hi);
    }
    for (int c = tid; c < XCW; c += XT) {
        unsigned __int128 v = 0;
        bool any = false;
#pragma unroll
        for (int i = 0; i < 7; ++i) {
            const uint32_t l = S.cold[i][c];
            any |= l != 0;
            v += (unsigned __int128)l << (14 * i);
            S.cold[i][c] = 0u;
        }
        const int32_t top = (int32_t)S.cold[7][c];
        any |= top != 0;
        S.cold[7][c] = 0u;
        v += (unsigned __int128)((__int128)top * ((__int128)1 << 98));
        if (any) push_limbs(acc, S.cbase + c, (uint64_t)v, (uint64_t)(v >> 64));
    }
    __syncthreads();
}

template <bool NORM, int PFD, bool QUEUE>
__device__ __forceinline__ void x_stream(XShared& S, const double* __restrict__ x, const double* __restrict__ y,
                                         int64_t n, int64_t* __restrict__ acc, bool vec, int base, int tid,
                                         uint32_t& nf, uint32_t& fb) {
    ulonglong2* __restrict__ my_slots = S.priv + tid;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t ntiles = (n + XTILE - 1) / XTILE;
    uint32_t qn = 0;                                    // warp queue fill (warp-uniform)
    int since = 0;
    const int64_t G = gridDim.x;
    // full tiles: 128-bit loads of one tile, a bulk L2 prefetch PFD grid-strides ahead
    const int64_t nfull = vec ? n / XTILE : 0;
    XTileRegs ta;
    int64_t t = blockIdx.x;
    if (t < nfull) x_load<NORM>(ta, x, y, t, tid);
    while (t < nfull) {
        if (t != (int64_t)blockIdx.x) x_load<NORM>(ta, x, y, t, tid);
        if (PFD > 0 && tid == 0 && t + PFD * G < nfull) {
            const int64_t p0 = (t + PFD * G) * XTILE;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(qd::bulk_aligned(x + p0)), "r"(XTILE * 8) : "memory");
            if (!NORM) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(qd::bulk_aligned(y + p0)), "r"(XTILE * 8) : "memory");
        }
#pragma unroll
        for (int j = 0; j < 2 * XV; ++j) {
            const bool c = x_elem<QUEUE>(S, my_slots, base, acc, ta.x[j], ta.y[j], nf, fb);
            if (QUEUE) x_enqueue(S, acc, warp, lane, qn, c, ta.x[j], ta.y[j], nf, fb);
        }
        if (++since == XFLUSH) {
            if (QUEUE) x_drain(S, acc, warp, lane, qn, nf, fb);
            x_flush(S, acc, tid);
            since = 0;
        }
        t += G;
    }
    // the partial last tile (and every tile of unaligned inputs): direct cold path
    for (int64_t t2 = blockIdx.x; t2 < ntiles; t2 += G) {
        if (t2 < nfull) continue;
        const int64_t e0 = t2 * XTILE;
        for (int j = 0; j < 2 * XV; ++j) {
            const int64_t i = e0 + 2 * ((int64_t)(j >> 1) * XT + tid) + (j & 1);
            if (i < n) {
                const double a = x[i];
                x_elem<false>(S, my_slots, base, acc, a, NORM ? a : y[i], nf, fb);
            }
        }
        if (++since == XFLUSH) { x_flush(S, acc, tid); since = 0; }
    }
    if (QUEUE) x_drain(S, acc, warp, lane, qn, nf, fb);
    x_flush(S, acc, tid);
}

template <bool NORM, int PFD>
__global__ void __launch_bounds__(XT, 3) k_exact(const double* __restrict__ x, const double* __restrict__ y,
                                                 int64_t n, int64_t* __restrict__ acc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    XShared& S = *reinterpret_cast<XShared*>(smem_raw);
    const int tid = threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15u) == 0;

    // ---- window: densest 16 consecutive keys of this CTA's first tile
    uint32_t* hist = reinterpret_cast<uint32_t*>(S.priv);              // XKEYS u32 (reuses the slots)
    for (int k = tid; k < XKEYS; k += XT) hist[k] = 0u;
    __syncthreads();
    uint32_t nsample = 0;                                            // block-uniform
    for (int j = 0; j < 2 * XV; ++j) {
        const int64_t i = (int64_t)blockIdx.x * XTILE + (int64_t)j * XT + tid;
        bool valid = false;
        if (i < n) {
            const double a = x[i], b = NORM ? a : y[i];
            const uint32_t fx = (uint32_t)(dbits(a) >> 52) & 0x7FFu, fy = (uint32_t)(dbits(b) >> 52) & 0x7FFu;
            valid = fx - 1u < 0x7FEu && fy - 1u < 0x7FEu;
            if (valid) atomicAdd(&hist[fx + fy - 2], 1u);
        }
        nsample += __syncthreads_count(valid);
    }
    __syncthreads();
    {
        unsigned long long best = 0ull;
        for (int b = X_SAFE_LO + tid; b <= X_SAFE_HI; b += XT) {
            uint32_t s = 0;
            for (int r = 0; r < XW; ++r) s += hist[b + r];
            const unsigned long long cand = ((unsigned long long)s << 32) | (uint32_t)(0xFFFFFFFFu - b);
            best = cand > best ? cand : best;
        }
        for (int o = 16; o; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
            best = t > best ? t : best;
        }
        __shared__ unsigned long long red[XT / 32];
        if ((tid & 31) == 0) red[tid >> 5] = best;
        __syncthreads();
        if (tid == 0) {
            unsigned long long m = 0ull;
            for (int w = 0; w < XT / 32; ++w) m = red[w] > m ? red[w] : m;
            S.base = (m >> 32) ? (int)(0xFFFFFFFFu - (uint32_t)m) : 2046;
            // queue mode when more than 1/128 of the sample lies outside the private window
            const uint32_t cov = (uint32_t)(m >> 32);
            S.queue = (nsample - cov) * 128u > nsample;
            int cb = S.base - (XCW - XW) / 2;
            S.cbase = cb < 0 ? 0 : (cb + XCW > XKEYS ? XKEYS - XCW : cb);
        }
    }
    __syncthreads();
    for (int k = tid; k < XW * XT; k += XT) S.priv[k] = make_ulonglong2(0ull, 0ull);
    for (int k = tid; k < 8 * XCW; k += XT) (&S.cold[0][0])[k] = 0u;
    __syncthreads();
    const int base = S.base;

    // ---- stream
    uint32_t nf = 0, fb = 0;
    if (S.queue) x_stream<NORM, PFD, true>(S, x, y, n, acc, vec, base, tid, nf, fb);
    else x_stream<NORM, PFD, false>(S, x, y, n, acc, vec, base, tid, nf, fb);
    unsigned long long a = nf, b = fb;
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((tid & 31) == 0) {
        if (a) atomicAdd(reinterpret_cast<unsigned long long*>(acc + X_NONFINITE), a);
        if (b) atomicAdd(reinterpret_cast<unsigned long long*>(acc + X_FALLBACK), b);
    }
}

// ReferenceResult.plain: left-to-right double sum of fl(x_i*y_i), chained
// across calls.  The reference's fast path starts at h[0]
// (np.add.accumulate); its Fraction path starts at 0.0 (kernel.py:127-129).
template <bool NORM>
__global__ void k_exact_plain(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                              int64_t* __restrict__ ws) {
    if (threadIdx.x != 0 || blockIdx.x != 0 || n <= 0) return;
    const bool fallback = ws[X_FALLBACK] != 0;
    double s = bitsd((uint64_t)ws[X_PLAIN]);
    int64_t i = 0;
    if (!ws[X_PLAIN_STARTED]) {
        const double h0 = __dmul_rn(x[0], NORM ? x[0] : y[0]);
        s = fallback ? __dadd_rn(0.0, h0) : h0;
        i = 1;
    }
    for (; i < n; ++i) {
        const double a = x[i];
        s = __dadd_rn(s, __dmul_rn(a, NORM ? a : y[i]));
    }
    ws[X_PLAIN] = (int64_t)dbits(s);
    ws[X_PLAIN_STARTED] = 1;
}

__global__ void __launch_bounds__(32, 1) k_exact_finalize(int64_t* __restrict__ ws) {
    // one thread folds the per-key limbs into one big integer (value =
    // sum_k sum_i limb[k][i] 2^(32 i) 2^(k - 2148)) and rounds it once
    if (threadIdx.x != 0) return;
    qdot_exact_result r;
    memset(&r, 0, sizeof(r));
    r.plain = bitsd((uint64_t)ws[X_PLAIN]);
    r.nonfinite = ws[X_NONFINITE];
    r.fallback = ws[X_FALLBACK] != 0;
    if (r.nonfinite) {
        r.status = QDOT_ERR_NONFINITE;
    } else {
        BigSum<140> big;
        big.init(-2148, 140);
        for (int k = 0; k < XKEYS; ++k) {
            const int64_t* l = ws + X_ACC + 4 * k;
            if (!(l[0] | l[1] | l[2] | l[3])) continue;
            for (int i = 0; i < 4; ++i)
                if (l[i]) big.add((__int128)l[i], k - 2148 + 32 * i);
        }
        int ovf = 0;
        r.value = big.round(52, -1022, 1023, &ovf);
        r.status = ovf ? QDOT_ERR_OVERFLOW : QDOT_OK;
        r.is_zero = r.value == 0.0;
        r.flexp_e = r.is_zero ? 0 : flexp_bits(dbits(r.value));
    }
    *reinterpret_cast<qdot_exact_result*>(ws + X_RESULT) = r;
}

static_assert(sizeof(qdot_exact_result) <= 16 * 8, "exact result block");

int sm_count() { return qd::device_sm_count(); }

template <bool NORM, int PFD>
cudaError_t launch_exact_t(const double* x, const double* y, int64_t n, int64_t* ws, cudaStream_t st) {
    auto kern = k_exact<NORM, PFD>;
    static qd::KernelDevCache cache;
    const int occ = qd::kernel_occupancy(kern, XT, sizeof(XShared), cache);
    const int64_t ntiles = (n + XTILE - 1) / XTILE;
    int64_t grid = (int64_t)sm_count() * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, XT, sizeof(XShared), st>>>(x, y, n, ws);
    return cudaGetLastError();
}

template <bool NORM>
cudaError_t launch_exact(const double* x, const double* y, int64_t n, int64_t* ws, cudaStream_t st) {
    return launch_exact_t<NORM, 3>(x, y, n, ws, st);   // bulk L2 prefetch 3 grid-strides ahead
}

int fail(cudaError_t e, const char* where) { return qd::report_cuda_error(e, where); }

}  // namespace

extern "C" {

size_t qdot_b200_exact_workspace_bytes(void) { return (size_t)X_WORDS * 8; }

int64_t qdot_b200_exact_region_words(void) { return X_REGION; }

int qdot_b200_exact_begin(void* xws, void* stream) {
    if (!xws) return QDOT_ERR_ARG;
    cudaError_t e = cudaMemsetAsync(xws, 0, (size_t)X_WORDS * 8, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? QDOT_OK : fail(e, "exact_begin");
}

int qdot_b200_exact_accumulate(const double* x, const double* y, int64_t n, int norm, void* xws, void* stream) {
    if (!xws || n < 0 || (n > 0 && (!x || (!norm && !y)))) return QDOT_ERR_ARG;
    if (n == 0) return QDOT_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t* ws = static_cast<int64_t*>(xws);
    cudaError_t e = norm ? launch_exact<true>(x, x, n, ws, st) : launch_exact<false>(x, y, n, ws, st);
    return e == cudaSuccess ? QDOT_OK : fail(e, "exact_accumulate");
}

int qdot_b200_exact_plain(const double* x, const double* y, int64_t n, int norm, void* xws, void* stream) {
    if (!xws || n < 0 || (n > 0 && (!x || (!norm && !y)))) return QDOT_ERR_ARG;
    if (n == 0) return QDOT_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t* ws = static_cast<int64_t*>(xws);
    if (norm) k_exact_plain<true><<<1, 32, 0, st>>>(x, x, n, ws);
    else k_exact_plain<false><<<1, 32, 0, st>>>(x, y, n, ws);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : fail(e, "exact_plain");
}

int qdot_b200_exact_finalize(void* xws, void* stream) {
    if (!xws) return QDOT_ERR_ARG;
    k_exact_finalize<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<int64_t*>(xws));
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : fail(e, "exact_finalize");
}

int qdot_b200_exact_fetch(const void* xws, qdot_exact_result* out, void* stream) {
    if (!xws || !out) return QDOT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(out, static_cast<const int64_t*>(xws) + X_RESULT, sizeof(qdot_exact_result),
                                    cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? QDOT_OK : fail(e, "exact_fetch");
}

}  // extern "C"
