// qdot_kernels.cu -- sm_100a kernels of the qdot hot path.
//
//   pass1     streaming pass over x, y (16 B/elem, 8 B/elem in norm mode):
//             exponent extraction, exact exponent-sum histogram, exact per-key
//             DOUBLE partials and exact-binning HALF/SINGLE partials
//             (replaces floatbits.py:57-93, binning.py:88-116 and, for every
//             bin whose products do not depend on the partition, the
//             emulate.py:116-154 bin_dot work).
//   score     one CTA: partition + bin scores + precisions + LUT from the
//             histogram alone (kernel.py:59-72, binning.py:191-284,
//             scoring.py:96-216).
//   pass2     second streaming pass, only when a HALF/SINGLE bin has upper
//             u != e for some member key (ranged / split / early bins).
//   finalize  one CTA: per-bin exact sums rounded like the reference, and the
//             ascending-upper Neumaier fold (emulate.py:154-163).
//   bin_ids   lazy Bin.indices support (binning.py:174).
//
// No tensor cores: this is a memory-bound integer/bit reduction.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "qdot_common.cuh"
#include "qdot_kernels.h"

namespace qd {

// =============================================================================
// pass 1
// =============================================================================
constexpr int P1_T = 256;                    // threads per CTA
constexpr int P1_W = 16;                     // keys with per-thread private slots
constexpr int P1_CW = 192;                   // keys with per-CTA smem-atomic slots
constexpr int P1_V = 4;                      // 16-byte vectors per thread per tile per operand
constexpr int P1_EPT = 2 * P1_V;             // elements per thread per tile
constexpr int P1_TILE = P1_T * P1_EPT;       // elements per tile
constexpr int P1_FLUSH = 255 / P1_EPT;       // tiles between flushes (<= 255 elements/thread)

struct __align__(16) P1Shared {
    ulonglong2 priv[P1_W * P1_T];            // .x = DOUBLE units (int64), .y = packed S|H|count
    __int128 t_d[P1_W];                      // CTA totals of the private window
    long long t_s[P1_W], t_h[P1_W], t_c[P1_W];
    unsigned long long c_cnt[P1_CW];         // cold window (smem atomics)
    unsigned long long c_dlo[P1_CW];
    unsigned long long c_dhi[P1_CW];
    unsigned long long c_s[P1_CW];
    unsigned long long c_h[P1_CW];
    unsigned long long red[2 * (P1_T / 32)];
    int base;                                // first key of the private window
    int cbase;                               // first key of the cold window
    int pick[2];
};

size_t pass1_smem_bytes() { return sizeof(P1Shared); }

// push one key's exact partials to the global tables (region A / B)
__device__ __forceinline__ void push_key(int64_t* __restrict__ A, int64_t* __restrict__ B, int key,
                                         unsigned long long cnt, __int128 d, long long s, long long h) {
    atomicAdd(reinterpret_cast<unsigned long long*>(A + A_CNT + key), cnt);
    unsigned long long l0 = (unsigned long long)(uint32_t)(uint64_t)d;
    unsigned long long l1 = (unsigned long long)(uint32_t)(uint64_t)(d >> 32);
    unsigned long long l2 = (unsigned long long)(uint32_t)(uint64_t)(d >> 64);
    unsigned long long l3 = (unsigned long long)(long long)(d >> 96);
    if (l0) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_D0 + key), l0);
    if (l1) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_D1 + key), l1);
    if (l2) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_D2 + key), l2);
    if (l3) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_D3 + key), l3);
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_S0 + key), (unsigned long long)s);
    if (h) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_H0 + key), (unsigned long long)h);
}

// exact-binning HALF/SINGLE units of the scaled mantissas mx, my in [1,2)
// (emulate.py:137-146 with u == e: sx = x 2^-ex, sy = y 2^-ey)
__device__ __forceinline__ void exact_variants(double mx, double my, int32_t& ks, int32_t& kh) {
    float rx = __double2float_rn(mx), ry = __double2float_rn(my);
    uint32_t sb = __float_as_uint(__fmul_rn(rx, ry));                    // in [1, 4]
    ks = (int32_t)(((sb & 0x7FFFFFu) | 0x800000u) << ((sb >> 23) - 127)); // units of 2^-23
    __half hx = __double2half(mx), hy = __double2half(my);
    uint32_t hb = __half_as_ushort(__hmul(hx, hy));                       // in [1, 4]
    kh = (int32_t)(((hb & 0x3FFu) | 0x400u) << ((hb >> 10) - 15));        // units of 2^-10
}

__device__ __forceinline__ void cold_add(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B,
                                         int key, int64_t kd, int32_t ks, int32_t kh) {
    int c = key - S.cbase;
    if ((unsigned)c < (unsigned)P1_CW) {
        atomicAdd(&S.c_cnt[c], 1ull);
        atomicAdd(&S.c_dlo[c], (unsigned long long)(uint32_t)(uint64_t)kd);
        atomicAdd(&S.c_dhi[c], (unsigned long long)(kd >> 32));
        atomicAdd(&S.c_s[c], (unsigned long long)(long long)ks);
        atomicAdd(&S.c_h[c], (unsigned long long)(long long)kh);
    } else {
        push_key(A, B, key, 1ull, (__int128)kd, ks, kh);
    }
}

// zero / subnormal / non-finite / extreme-exponent elements
__device__ __noinline__ void p1_slow(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B,
                                     double xv, double yv, uint32_t& zc, uint32_t& nf) {
    uint64_t bx = dbits(xv), by = dbits(yv);
    if (((bx >> 52) & 0x7FF) == 0x7FF || ((by >> 52) & 0x7FF) == 0x7FF) { nf++; return; }
    if (xv == 0.0 || yv == 0.0) { zc++; return; }                      // floatbits.py:74
    int e = flexp_bits(bx) + flexp_bits(by);
    int key = e + KOFF;
    double p = __dmul_rn(xv, yv);
    uint64_t pb = dbits(p);
    int64_t kd = 0;
    if (((pb >> 52) & 0x7FF) == 0x7FF) {                               // DOUBLE product overflow
        atomicAdd(reinterpret_cast<unsigned long long*>(B + ((pb >> 63) ? B_INFN : B_INFP) + key), 1ull);
    } else {
        kd = double_units(pb, e);
    }
    int32_t ks, kh;
    exact_variants(bitsd(mant_bits(bx)), bitsd(mant_bits(by)), ks, kh);
    int32_t sg = (int32_t)((bx ^ by) >> 63);
    sg = -sg;
    ks = (ks ^ sg) - sg;
    kh = (kh ^ sg) - sg;
    cold_add(S, A, B, key, kd, ks, kh);
}

__device__ __forceinline__ void p1_element(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B,
                                           double xv, double yv, int tid, uint32_t& zc, uint32_t& nf) {
    uint64_t bx = dbits(xv), by = dbits(yv);
    uint32_t fx = (uint32_t)(bx >> 52) & 0x7FFu, fy = (uint32_t)(by >> 52) & 0x7FFu;
    int e = (int)(fx + fy) - 2046;
    bool fast = (fx - 1u < 0x7FEu) & (fy - 1u < 0x7FEu) & ((unsigned)(e + 1022) <= 2043u);
    if (fast) {
        // DOUBLE: fl(x*y) in units of 2^(e-52)  (emulate.py:133)
        uint64_t pb = dbits(__dmul_rn(xv, yv));
        uint64_t pm = (pb & 0xFFFFFFFFFFFFFull) | (1ull << 52);
        int sh = (int)((pb >> 52) & 0x7FF) - 1023 - e;                   // 0..2
        int64_t kd = (int64_t)(pm << sh);
        int64_t sg = (int64_t)(bx ^ by) >> 63;                            // 0 / -1
        kd = (kd ^ sg) - sg;
        int32_t ks, kh;
        exact_variants(bitsd((bx & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull),
                       bitsd((by & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull), ks, kh);
        int32_t sg32 = (int32_t)sg;
        ks = (ks ^ sg32) - sg32;
        kh = (kh ^ sg32) - sg32;
        int key = e + KOFF;
        int rel = key - S.base;
        if ((unsigned)rel < (unsigned)P1_W) {
            long long inc = ((long long)ks << 29) + ((long long)kh << 8) + 1;
            ulonglong2* slot = &S.priv[rel * P1_T + tid];
            ulonglong2 v = *slot;
            v.x += (unsigned long long)kd;
            v.y += (unsigned long long)inc;
            *slot = v;
        } else {
            cold_add(S, A, B, key, kd, ks, kh);
        }
    } else {
        p1_slow(S, A, B, xv, yv, zc, nf);
    }
}

// reduce the private slots into the CTA totals and clear them (all threads)
__device__ __forceinline__ void p1_flush(P1Shared& S, int tid) {
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = warp; r < P1_W; r += P1_T / 32) {
        uint64_t dlo = 0;
        int64_t dhi = 0;
        long long ss = 0, hs = 0, cs = 0;
        for (int i = lane; i < P1_T; i += 32) {
            ulonglong2 v = S.priv[r * P1_T + i];
            S.priv[r * P1_T + i] = make_ulonglong2(0ull, 0ull);
            int64_t d = (int64_t)v.x;
            uint64_t nl = dlo + (uint64_t)d;
            dhi += (d >> 63) + (nl < dlo ? 1 : 0);
            dlo = nl;
            long long w = (long long)v.y;
            long long c = w & 0xFF;
            long long w1 = (w - c) >> 8;
            long long h = ((w1 & 0x1FFFFF) ^ 0x100000) - 0x100000;
            long long s = (w1 - h) >> 21;
            cs += c; hs += h; ss += s;
        }
        for (int o = 16; o; o >>= 1) {
            uint64_t olo = __shfl_xor_sync(0xffffffffu, dlo, o);
            int64_t ohi = __shfl_xor_sync(0xffffffffu, dhi, o);
            uint64_t nl = dlo + olo;
            dhi += ohi + (nl < dlo ? 1 : 0);
            dlo = nl;
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
            hs += __shfl_xor_sync(0xffffffffu, hs, o);
            cs += __shfl_xor_sync(0xffffffffu, cs, o);
        }
        if (lane == 0) {
            S.t_d[r] += ((__int128)dhi << 64) | (__int128)dlo;
            S.t_s[r] += ss;
            S.t_h[r] += hs;
            S.t_c[r] += cs;
        }
    }
    __syncthreads();
}

template <bool NORM, bool VEC>
__device__ __forceinline__ void p1_load(const double* __restrict__ x, const double* __restrict__ y,
                                        int64_t n, int64_t tile, int tid, double (&xv)[P1_EPT],
                                        double (&yv)[P1_EPT], bool& full) {
    const int64_t e0 = tile * P1_TILE;
    full = e0 + P1_TILE <= n;
    if (VEC && full) {
        const double2* x2 = reinterpret_cast<const double2*>(x + e0);
        const double2* y2 = reinterpret_cast<const double2*>(y + e0);
#pragma unroll
        for (int v = 0; v < P1_V; ++v) {
            double2 a = __ldcs(x2 + v * P1_T + tid);
            xv[2 * v] = a.x; xv[2 * v + 1] = a.y;
            if (!NORM) {
                double2 b = __ldcs(y2 + v * P1_T + tid);
                yv[2 * v] = b.x; yv[2 * v + 1] = b.y;
            }
        }
    } else {
#pragma unroll
        for (int v = 0; v < P1_V; ++v) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                int64_t i = e0 + 2 * ((int64_t)v * P1_T + tid) + k;
                bool ok = i < n;
                xv[2 * v + k] = ok ? __ldcs(x + i) : 0.0;
                if (!NORM) yv[2 * v + k] = ok ? __ldcs(y + i) : 0.0;
            }
        }
    }
    if (NORM) {
#pragma unroll
        for (int j = 0; j < P1_EPT; ++j) yv[j] = xv[j];
    }
}

template <bool NORM, bool VEC>
__global__ void __launch_bounds__(P1_T, 3)
k_pass1(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
        int64_t* __restrict__ A, int64_t* __restrict__ B) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    P1Shared& S = *reinterpret_cast<P1Shared*>(smem_raw);
    const int tid = threadIdx.x;
    const int64_t ntiles = (n + P1_TILE - 1) / P1_TILE;

    // ---- choose the private window from this CTA's first tile: the P1_W
    // consecutive keys holding most sampled elements (sliding-window argmax).
    uint32_t* hist = reinterpret_cast<uint32_t*>(S.priv);           // KEYS u32 (reuses priv)
    uint32_t* pref = hist + 4224;                                   // KEYS+1 u32
    for (int k = tid; k < 4224 * 2; k += P1_T) hist[k] = 0u;
    __syncthreads();
    if ((int64_t)blockIdx.x < ntiles) {
        double xv[P1_EPT], yv[P1_EPT];
        bool full;
        p1_load<NORM, VEC>(x, y, n, blockIdx.x, tid, xv, yv, full);
        const int64_t e0 = (int64_t)blockIdx.x * P1_TILE;
#pragma unroll
        for (int j = 0; j < P1_EPT; ++j) {
            int64_t i = e0 + 2 * ((int64_t)(j >> 1) * P1_T + tid) + (j & 1);
            if (i >= n) continue;
            uint64_t bx = dbits(xv[j]), by = dbits(yv[j]);
            uint32_t fx = (uint32_t)(bx >> 52) & 0x7FFu, fy = (uint32_t)(by >> 52) & 0x7FFu;
            if (fx - 1u < 0x7FEu && fy - 1u < 0x7FEu) atomicAdd(&hist[(int)(fx + fy) - 2046 + KOFF], 1u);
        }
    }
    __syncthreads();
    {   // inclusive prefix over KEYS (17 keys per thread)
        constexpr int PER = (KEYS + P1_T - 1) / P1_T;
        uint32_t loc[PER];
        uint32_t run = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            int k = tid * PER + i;
            run += k < KEYS ? hist[k] : 0u;
            loc[i] = run;
        }
        // block exclusive scan of per-thread totals
        const int lane = tid & 31, warp = tid >> 5;
        uint32_t incl = run;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) S.red[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += (uint32_t)S.red[w];
        uint32_t pre = wpre + incl - run;
        pref[0] = 0u;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            int k = tid * PER + i;
            if (k < KEYS) pref[k + 1] = pre + loc[i];
        }
    }
    __syncthreads();
    {   // argmax over window starts b: sum = pref[b+W] - pref[b]
        unsigned long long best = 0ull;
        for (int b = tid; b + P1_W <= KEYS; b += P1_T) {
            uint32_t s = pref[b + P1_W] - pref[b];
            unsigned long long cand = ((unsigned long long)s << 32) | (uint32_t)(0xFFFFFFFFu - b);
            best = cand > best ? cand : best;
        }
        for (int o = 16; o; o >>= 1) {
            unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
            best = t > best ? t : best;
        }
        __syncthreads();
        if ((tid & 31) == 0) S.red[tid >> 5] = best;
        __syncthreads();
        if (tid == 0) {
            unsigned long long m = 0ull;
            for (int w = 0; w < P1_T / 32; ++w) m = S.red[w] > m ? S.red[w] : m;
            int b = (m >> 32) ? (int)(0xFFFFFFFFu - (uint32_t)m) : (KOFF - 8);   // default near e = 0
            S.base = b;
            int cb = b - (P1_CW - P1_W) / 2;
            cb = cb < 0 ? 0 : cb;
            cb = cb + P1_CW > KEYS ? KEYS - P1_CW : cb;
            S.cbase = cb;
        }
    }
    __syncthreads();
    // ---- clear private slots, cold table and totals
    for (int k = tid; k < P1_W * P1_T; k += P1_T) S.priv[k] = make_ulonglong2(0ull, 0ull);
    for (int k = tid; k < P1_CW; k += P1_T) {
        S.c_cnt[k] = 0ull; S.c_dlo[k] = 0ull; S.c_dhi[k] = 0ull; S.c_s[k] = 0ull; S.c_h[k] = 0ull;
    }
    if (tid < P1_W) { S.t_d[tid] = 0; S.t_s[tid] = 0; S.t_h[tid] = 0; S.t_c[tid] = 0; }
    __syncthreads();

    // ---- main streaming loop (persistent grid over tiles)
    uint32_t zc = 0, nf = 0;
    int since = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        double xv[P1_EPT], yv[P1_EPT];
        bool full;
        p1_load<NORM, VEC>(x, y, n, t, tid, xv, yv, full);
        if (full) {
#pragma unroll
            for (int j = 0; j < P1_EPT; ++j) p1_element(S, A, B, xv[j], yv[j], tid, zc, nf);
        } else {
            const int64_t e0 = t * P1_TILE;
#pragma unroll
            for (int j = 0; j < P1_EPT; ++j) {
                int64_t i = e0 + 2 * ((int64_t)(j >> 1) * P1_T + tid) + (j & 1);
                if (i < n) p1_element(S, A, B, xv[j], yv[j], tid, zc, nf);
            }
        }
        if (++since == P1_FLUSH) { p1_flush(S, tid); since = 0; }
    }
    p1_flush(S, tid);

    // ---- publish CTA partials
    for (int r = tid; r < P1_W; r += P1_T)
        if (S.t_c[r]) push_key(A, B, S.base + r, (unsigned long long)S.t_c[r], S.t_d[r], S.t_s[r], S.t_h[r]);
    for (int c = tid; c < P1_CW; c += P1_T) {
        if (S.c_cnt[c]) {
            __int128 d = ((__int128)(long long)S.c_dhi[c] << 32) + (__int128)S.c_dlo[c];
            push_key(A, B, S.cbase + c, S.c_cnt[c], d, (long long)S.c_s[c], (long long)S.c_h[c]);
        }
    }
    // zero / non-finite counts
    unsigned long long z = zc, f = nf;
    for (int o = 16; o; o >>= 1) {
        z += __shfl_xor_sync(0xffffffffu, z, o);
        f += __shfl_xor_sync(0xffffffffu, f, o);
    }
    if ((tid & 31) == 0) {
        if (z) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_ZERO), z);
        if (f) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_NONFINITE), f);
    }
}

// =============================================================================
// score (one CTA)
// =============================================================================
constexpr int SC_T = 1024;
constexpr int SC_PER = (KEYS + SC_T - 1) / SC_T;   // 5 keys per thread

struct ScShared {
    unsigned long long off[KEYS + 1];   // exclusive prefix of counts over keys
    int first[KEYS];
    int last[KEYS];
    int bin_of[KEYS];
    unsigned long long red[SC_T / 32];
    long long red2[SC_T / 32];
    int s_status, s_deg, s_early, s_nb, s_need;
    int kmin, kmax;
    long long nnz;
    double eps_eff;
    long long fl;
};

size_t score_smem_bytes() { return sizeof(ScShared); }

template <typename T, typename Op>
__device__ T block_reduce(T v, T* red, Op op, T ident) {
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    T r = ident;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = op(r, red[w]);
    return r;
}

// exclusive scan of the block's items (thread-major order); returns block total
template <typename T>
__device__ T block_excl_scan(T (&it)[SC_PER], T* red) {
    T run = 0;
#pragma unroll
    for (int i = 0; i < SC_PER; ++i) { T v = it[i]; it[i] = run; run += v; }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl = run;
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    T pre = 0, tot = 0;
    for (int w = 0; w < SC_T / 32; ++w) { if (w < warp) pre += red[w]; tot += red[w]; }
    pre += incl - run;
#pragma unroll
    for (int i = 0; i < SC_PER; ++i) it[i] += pre;
    return tot;
}

// does a slice boundary of `levels` recursive halvings of [0, nz) fall in (a, b]?
// (binning.py:237-264)
__device__ bool split_boundary_in(unsigned long long nz, int levels, unsigned long long a,
                                  unsigned long long b) {
    unsigned long long slo[140], shi[140];
    int slev[140];
    int sp = 0;
    slo[0] = 0; shi[0] = nz; slev[0] = levels; sp = 1;
    while (sp) {
        --sp;
        unsigned long long lo = slo[sp], hi = shi[sp];
        int lev = slev[sp];
        unsigned long long m = hi - lo;
        if (m <= 1 || lev == 0) continue;
        unsigned long long mid = lo + m / 2;
        if (a < mid && mid <= b) return true;
        // left child boundaries lie in [lo+1, mid-1], right child in [mid+1, hi-1]
        if (mid >= lo + 2 && a < mid - 1 && b >= lo + 1 && sp < 139) {
            slo[sp] = lo; shi[sp] = mid; slev[sp] = lev - 1; ++sp;
        }
        if (hi >= mid + 2 && a < hi - 1 && b >= mid + 1 && sp < 139) {
            slo[sp] = mid; shi[sp] = hi; slev[sp] = lev - 1; ++sp;
        }
    }
    return false;
}

__device__ __forceinline__ int precision_of(long long score, int input_mu) {   // scoring.py:108-123
    if (score < 0) return QDOT_PERFORATE;
    const int mus[3] = {10, 23, 52};
    for (int l = 0; l < 3; ++l) {
        if (mus[l] > input_mu) break;
        if (score < mus[l]) return QDOT_HALF + l;
    }
    return input_mu == 10 ? QDOT_HALF : (input_mu == 23 ? QDOT_SINGLE : QDOT_DOUBLE);
}

__device__ __forceinline__ long long floor_log2_d(double v, bool* ok) {    // scoring.py:82-86
    if (!(v > 0.0) || !(v - v == 0.0)) { *ok = false; return 0; }
    *ok = true;
    return flexp_bits(dbits(v));
}

__global__ void __launch_bounds__(SC_T, 1)
k_score(const int64_t* __restrict__ A, int32_t* __restrict__ lut_bin, uint32_t* __restrict__ lut_p2,
        ScoreMeta* __restrict__ meta, qdot_result* __restrict__ res, qdot_bin* __restrict__ bins,
        int64_t n_total, qdot_config cfg) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScShared& S = *reinterpret_cast<ScShared*>(smem_raw);
    const int tid = threadIdx.x;

    unsigned long long cnt[SC_PER];
    int kmin = KEYS, kmax = -1;
    unsigned long long tot = 0;
#pragma unroll
    for (int i = 0; i < SC_PER; ++i) {
        int k = tid * SC_PER + i;
        cnt[i] = k < KEYS ? (unsigned long long)A[A_CNT + k] : 0ull;
        if (cnt[i]) { kmin = min(kmin, k); kmax = max(kmax, k); }
        tot += cnt[i];
    }
    kmin = block_reduce<int>(kmin, reinterpret_cast<int*>(S.red2), [](int a, int b) { return a < b ? a : b; }, KEYS);
    kmax = block_reduce<int>(kmax, reinterpret_cast<int*>(S.red2), [](int a, int b) { return a > b ? a : b; }, -1);
    // exclusive prefix of counts -> off[]
    unsigned long long ex[SC_PER];
#pragma unroll
    for (int i = 0; i < SC_PER; ++i) ex[i] = cnt[i];
    unsigned long long nnz = block_excl_scan<unsigned long long>(ex, S.red);
#pragma unroll
    for (int i = 0; i < SC_PER; ++i) {
        int k = tid * SC_PER + i;
        if (k < KEYS) S.off[k] = ex[i];
    }
    if (tid == 0) S.off[KEYS] = nnz;
    for (int k = tid; k < KEYS; k += SC_T) { S.first[k] = KEYS; S.last[k] = -1; S.bin_of[k] = -1; }

    if (tid == 0) {
        int status = QDOT_OK;
        if (A[A_NONFINITE]) status = QDOT_ERR_NONFINITE;                          // floatbits.py:70
        int deg = nnz == 0;
        int early = 0;
        bool ok = true;
        long long fle = floor_log2_d(cfg.epsilon, &ok);
        if (!ok) status = status ? status : QDOT_ERR_EPS;
        if (!deg && ok) {                                                         // scoring.py:126-136
            int mu_hat = cfg.input_mu == 52 ? 23 : (cfg.input_mu == 23 ? 10 : 0);
            early = (long long)(kmax - kmin) <= (-fle - mu_hat);
        }
        S.s_status = status; S.s_deg = deg; S.s_early = early;
        S.kmin = kmin; S.kmax = kmax; S.nnz = (long long)nnz;
    }
    __syncthreads();
    const int deg = S.s_deg, early = S.s_early;
    const int strategy = cfg.strategy;

    // ---- partition: F flags -> bin ids (binning.py:191-274, kernel.py:60-66)
    int bid[SC_PER];
    if (!deg) {
        int F[SC_PER];
        if (early) {
#pragma unroll
            for (int i = 0; i < SC_PER; ++i) F[i] = 0;
        } else if (strategy == QDOT_STRATEGY_EXACT) {
#pragma unroll
            for (int i = 0; i < SC_PER; ++i) F[i] = cnt[i] ? 1 : 0;                 // one bin per key
        } else if (strategy == QDOT_STRATEGY_SPLIT) {
            // levels clamp: binning.py:235
            long long levels = cfg.strategy_param;
            unsigned long long t = nnz > 1 ? nnz - 1 : 0;
            int bl = t ? 64 - __clzll((long long)t) : 0;
            if (levels > bl) levels = bl;
#pragma unroll
            for (int i = 0; i < SC_PER; ++i) {
                int k = tid * SC_PER + i;
                F[i] = 0;
                if (k < KEYS && cnt[i]) {
                    unsigned long long a = S.off[k], b = S.off[k] + cnt[i];
                    F[i] = (b < nnz && split_boundary_in(nnz, (int)levels, a, b)) ? 1 : 0;   // cut after key
                }
            }
        } else {   // ranged: a bin starts at the first present key of each width-w group
            // present-key exclusive count pc[], then start iff pc[k] == pc[group start]
            int pc[SC_PER];
#pragma unroll
            for (int i = 0; i < SC_PER; ++i) pc[i] = cnt[i] ? 1 : 0;
            block_excl_scan<int>(pc, reinterpret_cast<int*>(S.red2));
#pragma unroll
            for (int i = 0; i < SC_PER; ++i) {
                int k = tid * SC_PER + i;
                if (k < KEYS) S.first[k] = pc[i];                                   // temp: pc
            }
            __syncthreads();
            const long long w = cfg.strategy_param;
#pragma unroll
            for (int i = 0; i < SC_PER; ++i) {
                int k = tid * SC_PER + i;
                F[i] = 0;
                if (k < KEYS && cnt[i]) {
                    long long g = (long long)(k - S.kmin) / w;
                    int gs = (int)(S.kmin + g * w);
                    F[i] = S.first[k] == S.first[gs] ? 1 : 0;
                }
            }
            __syncthreads();
            for (int k = tid; k < KEYS; k += SC_T) S.first[k] = KEYS;
        }
        int ex2[SC_PER];
#pragma unroll
        for (int i = 0; i < SC_PER; ++i) ex2[i] = F[i];
        int nb_scan = block_excl_scan<int>(ex2, reinterpret_cast<int*>(S.red2));
        int nb;
        if (early) nb = 1;
        else if (strategy == QDOT_STRATEGY_SPLIT) nb = nb_scan + 1;   // cuts + 1
        else nb = nb_scan;
#pragma unroll
        for (int i = 0; i < SC_PER; ++i) {
            int k = tid * SC_PER + i;
            bid[i] = -1;
            if (k < KEYS && cnt[i]) {
                if (early) bid[i] = 0;
                else if (strategy == QDOT_STRATEGY_SPLIT) bid[i] = ex2[i];        // cuts before k
                else bid[i] = ex2[i] + F[i] - 1;                                  // starts through k
                S.bin_of[k] = bid[i];
                atomicMin(&S.first[bid[i]], k);
                atomicMax(&S.last[bid[i]], k);
            }
        }
        if (tid == 0) S.s_nb = nb;
    } else {
#pragma unroll
        for (int i = 0; i < SC_PER; ++i) bid[i] = -1;
        if (tid == 0) S.s_nb = 0;
    }
    __syncthreads();
    const int nb = S.s_nb;
    if (tid == 0) {   // scoring.py:192-193
        double eps_eff = (cfg.split == 1 && nb) ? __ddiv_rn(cfg.epsilon, (double)nb) : cfg.epsilon;
        bool ok = true;
        long long fl = floor_log2_d(eps_eff, &ok);
        if (!ok && S.s_status == QDOT_OK && !deg) S.s_status = QDOT_ERR_EPS;
        S.eps_eff = eps_eff;
        S.fl = fl;
    }
    __syncthreads();
    const int e_min = deg ? 0 : S.kmin - KOFF, e_max = deg ? 0 : S.kmax - KOFF;

    // ---- per-bin interval, score, precision (scoring.py:96-123, 181-199)
    for (int b = tid; b < nb; b += SC_T) {
        int f = S.first[b], l = S.last[b];
        long long M = (long long)(S.off[l + 1] - S.off[f]);
        long long upper, lower;
        if (early) { lower = e_min - 1; upper = e_max; }
        else if (strategy == QDOT_STRATEGY_EXACT) { upper = l - KOFF; lower = upper - 1; }
        else if (strategy == QDOT_STRATEGY_RANGED) {
            long long w = cfg.strategy_param;
            long long g = (long long)(f - S.kmin) / w;
            upper = (long long)e_min + (g + 1) * w - 1;
            lower = upper - w;
        } else {
            upper = l - KOFF;
            lower = b ? (long long)(S.last[b - 1] - KOFF) : (long long)e_min - 1;
        }
        unsigned long long mm = (unsigned long long)(M - 1);
        long long cl = mm ? 64 - __clzll((long long)mm) : 0;                    // ceil_log2
        long long score = cl + upper - e_max - S.fl + 1;
        qdot_bin ob;
        ob.lower = lower; ob.upper = upper; ob.cardinality = M; ob.score = score;
        ob.precision = precision_of(score, cfg.input_mu);
        ob.first_key = f; ob.last_key = l; ob.flags = 0; ob.value = 0.0;
        bins[b] = ob;
    }
    __syncthreads();
    __threadfence_block();
    // ---- LUTs
    int need = 0;
    for (int k = tid; k < KEYS; k += SC_T) {
        int b = S.bin_of[k];
        lut_bin[k] = b;
        uint32_t d = 0;
        if (b >= 0) {
            int pr = bins[b].precision;
            long long delta = bins[b].upper - (long long)(k - KOFF);
            if ((pr == QDOT_HALF || pr == QDOT_SINGLE) && delta > 0 && S.s_status == QDOT_OK) {
                d = P2_NEED | (pr == QDOT_HALF ? P2_HALF : 0u) |
                    (uint32_t)(delta > P2_DELTA_MAX ? P2_DELTA_MAX : delta);
                need = 1;
            }
        }
        lut_p2[k] = d;
    }
    need = block_reduce<int>(need, reinterpret_cast<int*>(S.red2), [](int a, int b) { return a | b; }, 0);
    if (tid == 0) {
        ScoreMeta m;
        m.status = S.s_status; m.n_bins = nb; m.e_min = e_min; m.e_max = e_max;
        m.early = early; m.need_p2 = need; m.degenerate = deg; m.input_mu = cfg.input_mu;
        m.nnz = S.nnz; m.zero = A[A_ZERO]; m.n_total = n_total; m.eps_eff = S.eps_eff;
        *meta = m;
    }
}

// =============================================================================
// pass 2 (scaled HALF/SINGLE products for bins with upper > e)
// =============================================================================
constexpr int P2_T = 256;
constexpr int P2_V = 4;
constexpr int P2_TILE = P2_T * P2_V * 2;

struct P2Shared {
    unsigned long long acc[KEYS];
    uint32_t lut[KEYS];
    int need;
};
size_t pass2_smem_bytes() { return sizeof(P2Shared); }

// emulate.py:137-147: sx = x 2^-ex (mantissa mx), sy = y 2^(ex-u) = my 2^-delta;
// round both into the bin format, multiply there; units of 2^qs
__device__ __forceinline__ long long scaled_units(double mx, double my, uint32_t info) {
    int d = (int)(info & 0xFFFFu);
    double sy = my * bitsd((uint64_t)(1023 - d) << 52);       // exact (d <= 255)
    if (info & P2_HALF) {
        __half rx = __double2half(mx), ry = __double2half(sy);
        uint32_t hb = __half_as_ushort(__hmul(rx, ry));
        int E = (hb >> 10) & 0x1F;
        uint32_t M = hb & 0x3FFu;
        if (E) M |= 0x400u; else E = 1;
        int qs = -d - 10 > -24 ? -d - 10 : -24;
        return (long long)M << ((E - 25) - qs);
    } else {
        float rx = __double2float_rn(mx), ry = __double2float_rn(sy);
        uint32_t sb = __float_as_uint(__fmul_rn(rx, ry));
        int E = (sb >> 23) & 0xFF;
        uint32_t M = sb & 0x7FFFFFu;
        if (E) M |= 0x800000u; else E = 1;
        int qs = -d - 23 > -149 ? -d - 23 : -149;
        return (long long)M << ((E - 150) - qs);
    }
}

template <bool NORM, bool VEC>
__global__ void __launch_bounds__(P2_T)
k_pass2(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
        const uint32_t* __restrict__ lut_p2, const ScoreMeta* __restrict__ meta, int64_t* __restrict__ B) {
    if (!meta->need_p2 || meta->status != QDOT_OK) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    P2Shared& S = *reinterpret_cast<P2Shared*>(smem_raw);
    const int tid = threadIdx.x;
    for (int k = tid; k < KEYS; k += P2_T) { S.acc[k] = 0ull; S.lut[k] = lut_p2[k]; }
    __syncthreads();
    const int64_t ntiles = (n + P2_TILE - 1) / P2_TILE;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        double xv[2 * P2_V], yv[2 * P2_V];
        const int64_t e0 = t * P2_TILE;
        const bool full = e0 + P2_TILE <= n;
        if (VEC && full) {
            const double2* x2 = reinterpret_cast<const double2*>(x + e0);
            const double2* y2 = reinterpret_cast<const double2*>(y + e0);
#pragma unroll
            for (int v = 0; v < P2_V; ++v) {
                double2 a = __ldcs(x2 + v * P2_T + tid);
                xv[2 * v] = a.x; xv[2 * v + 1] = a.y;
                if (!NORM) { double2 b2 = __ldcs(y2 + v * P2_T + tid); yv[2 * v] = b2.x; yv[2 * v + 1] = b2.y; }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 2 * P2_V; ++j) {
                int64_t i = e0 + 2 * ((int64_t)(j >> 1) * P2_T + tid) + (j & 1);
                bool ok = i < n;
                xv[j] = ok ? __ldcs(x + i) : 0.0;
                if (!NORM) yv[j] = ok ? __ldcs(y + i) : 0.0;
            }
        }
#pragma unroll
        for (int j = 0; j < 2 * P2_V; ++j) {
            double a = xv[j], b = NORM ? xv[j] : yv[j];
            if (a == 0.0 || b == 0.0) continue;   // zeros and tail padding
            uint64_t bx = dbits(a), by = dbits(b);
            int e = flexp_bits(bx) + flexp_bits(by);
            uint32_t info = S.lut[e + KOFF];
            if (!(info & P2_NEED)) continue;
            long long k = scaled_units(bitsd(mant_bits(bx)), bitsd(mant_bits(by)), info);
            if ((bx ^ by) >> 63) k = -k;
            atomicAdd(&S.acc[e + KOFF], (unsigned long long)k);
        }
    }
    __syncthreads();
    for (int k = tid; k < KEYS; k += P2_T)
        if (S.acc[k]) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_P2 + k), S.acc[k]);
}

// =============================================================================
// finalize (one CTA)
// =============================================================================
constexpr int FN_T = 256;

__device__ __forceinline__ __int128 key_double(const int64_t* __restrict__ B, int k) {
    __int128 v = (__int128)(unsigned long long)B[B_D0 + k];
    v += (__int128)(unsigned long long)B[B_D1 + k] << 32;
    v += (__int128)(unsigned long long)B[B_D2 + k] << 64;
    v += (__int128)(long long)B[B_D3 + k] << 96;
    return v;
}

__global__ void __launch_bounds__(FN_T, 1)
k_finalize(const int64_t* __restrict__ A, const int64_t* __restrict__ B, const ScoreMeta* __restrict__ meta,
           qdot_result* __restrict__ res, qdot_bin* __restrict__ bins) {
    __shared__ int s_ovf, s_half;
    const int tid = threadIdx.x;
    const ScoreMeta m = *meta;
    if (tid == 0) { s_ovf = 0; s_half = 0; }
    __syncthreads();
    const int nb = m.status == QDOT_OK ? m.n_bins : 0;
    for (int b = tid; b < nb; b += FN_T) {
        qdot_bin bn = bins[b];
        const int f = bn.first_key, l = bn.last_key;
        const long long u = bn.upper;
        double val = 0.0;
        int flags = 0;
        if (bn.precision == QDOT_DOUBLE) {
            long long ip = 0, in = 0;
            for (int k = f; k <= l; ++k) { ip += B[B_INFP + k]; in += B[B_INFN + k]; }
            if (ip && in) val = __longlong_as_double(0x7FF8000000000000ll);
            else if (ip) val = INFINITY;
            else if (in) val = -INFINITY;
            else {
                BigSum<104> acc;
                int lsb = qd_double(f - KOFF);
                acc.init(lsb, (qd_double(l - KOFF) - lsb + 160) / 32 + 2);
                for (int k = f; k <= l; ++k)
                    if (A[A_CNT + k]) acc.add(key_double(B, k), qd_double(k - KOFF));
                int ovf = 0;
                val = acc.round(52, -1022, 1023, &ovf);
            }
        } else if (bn.precision != QDOT_PERFORATE) {
            const bool half = bn.precision == QDOT_HALF;
            const int mu = half ? 10 : 23;
            const int qmin_fmt = half ? -24 : -149;
            auto qs_of = [&](int k) {
                long long d = u - (long long)(k - KOFF);
                int dd = d > P2_DELTA_MAX ? P2_DELTA_MAX : (int)d;
                return -dd - mu > qmin_fmt ? -dd - mu : qmin_fmt;
            };
            BigSum<16> acc;
            int lsb = qs_of(f);
            acc.init(lsb, (qs_of(l) - lsb + 128) / 32 + 2);
            double mass = 0.0;   // bound on sum |p| (scaled domain) for the fp32-exactness check
            for (int k = f; k <= l; ++k) {
                long long c = A[A_CNT + k];
                if (!c) continue;
                long long d = u - (long long)(k - KOFF);
                long long v = d == 0 ? (half ? B[B_H0 + k] : B[B_S0 + k]) : B[B_P2 + k];
                acc.add((__int128)v, qs_of(k));
                mass += (double)c * ldexp(4.0, (int)(d > 2000 ? -2000 : -d));
            }
            int ovf = 0;
            double a = half ? acc.round(23, -126, 127, &ovf) : acc.round(52, -1022, 1023, &ovf);
            val = ldexp_rn(a, u, &ovf);                                       // emulate.py:154
            if (ovf) atomicOr(&s_ovf, 1);
            if (half && mass > ldexp(1.0, 24 + lsb)) { flags |= 1; atomicOr(&s_half, 1); }
        }
        bins[b].value = val;
        bins[b].flags = flags;
    }
    __syncthreads();
    if (tid == 0) {
        qdot_result r;
        memset(&r, 0, sizeof(r));
        // qdot_accumulate: Neumaier over bins in ascending-upper order (emulate.py:55-72)
        double s = 0.0, c = 0.0;
        long long cnts[4] = {0, 0, 0, 0};
        for (int b = 0; b < nb; ++b) {
            double v = bins[b].value;
            double t = __dadd_rn(s, v);
            if (fabs(s) >= fabs(v)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), v));
            else c = __dadd_rn(c, __dadd_rn(__dsub_rn(v, t), s));
            s = t;
            cnts[bins[b].precision] += bins[b].cardinality;
        }
        r.value = (s - s == 0.0) ? __dadd_rn(s, c) : s;
        cnts[QDOT_PERFORATE] += m.zero;                                         // kernel.py:175
        for (int i = 0; i < 4; ++i) r.counts[i] = cnts[i];
        r.eps_eff = m.eps_eff;
        r.n = m.n_total;
        r.nnz = m.nnz;
        r.zero_count = m.zero;
        r.status = m.status != QDOT_OK ? m.status : (s_ovf ? QDOT_ERR_OVERFLOW : QDOT_OK);
        r.n_bins = m.n_bins;
        r.e_min = m.e_min;
        r.e_max = m.e_max;
        r.early_terminated = m.early;
        r.pass2_needed = m.need_p2;
        r.half_order_sensitive = s_half;
        *res = r;
    }
}

// =============================================================================
// bin ids (lazy Bin.indices)
// =============================================================================
template <bool NORM>
__global__ void k_bin_ids(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                          const int32_t* __restrict__ lut_bin, int32_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double a = x[i], b = NORM ? a : y[i];
        if (a == 0.0 || b == 0.0) { out[i] = -1; continue; }
        int e = flexp_bits(dbits(a)) + flexp_bits(dbits(b));
        out[i] = lut_bin[e + KOFF];
    }
}

// =============================================================================
// launchers
// =============================================================================
static int sm_count_cached() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (!sms) sms = 148;
    }
    return sms;
}

template <typename K>
static int occupancy(K kern, int threads, size_t smem) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    return occ > 0 ? occ : 1;
}

template <bool NORM, bool VEC>
static cudaError_t launch_pass1_t(const double* x, const double* y, int64_t n, int64_t* A, int64_t* B,
                                  cudaStream_t st) {
    auto kern = k_pass1<NORM, VEC>;
    const size_t smem = sizeof(P1Shared);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    static int occ = 0;
    if (!occ) occ = occupancy(kern, P1_T, smem);
    int64_t ntiles = (n + P1_TILE - 1) / P1_TILE;
    int64_t grid = (int64_t)sm_count_cached() * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, P1_T, smem, st>>>(x, y, n, A, B);
    return cudaGetLastError();
}

cudaError_t launch_pass1(const double* x, const double* y, int64_t n, bool norm, int64_t* A, int64_t* B,
                         cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    bool vec = ((reinterpret_cast<uintptr_t>(x) | (norm ? 0 : reinterpret_cast<uintptr_t>(y))) & 15u) == 0;
    if (norm) return vec ? launch_pass1_t<true, true>(x, x, n, A, B, st) : launch_pass1_t<true, false>(x, x, n, A, B, st);
    return vec ? launch_pass1_t<false, true>(x, y, n, A, B, st) : launch_pass1_t<false, false>(x, y, n, A, B, st);
}

cudaError_t launch_score(const int64_t* A, int32_t* lut_bin, uint32_t* lut_p2, ScoreMeta* meta,
                         qdot_result* res, qdot_bin* bins, int64_t n_total, const qdot_config& cfg,
                         cudaStream_t st) {
    const size_t smem = sizeof(ScShared);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_score, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    k_score<<<1, SC_T, smem, st>>>(A, lut_bin, lut_p2, meta, res, bins, n_total, cfg);
    return cudaGetLastError();
}

template <bool NORM, bool VEC>
static cudaError_t launch_pass2_t(const double* x, const double* y, int64_t n, const uint32_t* lut_p2,
                                  const ScoreMeta* meta, int64_t* B, cudaStream_t st) {
    auto kern = k_pass2<NORM, VEC>;
    const size_t smem = sizeof(P2Shared);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    static int occ = 0;
    if (!occ) occ = occupancy(kern, P2_T, smem);
    int64_t ntiles = (n + P2_TILE - 1) / P2_TILE;
    int64_t grid = (int64_t)sm_count_cached() * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, P2_T, smem, st>>>(x, y, n, lut_p2, meta, B);
    return cudaGetLastError();
}

cudaError_t launch_pass2(const double* x, const double* y, int64_t n, bool norm, const uint32_t* lut_p2,
                         const ScoreMeta* meta, int64_t* B, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    bool vec = ((reinterpret_cast<uintptr_t>(x) | (norm ? 0 : reinterpret_cast<uintptr_t>(y))) & 15u) == 0;
    if (norm) return vec ? launch_pass2_t<true, true>(x, x, n, lut_p2, meta, B, st)
                         : launch_pass2_t<true, false>(x, x, n, lut_p2, meta, B, st);
    return vec ? launch_pass2_t<false, true>(x, y, n, lut_p2, meta, B, st)
               : launch_pass2_t<false, false>(x, y, n, lut_p2, meta, B, st);
}

cudaError_t launch_finalize(const int64_t* A, const int64_t* B, const ScoreMeta* meta, qdot_result* res,
                            qdot_bin* bins, cudaStream_t st) {
    k_finalize<<<1, FN_T, 0, st>>>(A, B, meta, res, bins);
    return cudaGetLastError();
}

cudaError_t launch_bin_ids(const double* x, const double* y, int64_t n, bool norm, const int32_t* lut_bin,
                           int32_t* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t grid = (n + 255) / 256;
    int64_t cap = (int64_t)sm_count_cached() * 8;
    if (grid > cap) grid = cap;
    if (norm) k_bin_ids<true><<<(unsigned)grid, 256, 0, st>>>(x, x, n, lut_bin, out);
    else k_bin_ids<false><<<(unsigned)grid, 256, 0, st>>>(x, y, n, lut_bin, out);
    return cudaGetLastError();
}

}  // namespace qd
