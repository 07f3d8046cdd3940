// qdot_kernels.cu -- sm_100a kernels of the qdot hot path.
//
//   begin     zero the exchange regions and rank-local counters (a normal
//             launch: it orders the call after any kernel that wrote x, y)
//   pass1     streaming pass over x, y (16 B/elem, 8 B/elem in norm mode):
//             exponent extraction, exact exponent-sum histogram, exact per-key
//             DOUBLE partials and exact-binning HALF/SINGLE partials
//             (replaces floatbits.py:57-93, binning.py:88-116 and, for every
//             bin whose products do not depend on the partition, the
//             emulate.py:116-154 bin_dot work).
//   score     one CTA: partition + bin scores + precisions + LUT from the
//             histogram alone (kernel.py:59-72, binning.py:191-284,
//             scoring.py:96-216); single-device calls also finalize here when
//             no pass 2 follows, from key rows staged in shared memory.
//   pass2     second streaming pass, only when a HALF/SINGLE bin has upper
//             u != e for some member key (ranged / split / early bins); on a
//             single device its last CTA finalizes.
//   finalize  one CTA: per-bin exact sums rounded like the reference, and the
//             ascending-upper Neumaier fold (emulate.py:154-163); a separate
//             launch only after the multi-GPU allreduce of region B.
//   pass1, score and pass2 are launched with programmatic dependent launch
//   (eager launches; each waits in griddepcontrol.wait before the workspace).
//   bin_ids   lazy Bin.indices support (binning.py:174).
//
// No tensor cores: this is a memory-bound integer/bit reduction.
#include <cstdlib>

#include <cooperative_groups.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "qdot_common.cuh"
#include "qdot_kernels.h"

namespace qd {

#include "qdot_pass1.cuh"
// norm mode's pass 1: the same code with 11 private slots, four CTAs per SM
namespace p1n {
#undef QDOT_P1_W
#undef QDOT_P1_WW
#undef QDOT_P1_MINB
#define QDOT_P1_W 11
#define QDOT_P1_WW 17
#define QDOT_P1_MINB 4
#include "qdot_pass1.cuh"
}  // namespace p1n

// phase clocks of the score/finalize CTA (scripts/score_prof.cu builds with it)
#ifdef QDOT_SCORE_PROFILE
__device__ long long g_sc_prof[16];
#define SC_STAMP(i) do { if (threadIdx.x == 0) g_sc_prof[i] = clock64(); } while (0)
#else
#define SC_STAMP(i) do { } while (0)
#endif

// =============================================================================
// score (one CTA)
// =============================================================================
constexpr int SC_T = 1024;
constexpr int SC_PER = (KEYS + SC_T - 1) / SC_T;   // 5 keys per thread

// key rows staged in shared memory by the score CTA (cp.async, issued as soon
// as [kmin, kmax] is known, consumed by the per-bin values and the LUT pass)
constexpr int KR_D0 = 0, KR_S0 = 4, KR_H0 = 5, KR_INFP = 6, KR_INFN = 7, KR_HOT = 8, KR_PRIV = 9, KR_ROWS = 10;
constexpr int KC_SPAN = 1024;   // keys cached: spans wider than this read global memory

struct ScShared {
    long long kc[KR_ROWS][KC_SPAN];     // key rows of [kmin, kmin + KC_SPAN)
    double sval[KC_SPAN];               // per-bin values for the fold (cached path)
    unsigned char sflag[KC_SPAN];       // per-bin flags (cached path)
    unsigned long long off[KEYS + 1];   // exclusive prefix of counts over keys
    long long bup[KEYS];                // per-bin upper bound (staged for the LUT pass)
    signed char bprec[KEYS];            // per-bin precision
    int first[KEYS];
    int last[KEYS];
    int bin_of[KEYS];
    unsigned long long red[SC_T / 32];
    long long red2[SC_T / 32];
    int s_status, s_deg, s_early, s_nb, s_need, s_ovf, s_half;
    unsigned long long s_cnt[4];
    int kmin, kmax;
    long long nnz;
    long long a_zero, a_listovf;
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

// round an exact signed integer v * 2^lsb to a binary format (see round_scaled)
__device__ __forceinline__ double round_i128(__int128 v, int lsb, int mu, int emin, int emax, int* ovf) {
    if (v == 0) return 0.0;
    const bool neg = v < 0;
    unsigned __int128 a = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
    const uint64_t hi = (uint64_t)(a >> 64);
    if (mu == 52 || mu == 23) {
        // fast path: the hardware's round-to-nearest-even conversion of the leading
        // 64 bits (the discarded bits OR-ed into bit 0 as sticky: >= 11 bits are
        // dropped, so the round bit is kept), then an exact exponent shift when the
        // result is a normal number strictly inside [emin, emax]
        int sh = 0;
        uint64_t top = (uint64_t)a;
        if (hi) {
            sh = 64 - clz64(hi);
            top = (uint64_t)(a >> sh) | ((a & (((unsigned __int128)1 << sh) - 1)) != 0 ? 1ull : 0ull);
        }
        const double r = mu == 52 ? __ull2double_rn(top) : (double)__ull2float_rn(top);
        const int er = (int)((dbits(r) >> 52) & 0x7FF) - 1023 + lsb + sh;
        if (er > emin && er < emax) {
            const double s = bitsd(dbits(r) + ((uint64_t)(int64_t)(lsb + sh) << 52));
            return neg ? -s : s;
        }
    }
    if (!hi) return round_scaled((uint64_t)a, lsb, false, neg, mu, emin, emax, ovf);
    const int sh = 64 - clz64(hi);                 // bits above the low 64
    const uint64_t top = (uint64_t)(a >> sh);
    const bool sticky = (a & (((unsigned __int128)1 << sh) - 1)) != 0;
    return round_scaled(top, lsb + sh, sticky, neg, mu, emin, emax, ovf);
}

constexpr int FN_CHUNK = 1024;

// key rows of the bin values: global memory (k_finalize, after pass 2) ...
struct GlobalKeys {
    const int64_t* __restrict__ A;
    const int64_t* __restrict__ B;
    const uint32_t* __restrict__ lut_p2;
    __device__ __forceinline__ long long d(int i, int k) const { return B[B_D0 + i * (int64_t)KEYS + k]; }
    __device__ __forceinline__ long long infp(int k) const { return B[B_INFP + k]; }
    __device__ __forceinline__ long long infn(int k) const { return B[B_INFN + k]; }
    __device__ __forceinline__ long long cnt(int k) const { return A[A_CNT + k]; }
    __device__ __forceinline__ long long keyval(int k, bool half) const {
        return (lut_p2[k] & P2_NEED) ? B[B_P2 + k] : (half ? B[B_H0 + k] : B[B_S0 + k]);
    }
};
// ... or the score CTA's shared-memory cache (no pass 2: HALF/SINGLE sums are pass 1's)
struct CachedKeys {
    const long long* kc;                 // [KR_ROWS][KC_SPAN]
    int k0;
    const unsigned long long* off;       // exclusive prefix of counts
    __device__ __forceinline__ long long d(int i, int k) const { return kc[(KR_D0 + i) * KC_SPAN + k - k0]; }
    __device__ __forceinline__ long long infp(int k) const { return kc[KR_INFP * KC_SPAN + k - k0]; }
    __device__ __forceinline__ long long infn(int k) const { return kc[KR_INFN * KC_SPAN + k - k0]; }
    __device__ __forceinline__ long long cnt(int k) const { return (long long)(off[k + 1] - off[k]); }
    __device__ __forceinline__ long long keyval(int k, bool half) const {
        return kc[(half ? KR_H0 : KR_S0) * KC_SPAN + k - k0];
    }
};

template <class K>
__device__ __forceinline__ __int128 key_double(const K& kk, int k) {
    __int128 v = (__int128)(unsigned long long)kk.d(0, k);
    v += (__int128)(unsigned long long)kk.d(1, k) << 32;
    v += (__int128)(unsigned long long)kk.d(2, k) << 64;
    v += (__int128)(long long)kk.d(3, k) << 96;
    return v;
}

// the value of one bin from its exact per-key sums, rounded like the
// reference (emulate.py:116-154); *ovf: a HALF/SINGLE result overflowed,
// *hf: a HALF bin whose fp32 sequential sum could depend on order
template <class K>
__device__ double bin_value(const K& kk, const qdot_bin& bn, int* ovf, int* hf) {
    const int f = bn.first_key, l = bn.last_key;
    const long long u = bn.upper;
    double val = 0.0;
    if (bn.precision == QDOT_DOUBLE) {                                      // emulate.py:132-133
        long long ip = 0, in = 0;
        for (int k = f; k <= l; ++k) { ip += kk.infp(k); in += kk.infn(k); }
        int o = 0;
        if (ip && in) val = __longlong_as_double(0x7FF8000000000000ll);
        else if (ip) val = INFINITY;
        else if (in) val = -INFINITY;
        else if (f == l) val = round_i128(key_double(kk, f), qd_double(f - KOFF), 52, -1022, 1023, &o);
        else {
            BigSum<104> acc;
            int lsb = qd_double(f - KOFF);
            acc.init(lsb, (qd_double(l - KOFF) - lsb + 160) / 32 + 2);
            for (int k = f; k <= l; ++k)
                if (kk.cnt(k)) acc.add(key_double(kk, k), qd_double(k - KOFF));
            val = acc.round(52, -1022, 1023, &o);
        }
    } else if (bn.precision != QDOT_PERFORATE) {                             // emulate.py:135-154
        const bool half = bn.precision == QDOT_HALF;
        const int mu = half ? 10 : 23;
        const int qmin_fmt = half ? -24 : -149;
        auto qs_of = [&](int k) {
            long long d = u - (long long)(k - KOFF);
            int dd = d > P2_DELTA_MAX ? P2_DELTA_MAX : (int)d;
            return -dd - mu > qmin_fmt ? -dd - mu : qmin_fmt;
        };
        const int lsb = qs_of(f);
        double mass = 0.0;   // bound on sum |p| (scaled domain) for the fp32-exactness check
        double a;
        int o = 0;
        if (f == l) {
            a = half ? round_i128((__int128)kk.keyval(f, half), lsb, 23, -126, 127, &o)
                     : round_i128((__int128)kk.keyval(f, half), lsb, 52, -1022, 1023, &o);
            long long d = u - (long long)(f - KOFF);
            mass = (double)kk.cnt(f) * pow2d(2 - (int)(d > 2000 ? 2000 : d));
        } else {
            BigSum<16> acc;
            acc.init(lsb, (qs_of(l) - lsb + 128) / 32 + 2);
            for (int k = f; k <= l; ++k) {
                long long c = kk.cnt(k);
                if (!c) continue;
                long long d = u - (long long)(k - KOFF);
                acc.add((__int128)kk.keyval(k, half), qs_of(k));
                mass += (double)c * pow2d(2 - (int)(d > 2000 ? 2000 : d));
            }
            a = half ? acc.round(23, -126, 127, &o) : acc.round(52, -1022, 1023, &o);
        }
        val = ldexp_rn(a, u, &o);                                             // emulate.py:154
        if (o) *ovf = 1;
        if (half && mass > pow2d(24 + lsb)) *hf = 1;
    }
    return val;
}

// qdot_accumulate: Neumaier over bins in ascending-upper order (emulate.py:55-72)
__device__ __forceinline__ void neumaier_fold(const double* v, int cn, double& sum, double& c) {
    // branch-free: the larger-magnitude operand is the one t is subtracted from
#pragma unroll 4
    for (int i = 0; i < cn; ++i) {
        const double x = v[i];
        const double t = __dadd_rn(sum, x);
        const bool ge = fabs(sum) >= fabs(x);
        const double big = ge ? sum : x, small = ge ? x : sum;
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(big, t), small));
        sum = t;
    }
}

// per-thread precision counts -> shared totals (any block size)
__device__ __forceinline__ void block_count_reduce(const long long (&cnt_local)[4], unsigned long long* s_cnt) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        long long v = cnt_local[p];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_cnt[p], (unsigned long long)v);
    }
}

// the result header (kernel.py:175, scoring.py:192-216) and the phase times
__device__ void write_result(unsigned long long ts0, unsigned long long ts1, const ScoreMeta& m, double sum, double c,
                             const unsigned long long* s_cnt, int s_ovf, int s_half, qdot_result* __restrict__ res) {
    // field by field (a local struct + memset would go through local memory)
    qdot_result* r = res;
    r->value = (sum - sum == 0.0) ? __dadd_rn(sum, c) : sum;
    for (int i = 0; i < 4; ++i)
        r->counts[i] = (long long)s_cnt[i] + (i == QDOT_PERFORATE ? m.zero : 0);   // kernel.py:175
    r->eps_eff = m.eps_eff;
    r->n = m.n_total;
    r->nnz = m.nnz;
    r->zero_count = m.zero;
    r->status = m.status != QDOT_OK ? m.status : (s_ovf ? QDOT_ERR_OVERFLOW : QDOT_OK);
    r->n_bins = m.n_bins;
    r->e_min = m.e_min;
    r->e_max = m.e_max;
    r->early_terminated = m.early;
    r->pass2_needed = m.need_p2;
    r->half_order_sensitive = s_half;
    const unsigned long long now = global_ns();
    const unsigned long long sel = ts1 > ts0 ? ts1 - ts0 : 0ull, cmp = now > ts1 ? now - ts1 : 0ull;
    r->select_ns = (int32_t)(sel < 0x7FFFFFFFull ? sel : 0x7FFFFFFFull);
    r->compute_ns = (int32_t)(cmp < 0x7FFFFFFFull ? cmp : 0x7FFFFFFFull);
    r->reserved[0] = 0; r->reserved[1] = 0; r->reserved[2] = 0;
}

// per-bin values + Neumaier fold + result header from global memory; any
// block size (k_finalize, and k_score when its key cache does not apply)
__device__ void finalize_body(const int64_t* __restrict__ A, const int64_t* __restrict__ B,
                              const uint32_t* __restrict__ lut_p2, const ScoreMeta& m, qdot_result* __restrict__ res,
                              qdot_bin* __restrict__ bins) {
    const int nthr = blockDim.x;
    __shared__ double s_val[FN_CHUNK];
    __shared__ int s_ovf, s_half;
    __shared__ double s_s, s_c;
    __shared__ unsigned long long s_cnt[4];
    const int tid = threadIdx.x;
    if (tid == 0) { s_ovf = 0; s_half = 0; s_s = 0.0; s_c = 0.0; s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0; }
    SC_STAMP(8);
    __syncthreads();
    const int nb = m.status == QDOT_OK ? m.n_bins : 0;
    const GlobalKeys kk{A, B, lut_p2};
    long long cnt_local[4] = {0, 0, 0, 0};   // per-thread precision counts (summed after the bins)
    for (int base = 0; base < nb; base += FN_CHUNK) {
        const int cn = nb - base < FN_CHUNK ? nb - base : FN_CHUNK;
        for (int i = tid; i < cn; i += nthr) {
            const int b = base + i;
            const qdot_bin bn = bins[b];
            int ovf = 0, hf = 0;
            const double val = bin_value(kk, bn, &ovf, &hf);
            if (ovf) atomicOr(&s_ovf, 1);
            if (hf) atomicOr(&s_half, 1);
            bins[b].value = val;
            bins[b].flags = hf;
            s_val[i] = val;
#pragma unroll
            for (int p = 0; p < 4; ++p) cnt_local[p] += bn.precision == p ? bn.cardinality : 0;
        }
        __syncthreads();
        SC_STAMP(9);
        if (tid == 0) {
            double sum = s_s, c = s_c;
            neumaier_fold(s_val, cn, sum, c);
            s_s = sum;
            s_c = c;
        }
        __syncthreads();
        SC_STAMP(10);
    }
    block_count_reduce(cnt_local, s_cnt);
    __syncthreads();
    SC_STAMP(11);
    if (tid == 0) write_result(ws_stamps(A)[0], ws_stamps(A)[1], m, s_s, s_c, s_cnt, s_ovf, s_half, res);
    SC_STAMP(12);
}

__global__ void __launch_bounds__(FN_T, 1)
k_finalize(const int64_t* __restrict__ A, const int64_t* __restrict__ B, const uint32_t* __restrict__ lut_p2,
           const ScoreMeta* __restrict__ meta, qdot_result* __restrict__ res, qdot_bin* __restrict__ bins) {
    const ScoreMeta m = *meta;
    if (m.done) return;
    finalize_body(A, B, lut_p2, m, res, bins);
}


// =============================================================================
// score, one warp (single device, keys spanning < 64 exponents: the solver
// regime).  The same partition / scores / precisions / LUTs / meta as the
// block path below, from bit masks over the 64 keys [kmin, kmin + 64) (lane
// owns keys kmin + lane and kmin + lane + 32); when no pass 2 follows, the
// bin values (bin_value over the global key rows), the fold and the result
// header too.  Saves the block path's ~15 barrier phases per call.
// =============================================================================
constexpr int SW_KEYS = 64;

// where score_warp reads the per-key totals: the global exchange regions (k_score) ...
struct GlobalSrc {
    const int64_t* __restrict__ A;
    const int64_t* __restrict__ B;
    const uint32_t* __restrict__ lut_p2;
    __device__ __forceinline__ long long cnt(int k) const { return A[A_CNT + k]; }
    __device__ __forceinline__ long long hot(int k) const { return A[A_HOT + k]; }
    __device__ __forceinline__ long long priv(int k) const { return A[A_PRIV + k]; }
    __device__ __forceinline__ GlobalKeys keys() const { return GlobalKeys{A, B, lut_p2}; }
};

template <class Src>
__device__ int score_warp(const Src& src, const int64_t* __restrict__ A, int32_t* __restrict__ lut_bin,
                           uint32_t* __restrict__ lut_p2, ScoreMeta* __restrict__ meta, qdot_result* __restrict__ res,
                           qdot_bin* __restrict__ bins, int64_t n_total, const qdot_config& cfg, int kmin, int kmax,
                           unsigned long long ts0, long long a_nonfinite, long long a_zero, long long a_listovf,
                           double* sval, long long* bup, signed char* bprec, long long* dbg = nullptr) {
    const int lane = threadIdx.x & 31;
    const long long dc0 = clock64();
    auto mark = [&](int i) { if (dbg && lane == 0) dbg[i] = clock64() - dc0; };
    long long c[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = kmin + lane + 32 * h;
        c[h] = (k <= kmax) ? src.cnt(k) : 0;
    }
    const unsigned long long P = (unsigned long long)__ballot_sync(0xffffffffu, c[0] != 0) |
                                 ((unsigned long long)__ballot_sync(0xffffffffu, c[1] != 0) << 32);
    // exclusive prefix of the counts: off(j) for the lane's keys, nnz
    unsigned long long i0 = (unsigned long long)c[0], i1 = (unsigned long long)c[1];
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= o) { i0 += t0; i1 += t1; }
    }
    const unsigned long long tot0 = __shfl_sync(0xffffffffu, i0, 31);
    const unsigned long long nnz = tot0 + __shfl_sync(0xffffffffu, i1, 31);
    const unsigned long long off[2] = {i0 - (unsigned long long)c[0], tot0 + i1 - (unsigned long long)c[1]};
    auto off_of = [&](int j) -> unsigned long long {     // exclusive prefix at key kmin + j (j <= 64)
        // every lane supplies both halves: lanes may ask for different ones
        const unsigned long long v0 = __shfl_sync(0xffffffffu, off[0], j & 31);
        const unsigned long long v1 = __shfl_sync(0xffffffffu, off[1], j & 31);
        return j >= SW_KEYS ? nnz : (j < 32 ? v0 : v1);
    };
    int status = a_nonfinite ? QDOT_ERR_NONFINITE : QDOT_OK;                   // floatbits.py:70
    bool ok = true;
    const long long fle = floor_log2_d(cfg.epsilon, &ok);
    if (!ok && status == QDOT_OK) status = QDOT_ERR_EPS;
    int early = 0;
    if (ok) {                                                                  // scoring.py:126-136
        const int mu_hat = cfg.input_mu == 52 ? 23 : (cfg.input_mu == 23 ? 10 : 0);
        early = (long long)(kmax - kmin) <= (-fle - mu_hat);
    }
    // ---- bin starts (bit j: key kmin + j starts a bin)
    const int jmin = 0;
    unsigned long long S;
    const int strategy = cfg.strategy;
    if (early) {
        S = 1ull;
    } else if (strategy == QDOT_STRATEGY_EXACT) {
        S = P;
    } else if (strategy == QDOT_STRATEGY_RANGED) {
        const long long w = cfg.strategy_param;
        bool f[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            f[h] = false;
            if ((P >> j) & 1ull) {
                const int gs = jmin + (int)(((long long)(j - jmin) / w) * w);
                const unsigned long long below = ((1ull << j) - 1ull) ^ ((1ull << gs) - 1ull);
                f[h] = (P & below) == 0ull;
            }
        }
        S = (unsigned long long)__ballot_sync(0xffffffffu, f[0]) |
            ((unsigned long long)__ballot_sync(0xffffffffu, f[1]) << 32);
    } else {
        long long levels = cfg.strategy_param;                                  // binning.py:235
        const unsigned long long t = nnz > 1 ? nnz - 1 : 0;
        const int bl = t ? 64 - __clzll((long long)t) : 0;
        if (levels > bl) levels = bl;
        uint32_t nx[2] = {0u, 0u};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            if (!((P >> j) & 1ull)) continue;
            const unsigned long long a = off[h], b = a + (unsigned long long)c[h];
            if (b < nnz && split_boundary_in(nnz, (int)levels, a, b)) {
                const unsigned long long rest = j == 63 ? 0ull : (P & ~((2ull << j) - 1ull));
                const int nj = __ffsll((long long)rest) - 1;
                nx[nj >> 5] |= 1u << (nj & 31);
            }
        }
        S = (unsigned long long)__reduce_or_sync(0xffffffffu, nx[0]) |
            ((unsigned long long)__reduce_or_sync(0xffffffffu, nx[1]) << 32) | 1ull;
    }
    mark(0);
    const int nb = __popcll(S);
    const double eps_eff = (cfg.split == 1 && nb) ? __ddiv_rn(cfg.epsilon, (double)nb) : cfg.epsilon;   // scoring.py:192
    bool okf = true;
    const long long fl = floor_log2_d(eps_eff, &okf);
    if (!okf && status == QDOT_OK) status = QDOT_ERR_EPS;
    const int e_min = kmin - KOFF, e_max = kmax - KOFF;
    // ---- per bin (lane owning its first key): interval, score, precision, LUT entries
    int need = 0, priv = 0;
    qdot_bin ob[2];
    int bidx[2] = {-1, -1};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (!((S >> j) & 1ull)) continue;
        const int b = __popcll(S & ((1ull << j) - 1ull));
        const unsigned long long rest = j == 63 ? 0ull : (S & ~((2ull << j) - 1ull));
        const int nf = rest ? __ffsll((long long)rest) - 1 : SW_KEYS;
        const unsigned long long upto = nf == SW_KEYS ? ~0ull : ((1ull << nf) - 1ull);
        const int l = 63 - __clzll((long long)(P & upto));
        bidx[h] = b;
        ob[h].first_key = kmin + j;
        ob[h].last_key = kmin + l;
        ob[h].flags = 0;
        ob[h].value = 0.0;
    }
    // M needs the prefix at arbitrary keys: shuffles are warp-collective, so
    // every lane evaluates them for both of its (possible) bins
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        const unsigned long long rest = j == 63 ? 0ull : (S & ~((2ull << j) - 1ull));
        const int nf = rest ? __ffsll((long long)rest) - 1 : SW_KEYS;
        const unsigned long long a = off_of(j & 63), b = off_of(nf);
        if (bidx[h] < 0) continue;
        const long long M = (long long)(b - a);
        const int f = ob[h].first_key, l = ob[h].last_key;
        long long upper, lower;
        if (early) { lower = e_min - 1; upper = e_max; }
        else if (strategy == QDOT_STRATEGY_EXACT) { upper = l - KOFF; lower = upper - 1; }
        else if (strategy == QDOT_STRATEGY_RANGED) {
            const long long w = cfg.strategy_param;
            const long long g = (long long)(f - kmin) / w;
            upper = (long long)e_min + (g + 1) * w - 1;
            lower = upper - w;
        } else {
            upper = l - KOFF;
            const unsigned long long pb = P & ((1ull << j) - 1ull);
            lower = pb ? (long long)(kmin + (63 - __clzll((long long)pb)) - KOFF) : (long long)e_min - 1;
        }
        const unsigned long long mm = (unsigned long long)(M - 1);
        const long long score = (mm ? 64 - __clzll((long long)mm) : 0) + upper - e_max - fl + 1;   // bin_score
        ob[h].lower = lower; ob[h].upper = upper; ob[h].cardinality = M; ob[h].score = score;
        ob[h].precision = precision_of(score, cfg.input_mu);
        bins[bidx[h]] = ob[h];
        bup[bidx[h]] = upper;
        bprec[bidx[h]] = (signed char)ob[h].precision;
    }
    __syncwarp();
    mark(1);
    // ---- LUTs over [kmin, kmax] (lane's keys): bin id, pass-2 descriptor
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        const int k = kmin + j;
        if (k > kmax) continue;
        const bool present = (P >> j) & 1ull;
        const int b = present ? __popcll(S & ((2ull << j) - 1ull)) - 1 : -1;   // starts <= j, minus 1
        lut_bin[k] = b;
        uint32_t d = 0;
        if (b >= 0) {
            const int pr = bprec[b];
            if ((pr == QDOT_HALF || pr == QDOT_SINGLE) && status == QDOT_OK) {
                const long long delta = bup[b] - (long long)(k - KOFF);
                if (delta > 0 || src.hot(k) > 0) {
                    d = P2_NEED | (pr == QDOT_HALF ? P2_HALF : 0u) | (uint32_t)(delta > P2_DELTA_MAX ? P2_DELTA_MAX : delta);
                    need = 1;
                    if (src.priv(k) > 0) priv = 1;
                }
            }
        }
        lut_p2[k] = d;
    }
    need = __reduce_or_sync(0xffffffffu, need);
    priv = __reduce_or_sync(0xffffffffu, priv);
    if (need) need = (!priv && a_listovf == 0) ? 2 : 1;
    ScoreMeta m;
    m.status = status; m.n_bins = nb; m.e_min = e_min; m.e_max = e_max;
    m.early = early; m.need_p2 = need; m.degenerate = 0; m.input_mu = cfg.input_mu;
    m.done = need ? 0 : 1; m.pad_ = 0;
    m.nnz = (long long)nnz; m.zero = a_zero; m.n_total = n_total; m.eps_eff = eps_eff;
    if (lane == 0) *meta = m;
    unsigned long long ts1 = 0;
    if (lane == 0) { ts1 = global_ns(); ws_stamps(A)[1] = ts1; }
    mark(2);
    if (need) return need;                                               // pass 2 finalizes
    __syncwarp();
    // ---- bin values, precision counts, fold, header
    long long cnt_local[4] = {0, 0, 0, 0};
    int ovf = 0, half = 0;
    const auto kk = src.keys();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (bidx[h] < 0 || status != QDOT_OK) continue;
        int o = 0, hf = 0;
        const double v = bin_value(kk, ob[h], &o, &hf);
        ovf |= o;
        half |= hf;
        bins[bidx[h]].value = v;
        bins[bidx[h]].flags = hf;
        sval[bidx[h]] = v;
#pragma unroll
        for (int p = 0; p < 4; ++p) cnt_local[p] += ob[h].precision == p ? ob[h].cardinality : 0;
    }
    mark(3);
    ovf = __reduce_or_sync(0xffffffffu, ovf);
    half = __reduce_or_sync(0xffffffffu, half);
    unsigned long long s_cnt[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        long long v = cnt_local[p];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        s_cnt[p] = (unsigned long long)v;
    }
    __syncwarp();
    if (lane == 0) {
        double sum = 0.0, cc = 0.0;
        neumaier_fold(sval, status == QDOT_OK ? nb : 0, sum, cc);
        mark(4);
        write_result(ts0, ts1, m, sum, cc, s_cnt, ovf, half, res);
        mark(5);
    }
    return 0;
}
// =============================================================================
// score (one CTA)
// =============================================================================
__global__ void __launch_bounds__(SC_T, 1)
k_score(const int64_t* __restrict__ A, const int64_t* __restrict__ B, int32_t* __restrict__ lut_bin, uint32_t* __restrict__ lut_p2,
        ScoreMeta* __restrict__ meta, qdot_result* __restrict__ res, qdot_bin* __restrict__ bins,
        int64_t n_total, qdot_config cfg, int fuse) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScShared& S = *reinterpret_cast<ScShared*>(smem_raw);
    const int tid = threadIdx.x;
    pdl_wait();
    pdl_trigger();
    if (A[A_SMALL] == 1) return;          // k_small scored and finalized this call
    SC_STAMP(0);

    // the flag words are loaded up front so their latency overlaps the counts'
    long long a_nonfinite = 0, a_zero = 0, a_listovf = 0;
    unsigned long long ts0 = 0, ts1 = 0;
    if (tid == 0) {
        a_nonfinite = A[A_NONFINITE]; a_zero = A[A_ZERO]; a_listovf = A[A_LISTOVF];
        ts0 = ws_stamps(A)[0];
    }
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
    {   // one reduction for both, component-wise min of (kmin, KEYS - kmax) in 16-bit halves
        const unsigned packed = ((unsigned)kmin << 16) | (unsigned)(KEYS - kmax);
        const unsigned r = block_reduce<unsigned>(
            packed, reinterpret_cast<unsigned*>(S.red2),
            [](unsigned a, unsigned b) { return (min(a >> 16, b >> 16) << 16) | min(a & 0xFFFFu, b & 0xFFFFu); },
            0xFFFFFFFFu);
        kmin = (int)(r >> 16);
        kmax = KEYS - (int)(r & 0xFFFFu);
    }
    // one device, keys spanning < 64 exponents: one warp scores (and finalizes)
#ifndef QDOT_NO_SCORE_WARP
    if (fuse && kmax >= kmin && kmax - kmin < SW_KEYS) {
        if (tid < 32) {
            const long long nf0 = __shfl_sync(0xffffffffu, a_nonfinite, 0);
            const long long z0 = __shfl_sync(0xffffffffu, a_zero, 0);
            const long long lo0 = __shfl_sync(0xffffffffu, a_listovf, 0);
            const unsigned long long t0 = __shfl_sync(0xffffffffu, ts0, 0);
            score_warp(GlobalSrc{A, B, lut_p2}, A, lut_bin, lut_p2, meta, res, bins, n_total, cfg, kmin, kmax, t0, nf0,
                       z0, lo0, S.sval, S.bup, S.bprec);
        }
        return;
    }
#endif
    // cached path: stage the key rows the bin values and the LUT read
    const bool kcache = fuse && kmax >= kmin && kmax - kmin < KC_SPAN;
    for (int j = tid; kcache && j <= kmax - kmin; j += SC_T) {
        const int k = kmin + j;
        const int64_t* src[KR_ROWS] = {B + B_D0 + k, B + B_D1 + k, B + B_D2 + k, B + B_D3 + k, B + B_S0 + k,
                                       B + B_H0 + k, B + B_INFP + k, B + B_INFN + k, A + A_HOT + k, A + A_PRIV + k};
#pragma unroll
        for (int r = 0; r < KR_ROWS; ++r) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(&S.kc[r][j]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(src[r]) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    SC_STAMP(1);
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
        if (a_nonfinite) status = QDOT_ERR_NONFINITE;                             // floatbits.py:70
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
        S.a_zero = a_zero; S.a_listovf = a_listovf;
        S.s_ovf = 0; S.s_half = 0;
        S.s_cnt[0] = S.s_cnt[1] = S.s_cnt[2] = S.s_cnt[3] = 0;
    }
    __syncthreads();
    SC_STAMP(2);
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
    SC_STAMP(3);
    const int nb = S.s_nb;
    if (tid == 0) {   // scoring.py:192-193
        double eps_eff = (cfg.split == 1 && nb) ? __ddiv_rn(cfg.epsilon, (double)nb) : cfg.epsilon;
        bool ok = true;
        long long fl = floor_log2_d(eps_eff, &ok);
        if (!ok && S.s_status == QDOT_OK && !deg) S.s_status = QDOT_ERR_EPS;
        S.eps_eff = eps_eff;
        S.fl = fl;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    SC_STAMP(4);
    const int e_min = deg ? 0 : S.kmin - KOFF, e_max = deg ? 0 : S.kmax - KOFF;

    // ---- per-bin interval, score, precision (scoring.py:96-123, 181-199)
    int my_ovf = 0, my_half = 0;
    long long cnt_local[4] = {0, 0, 0, 0};
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
        S.bup[b] = upper;
        S.bprec[b] = (signed char)ob.precision;
        if (kcache) {   // speculative: valid when no pass 2 follows (then finalized below)
            int ovf = 0, hf = 0;
            SC_STAMP(9);
            S.sval[b] = bin_value(CachedKeys{&S.kc[0][0], S.kmin, S.off}, ob, &ovf, &hf);
            SC_STAMP(10);
            S.sflag[b] = (unsigned char)hf;
            my_ovf |= ovf;
            my_half |= hf;
#pragma unroll
            for (int p = 0; p < 4; ++p) cnt_local[p] += ob.precision == p ? M : 0;
        }
    }
    __syncthreads();
    SC_STAMP(5);
    __threadfence_block();
    // ---- LUTs.  need: some key needs pass 2; priv: such a key also has
    // elements accumulated in private windows (not in the cold-element list)
    // only keys in [kmin, kmax] are ever looked up (pass 2 by element keys,
    // finalize by bin keys), so stale entries outside the range are harmless
    int need = 0, priv = 0;
    const int lut_lo = deg ? 0 : S.kmin, lut_hi = deg ? -1 : S.kmax;
    for (int k = lut_lo + tid; k <= lut_hi; k += SC_T) {
        int b = S.bin_of[k];
        lut_bin[k] = b;
        uint32_t d = 0;
        if (b >= 0) {
            int pr = S.bprec[b];
            long long delta = S.bup[b] - (long long)(k - KOFF);
            const long long hot = kcache ? S.kc[KR_HOT][k - lut_lo] : A[A_HOT + k];
            if ((pr == QDOT_HALF || pr == QDOT_SINGLE) && (delta > 0 || hot > 0) && S.s_status == QDOT_OK) {
                d = P2_NEED | (pr == QDOT_HALF ? P2_HALF : 0u) |
                    (uint32_t)(delta > P2_DELTA_MAX ? P2_DELTA_MAX : delta);
                need = 1;
                if ((kcache ? S.kc[KR_PRIV][k - lut_lo] : A[A_PRIV + k]) > 0) priv = 1;
            }
        }
        lut_p2[k] = d;
    }
    SC_STAMP(6);
    {
        const int np = block_reduce<int>(need | (priv << 1), reinterpret_cast<int*>(S.red2),
                                         [](int a, int b) { return a | b; }, 0);
        need = np & 1;
        priv = np >> 1;
    }
    // pass 2 mode: 2 = only over the cold-element list (every element of every
    // pass-2 key is in it, no slot overflowed), 1 = stream x and y again
    if (need) need = (!priv && S.a_listovf == 0) ? 2 : 1;
    __shared__ ScoreMeta sm;
    if (tid == 0) {
        ScoreMeta m;
        m.status = S.s_status; m.n_bins = nb; m.e_min = e_min; m.e_max = e_max;
        m.early = early; m.need_p2 = need; m.degenerate = deg; m.input_mu = cfg.input_mu;
        m.done = (fuse && !need) ? 1 : 0; m.pad_ = 0;
        m.nnz = S.nnz; m.zero = S.a_zero; m.n_total = n_total; m.eps_eff = S.eps_eff;
        sm = m;
        *meta = m;
    }
    if (tid == 0) { ts1 = global_ns(); ws_stamps(A)[1] = ts1; }   // parameter selection done
    __syncthreads();
    SC_STAMP(7);
    // no pass 2 needed (the common case): finalize here and save a launch;
    // k_finalize then exits on meta->done
    if (!sm.done) return;
    if (!kcache) { finalize_body(A, B, lut_p2, sm, res, bins); return; }
    // cached path: the bin values are already computed; fold + header
    SC_STAMP(8);
    const int nbv = sm.status == QDOT_OK ? nb : 0;
    if (nbv) {
        for (int b = tid; b < nbv; b += SC_T) { bins[b].value = S.sval[b]; bins[b].flags = S.sflag[b]; }
        if (my_ovf) atomicOr(&S.s_ovf, 1);
        if (my_half) atomicOr(&S.s_half, 1);
        block_count_reduce(cnt_local, S.s_cnt);
    }
    __syncthreads();
    SC_STAMP(11);
    if (tid == 0) {
        double sum = 0.0, c = 0.0;
        neumaier_fold(S.sval, nbv, sum, c);
        write_result(ts0, ts1, sm, sum, c, S.s_cnt, S.s_ovf, S.s_half, res);
    }
    SC_STAMP(12);
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

// one element of pass 2 (zeros and tail padding contribute nothing)
__device__ __forceinline__ void p2_elem(P2Shared& S, double a, double b) {
    if (a == 0.0 || b == 0.0) return;
    const uint64_t bx = dbits(a), by = dbits(b);
    const int e = flexp_bits(bx) + flexp_bits(by);
    const uint32_t info = S.lut[e + KOFF];
    if (!(info & P2_NEED)) return;
    long long k = scaled_units(bitsd(mant_bits(bx)), bitsd(mant_bits(by)), info);
    if ((bx ^ by) >> 63) k = -k;
    atomicAdd(&S.acc[e + KOFF], (unsigned long long)k);
}

template <bool NORM, bool VEC>
__device__ __forceinline__ void p2_body(P2Shared& S, const double* __restrict__ x, const double* __restrict__ y,
                                        int64_t n, const uint32_t* __restrict__ lut_p2, int mode,
                                        int64_t* __restrict__ B, const double2* __restrict__ list,
                                        const uint32_t* __restrict__ list_fill) {
    const int tid = threadIdx.x;
    for (int k = tid; k < KEYS; k += P2_T) { S.acc[k] = 0ull; S.lut[k] = lut_p2[k]; }
    __syncthreads();
    if (mode == 2) {
        // only the cold-element list: slot s holds list_fill[s] entries
        for (int sl = blockIdx.x; sl < (int)LIST_SLOTS; sl += gridDim.x) {
            const uint32_t cnt = min(list_fill[sl], (uint32_t)LIST_PER_SLOT);
            for (uint32_t i = tid; i < cnt; i += P2_T) {
                const double2 e = list[(int64_t)sl * LIST_PER_SLOT + i];
                p2_elem(S, e.x, e.y);
            }
        }
        __syncthreads();
        for (int k = tid; k < KEYS; k += P2_T)
            if (S.acc[k]) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_P2 + k), S.acc[k]);
        return;
    }
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
        for (int j = 0; j < 2 * P2_V; ++j) p2_elem(S, xv[j], NORM ? xv[j] : yv[j]);
    }
    __syncthreads();
    for (int k = tid; k < KEYS; k += P2_T)
        if (S.acc[k]) atomicAdd(reinterpret_cast<unsigned long long*>(B + B_P2 + k), S.acc[k]);
}

template <bool NORM, bool VEC>
__global__ void __launch_bounds__(P2_T)
k_pass2(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
        const uint32_t* __restrict__ lut_p2, const ScoreMeta* __restrict__ meta, int64_t* __restrict__ B,
        const double2* __restrict__ list, const uint32_t* __restrict__ list_fill, int fin,
        const int64_t* __restrict__ A, qdot_result* __restrict__ res, qdot_bin* __restrict__ bins) {
    pdl_wait();
    const int mode = meta->need_p2;
    const bool work = mode && meta->status == QDOT_OK;
    // fin: the last CTA to finish also finalizes (unless score already did)
    const bool finish = fin && !meta->done;
    if (!work && !finish) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    P2Shared& S = *reinterpret_cast<P2Shared*>(smem_raw);
    const int tid = threadIdx.x;
    if (work) p2_body<NORM, VEC>(S, x, y, n, lut_p2, mode, B, list, list_fill);
    if (!finish) return;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        unsigned long long* ticket = ws_stamps(A) + 4;     // zeroed by begin
        S.need = atomicAdd(ticket, 1ull) == gridDim.x - 1ull;
    }
    __syncthreads();
    if (!S.need) return;
    __threadfence();
    const ScoreMeta m = *meta;
    finalize_body(A, B, lut_p2, m, res, bins);
}


#include "qdot_batched.cuh"
#include "qdot_small.cuh"

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
// launch with programmatic stream serialization (QDOT_B200_PDL=0 disables):
// the kernel may begin while its predecessor in the stream drains and calls
// pdl_wait() before it touches anything that predecessor writes
static bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("QDOT_B200_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(block);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    // eager launches only: inside a CUDA graph capture the programmatic edges
    // measured no gain (graph replay already removes the launch gaps)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (pdl_enabled()) cudaStreamIsCapturing(st, &cap);
    at[0].val.programmaticStreamSerializationAllowed = (pdl_enabled() && cap == cudaStreamCaptureStatusNone) ? 1 : 0;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, kern, static_cast<KArgs>(args)...);
}

// zero regions A, B and the rank-local counters (replaces a memset so that
// pass 1, launched after it with programmatic serialization, can sample its
// inputs while this runs); launched normally: it waits for all prior work
__global__ void __launch_bounds__(256) k_begin(ulonglong2* __restrict__ p, int64_t n16) {
    pdl_trigger();
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n16; i += (int64_t)gridDim.x * 256)
        p[i] = make_ulonglong2(0ull, 0ull);
}

static int sm_count_cached() { return device_sm_count(); }

// NARROW: the 11-slot build (namespace p1n; norm mode)
template <bool NORM, bool VEC, int V, bool PF, int L2D, bool SMALL = false, bool NARROW = false>
static cudaError_t launch_pass1_t(const double* x, const double* y, int64_t n, int64_t* A, int64_t* B,
                                  const P1Params& prm, cudaStream_t st) {
    auto kern = NARROW ? p1n::k_pass1<NORM, VEC, V, PF, L2D, SMALL> : k_pass1<NORM, VEC, V, PF, L2D, SMALL>;
    const size_t smem = NARROW ? sizeof(p1n::P1Shared) : sizeof(P1Shared);
    static KernelDevCache cache;
    int occ = kernel_occupancy(kern, P1_T, smem, cache);
    {   // QDOT_B200_P1_OCC=k: at most k CTAs per SM in the grid (occupancy experiments)
        static int cap = -1;
        if (cap < 0) { const char* e = getenv("QDOT_B200_P1_OCC"); cap = e ? atoi(e) : 0; }
        if (cap > 0 && cap < occ) occ = cap;
    }
    const int64_t tile = (int64_t)P1_T * 2 * V;
    int64_t ntiles = (n + tile - 1) / tile;
    int64_t grid = (int64_t)sm_count_cached() * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    return launch_pdl(kern, (unsigned)grid, P1_T, smem, st, x, y, n, A, B, prm);
}

#ifdef QDOT_B200_P1_TUNING
// pass-1 variant (vector width / prefetch); QDOT_B200_P1_VARIANT overrides for tuning
static int p1_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("QDOT_B200_P1_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}
#endif

template <bool NORM, bool VEC>
static cudaError_t launch_pass1_v(const double* x, const double* y, int64_t n, int64_t* A, int64_t* B,
                                  const P1Params& prm, cudaStream_t st) {
    // short inputs (at most two tiles per SM): the compact variant
    if ((prm.mode >> 2) == 0 && (prm.mode & 3) == 0 && n <= (int64_t)sm_count_cached() * 2 * (P1_T * 8))
        return launch_pass1_t<NORM, VEC, 4, false, 0, true>(x, y, n, A, B, prm, st);
#ifdef QDOT_B200_P1_TUNING
    // tuning builds only (-DQDOT_B200_P1_TUNING): alternative pass-1 shapes
    switch (p1_variant()) {
        case 1: return launch_pass1_t<NORM, VEC, 4, false, 0>(x, y, n, A, B, prm, st);   // no L2 prefetch
        case 2: return launch_pass1_t<NORM, VEC, 2, false, 3>(x, y, n, A, B, prm, st);
        case 3: return launch_pass1_t<NORM, VEC, 4, false, 2>(x, y, n, A, B, prm, st);
        case 4: return launch_pass1_t<NORM, VEC, 2, true, 0>(x, y, n, A, B, prm, st);    // register double buffer
        case 5: return launch_pass1_t<NORM, VEC, 4, false, 5>(x, y, n, A, B, prm, st);
        case 6: return launch_pass1_t<NORM, VEC, 4, false, 7>(x, y, n, A, B, prm, st);
        case 7: return launch_pass1_t<NORM, VEC, 2, false, 6>(x, y, n, A, B, prm, st);
        case 8: return launch_pass1_t<NORM, VEC, 2, false, 10>(x, y, n, A, B, prm, st);
        case 9: return launch_pass1_t<NORM, VEC, 4, true, 3>(x, y, n, A, B, prm, st);    // registers + L2
        case 10: return launch_pass1_t<NORM, VEC, 2, true, 3>(x, y, n, A, B, prm, st);
        case 11: return launch_pass1_t<NORM, VEC, 2, true, 6>(x, y, n, A, B, prm, st);
        default: break;
    }
#endif
    // V = 4 double2 per thread per tile, bulk L2 prefetch 4 tiles ahead: tuned on
    // B200 (norm mode: V = 8 measured slower)
    if (NORM) {   // norm mode: the 11-slot build, four CTAs per SM (QDOT_B200_P1_NARROW=0: the 16-slot one)
        static int narrow = -1;
        if (narrow < 0) { const char* e = getenv("QDOT_B200_P1_NARROW"); narrow = (e && e[0] == '0') ? 0 : 1; }
        if (narrow) return launch_pass1_t<NORM, VEC, 4, false, 3, false, true>(x, y, n, A, B, prm, st);
    }
    return launch_pass1_t<NORM, VEC, 4, false, 3>(x, y, n, A, B, prm, st);
}

cudaError_t launch_pass1(const double* x, const double* y, int64_t n, bool norm, int64_t* A, int64_t* B,
                         const P1Params& prm, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    bool vec = ((reinterpret_cast<uintptr_t>(x) | (norm ? 0 : reinterpret_cast<uintptr_t>(y))) & 15u) == 0;
    if (norm) return vec ? launch_pass1_v<true, true>(x, x, n, A, B, prm, st)
                         : launch_pass1_v<true, false>(x, x, n, A, B, prm, st);
    return vec ? launch_pass1_v<false, true>(x, y, n, A, B, prm, st)
               : launch_pass1_v<false, false>(x, y, n, A, B, prm, st);
}

cudaError_t launch_score(const int64_t* A, const int64_t* B, int32_t* lut_bin, uint32_t* lut_p2, ScoreMeta* meta,
                         qdot_result* res, qdot_bin* bins, int64_t n_total, const qdot_config& cfg,
                         bool fuse, cudaStream_t st) {
    const size_t smem = sizeof(ScShared);
    static KernelDevCache cache;
    kernel_occupancy(k_score, SC_T, smem, cache);   // per-device shared-memory opt-in
    return launch_pdl(k_score, 1, SC_T, smem, st, A, B, lut_bin, lut_p2, meta, res, bins, n_total, cfg, fuse ? 1 : 0);
}

template <int CL>
static cudaError_t launch_small_cl(const double* x, const double* y, int64_t n, bool norm, int64_t* A, int64_t* B,
                                   int32_t* lut_bin, uint32_t* lut_p2, ScoreMeta* meta, qdot_result* res,
                                   qdot_bin* bins, const qdot_config& cfg, cudaStream_t st, bool vec) {
    auto kern = norm ? (vec ? k_small<true, true, CL> : k_small<true, false, CL>)
                     : (vec ? k_small<false, true, CL> : k_small<false, false, CL>);
    static KernelDevCache cache[4];
    const size_t smem = sizeof(SmShared);
    const int d = current_device();
    KernelDevCache& c = cache[(norm ? 2 : 0) + (vec ? 1 : 0)];
    if (!c.occ[d]) {        // per-device attributes: shared-memory opt-in, 16-CTA clusters
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess && CL > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        c.occ[d] = 1;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(CL);
    lc.blockDim = dim3(SM_T);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, kern, x, norm ? x : y, n, A, B, lut_bin, lut_p2, meta, res, bins, cfg);
}

cudaError_t launch_small(const double* x, const double* y, int64_t n, bool norm, int64_t* A, int64_t* B,
                         int32_t* lut_bin, uint32_t* lut_p2, ScoreMeta* meta, qdot_result* res, qdot_bin* bins,
                         const qdot_config& cfg, cudaStream_t st) {
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | (norm ? 0 : reinterpret_cast<uintptr_t>(y))) & 15u) == 0;
    // the portable 8-CTA cluster up to SM_CL_SPLIT elements, 16 CTAs above
    return n <= SM_CL_SPLIT
        ? launch_small_cl<SM_CL_SMALL>(x, y, n, norm, A, B, lut_bin, lut_p2, meta, res, bins, cfg, st, vec)
        : launch_small_cl<SM_CL>(x, y, n, norm, A, B, lut_bin, lut_p2, meta, res, bins, cfg, st, vec);
}

int64_t small_max() { return SM_MAX; }

cudaError_t launch_begin(void* region, size_t bytes, cudaStream_t st) {
    const int64_t n16 = (int64_t)(bytes / 16);
    int64_t grid = (n16 + 255) / 256;
    if (grid > sm_count_cached()) grid = sm_count_cached();
    k_begin<<<(unsigned)(grid < 1 ? 1 : grid), 256, 0, st>>>(static_cast<ulonglong2*>(region), n16);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const int64_t* A, const int64_t* B, const uint32_t* lut_p2, const ScoreMeta* meta,
                            qdot_result* res, qdot_bin* bins, cudaStream_t st) {
    k_finalize<<<1, FN_T, 0, st>>>(A, B, lut_p2, meta, res, bins);
    return cudaGetLastError();
}

template <bool NORM, bool VEC>
static cudaError_t launch_pass2_t(const double* x, const double* y, int64_t n, const uint32_t* lut_p2,
                                  const ScoreMeta* meta, int64_t* B, const double2* list, const uint32_t* list_fill,
                                  const P2Fin& fin, cudaStream_t st) {
    auto kern = k_pass2<NORM, VEC>;
    const size_t smem = sizeof(P2Shared);
    static KernelDevCache cache;
    const int occ = kernel_occupancy(kern, P2_T, smem, cache);
    int64_t ntiles = (n + P2_TILE - 1) / P2_TILE;
    int64_t grid = (int64_t)sm_count_cached() * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    return launch_pdl(kern, (unsigned)grid, P2_T, smem, st, x, y, n, lut_p2, meta, B, list, list_fill, fin.A ? 1 : 0,
                      fin.A, fin.res, fin.bins);
}

cudaError_t launch_pass2(const double* x, const double* y, int64_t n, bool norm, const uint32_t* lut_p2,
                         const ScoreMeta* meta, int64_t* B, const double2* list, const uint32_t* list_fill,
                         const P2Fin& fin, cudaStream_t st) {
    if (n <= 0) return fin.A ? launch_finalize(fin.A, B, lut_p2, meta, fin.res, fin.bins, st) : cudaSuccess;
    bool vec = ((reinterpret_cast<uintptr_t>(x) | (norm ? 0 : reinterpret_cast<uintptr_t>(y))) & 15u) == 0;
    if (norm) return vec ? launch_pass2_t<true, true>(x, x, n, lut_p2, meta, B, list, list_fill, fin, st)
                         : launch_pass2_t<true, false>(x, x, n, lut_p2, meta, B, list, list_fill, fin, st);
    return vec ? launch_pass2_t<false, true>(x, y, n, lut_p2, meta, B, list, list_fill, fin, st)
               : launch_pass2_t<false, false>(x, y, n, lut_p2, meta, B, list, list_fill, fin, st);
}


// copy the result header and the first `nbins` bins into host-mapped memory,
// then bump the sequence word the host spins on (written last, after a
// system-scope fence)
__global__ void __launch_bounds__(256, 1)
k_publish(const unsigned char* __restrict__ block, int nbytes, unsigned char* __restrict__ host, uint32_t* dev_seq,
          volatile uint32_t* host_seq) {
    const uint4* src = reinterpret_cast<const uint4*>(block);
    uint4* dst = reinterpret_cast<uint4*>(host);
    for (int i = threadIdx.x; i < nbytes / 16; i += blockDim.x) dst[i] = src[i];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t sq = *dev_seq + 1;
        *dev_seq = sq;
        __threadfence_system();
        *host_seq = sq;
    }
}

cudaError_t launch_publish(const void* block, int nbytes, void* host_dev, uint32_t* dev_seq, uint32_t* host_seq_dev,
                           cudaStream_t st) {
    k_publish<<<1, 256, 0, st>>>(static_cast<const unsigned char*>(block), nbytes, static_cast<unsigned char*>(host_dev),
                                 dev_seq, host_seq_dev);
    return cudaGetLastError();
}

template <bool NORM, bool VEC, bool GEN>
static cudaError_t launch_batched_t(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld,
                                    const BParams& prm, double* values, int64_t* counts, int32_t* info,
                                    qdot_bin* bins, cudaStream_t st);
template <bool NORM, bool VEC>
static cudaError_t launch_batched_g(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld,
                                    const BParams& prm, double* values, int64_t* counts, int32_t* info,
                                    qdot_bin* bins, cudaStream_t st) {
    if (prm.strategy != QDOT_STRATEGY_EXACT)
        return launch_batched_t<NORM, VEC, true>(X, Y, rows, len, ld, prm, values, counts, info, bins, st);
    return launch_batched_t<NORM, VEC, false>(X, Y, rows, len, ld, prm, values, counts, info, bins, st);
}

cudaError_t launch_batched(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld, bool norm,
                           const qdot_config& cfg, double* values, int64_t* counts, int32_t* info, qdot_bin* bins,
                           cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    BParams prm;
    prm.epsilon = cfg.epsilon;
    prm.split = cfg.split;
    prm.input_mu = cfg.input_mu;
    prm.strategy = cfg.strategy;
    prm.norm = norm ? 1 : 0;
    prm.strategy_param = cfg.strategy_param;
    const bool vec = ((ld & 1) == 0) &&
                     ((reinterpret_cast<uintptr_t>(X) | (norm ? 0 : reinterpret_cast<uintptr_t>(Y))) & 15u) == 0;
    if (norm) return vec ? launch_batched_g<true, true>(X, X, rows, len, ld, prm, values, counts, info, bins, st)
                         : launch_batched_g<true, false>(X, X, rows, len, ld, prm, values, counts, info, bins, st);
    return vec ? launch_batched_g<false, true>(X, Y, rows, len, ld, prm, values, counts, info, bins, st)
               : launch_batched_g<false, false>(X, Y, rows, len, ld, prm, values, counts, info, bins, st);
}

template <bool NORM, bool VEC, bool GEN>
static cudaError_t launch_batched_t(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld,
                                    const BParams& prm, double* values, int64_t* counts, int32_t* info,
                                    qdot_bin* bins, cudaStream_t st) {
    auto kern = k_batched<NORM, VEC, GEN>;
    static KernelDevCache cache;
    const int occ = kernel_occupancy(kern, B_WARPS * 32, 0, cache);
    int64_t grid = (rows + B_WARPS - 1) / B_WARPS;
    int64_t cap = (int64_t)sm_count_cached() * occ;
    if (grid > cap) grid = cap;
    kern<<<(unsigned)grid, B_WARPS * 32, 0, st>>>(X, Y, rows, len, ld, prm, values, counts, info, bins);
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

#ifdef QDOT_SCORE_PROFILE
extern "C" int qdot_b200_score_prof(long long* out) {
    return (int)cudaMemcpyFromSymbol(out, qd::g_sc_prof, sizeof(long long) * 16);
}
#endif
