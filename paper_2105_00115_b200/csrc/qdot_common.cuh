// qdot_common.cuh -- constants, workspace layout and exact-arithmetic helpers
// shared by the sm_100a kernels and the host side of the C ABI.
//
// Number formats used throughout:
//  * key     = exponent sum e = flexp(x) + flexp(y) offset by +2148 into [0, 4195)
//              (floatbits.py:17-32, 82; sum range floatbits.py:10-14).
//  * D(e)    = sum over elements with key e of fl(x*y) / 2^qd(e), an exact
//              integer, qd(e) = max(e - 52, -1074): every fl(x*y) of such an
//              element is an integer multiple of 2^qd(e) with |k| <= 2^54.
//  * S0/H0   = exact-binning (u == e) SINGLE / HALF products of the scaled
//              mantissas (emulate.py:137-146), integers in units of 2^-23 / 2^-10.
//  * P2(e)   = scaled SINGLE / HALF products for bins with upper u > e, in
//              units of 2^qs(e,u), qs = max(e - u - mu, 1 - bias - mu).
// All partials are integers, so every reduction (threads, CTAs, ranks) is
// exact and order independent.
#pragma once

#include <cstdint>
#include <cstring>
#include <cmath>

#include "../../include/qdot_b200.h"

#ifdef __CUDACC__
#define QD_HD __host__ __device__ __forceinline__
#else
#define QD_HD inline
#endif

namespace qd {

#ifdef __CUDACC__
// ---- per-device launch facts ------------------------------------------------
// Function attributes (the dynamic shared-memory opt-in), occupancy and the SM
// count belong to a device context, so every cache of them is indexed by the
// current device: one process may drive several GPUs.
constexpr int MAX_DEVICES = 64;

inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return (d >= 0 && d < MAX_DEVICES) ? d : 0;
}

inline int device_sm_count() {
    static int sms[MAX_DEVICES] = {};
    const int d = current_device();
    if (!sms[d]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        sms[d] = v > 0 ? v : 148;
    }
    return sms[d];
}

// occupancy of `kern` at (threads, smem) on the current device; the first use
// on a device also opts the kernel into `smem` bytes of dynamic shared memory
struct KernelDevCache {
    int occ[MAX_DEVICES] = {};
};

template <typename K>
inline int kernel_occupancy(K kern, int threads, size_t smem, KernelDevCache& c) {
    const int d = current_device();
    if (!c.occ[d]) {
        if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem);
        c.occ[d] = o > 0 ? o : 1;
    }
    return c.occ[d];
}
#endif

constexpr int KEYS = QDOT_KEYS;
constexpr int KOFF = QDOT_KEY_OFFSET;

// ---- workspace layout (int64 words unless noted) ---------------------------
constexpr int64_t A_CNT = 0;            // counts[KEYS]
constexpr int64_t A_ZERO = KEYS;        // zero-product count
constexpr int64_t A_NONFINITE = KEYS + 1;
constexpr int64_t A_FULLCTAS = KEYS + 2;  // pass-1 CTAs that ran the full-variant loop (diagnostic)
constexpr int64_t A_LEANCTAS = KEYS + 3;  // pass-1 CTAs that ran the lean loop (diagnostic)
constexpr int64_t A_LISTOVF = KEYS + 4;   // ranks whose cold-element list overflowed
constexpr int64_t A_HOT = 4224;         // [KEYS]: elements of the key accumulated by a lean
                                        // private window (exact HALF/SINGLE variants absent)
constexpr int64_t A_PRIV = 8448;        // [KEYS]: elements of the key accumulated by any private
                                        // window (absent from the cold-element list)
constexpr int64_t A_SMALL = 12664;      // k_small's outcome: 1 finished the call, 2 handed it to k_score
                                        // (0 after begin: the multi-CTA pipeline)
constexpr int64_t A_LEN = 12672;        // padded

constexpr int64_t B_D0 = 0;             // DOUBLE limbs, weights 2^0, 2^32, 2^64, 2^96
constexpr int64_t B_D1 = 1 * (int64_t)KEYS;
constexpr int64_t B_D2 = 2 * (int64_t)KEYS;
constexpr int64_t B_D3 = 3 * (int64_t)KEYS;
constexpr int64_t B_S0 = 4 * (int64_t)KEYS;
constexpr int64_t B_H0 = 5 * (int64_t)KEYS;
constexpr int64_t B_P2 = 6 * (int64_t)KEYS;
constexpr int64_t B_INFP = 7 * (int64_t)KEYS;  // +inf DOUBLE products (overflow)
constexpr int64_t B_INFN = 8 * (int64_t)KEYS;  // -inf DOUBLE products
constexpr int64_t B_LEN = 37760;        // >= 9*KEYS, padded

// pass-2 descriptor per key (int32): 0 = nothing to do in pass 2
//   bit 31: needed; bit 16: HALF (else SINGLE); bits 0..15: delta = u - e clamped to 255
constexpr uint32_t P2_NEED = 0x80000000u;
constexpr uint32_t P2_HALF = 0x00010000u;
constexpr int P2_DELTA_MAX = 255;

// pass-1 parameters (what the per-CTA lean/full decision needs)
struct P1Params {
    double epsilon;
    int64_t n_total;
    int32_t input_mu;
    int32_t mode;            // 0 auto, 1 force lean, 2 force full variants
    double2* list;           // cold-element list: LIST_SLOTS slots of LIST_PER_SLOT entries,
    uint32_t* list_fill;     // slot b filled by pass-1 CTA b (fill kept across launches)
    int32_t collect;         // fill the list (ranged / split strategies: pass 2 may need it)
    int32_t per_bin;         // exact strategy with SplitMode.PER_BIN: eps_eff = eps / n_bins
};

struct ScoreMeta {         // written by the score kernel, read by pass2 / finalize
    int32_t status;
    int32_t n_bins;
    int32_t e_min, e_max;   // exponent sums (not keys)
    int32_t early;
    int32_t need_p2;
    int32_t degenerate;
    int32_t input_mu;
    int32_t done;            // finalize already ran (fused into score: no pass 2 needed)
    int32_t pad_;
    int64_t nnz;
    int64_t zero;
    int64_t n_total;
    double eps_eff;
};

constexpr int64_t BYTES_A = A_LEN * 8;
constexpr int64_t BYTES_B = B_LEN * 8;
constexpr int64_t OFF_A = 0;
constexpr int64_t OFF_B = OFF_A + BYTES_A;
constexpr int64_t OFF_LOCAL = OFF_B + BYTES_B;                   // rank-local counters (zeroed by begin)
constexpr int64_t LIST_SLOTS = 1024;                             // one list slot per pass-1 CTA index
constexpr int64_t BYTES_LOCAL = LIST_SLOTS * 4 + 64;             // uint32 fill per slot, then phase stamps
constexpr int64_t OFF_LUT_BIN = OFF_LOCAL + BYTES_LOCAL;         // int32[KEYS]
constexpr int64_t OFF_LUT_P2 = OFF_LUT_BIN + 4224 * 4;           // uint32[KEYS]
constexpr int64_t OFF_META = OFF_LUT_P2 + 4224 * 4;              // ScoreMeta
constexpr int64_t OFF_RESULT = OFF_META + 256;                   // qdot_result
constexpr int64_t OFF_BINS = OFF_RESULT + 256;                   // qdot_bin[KEYS + 1]
constexpr int64_t BYTES_BINS = (int64_t)sizeof(qdot_bin) * (KEYS + 1);
#ifdef __CUDACC__
// device timestamps of the phases (ns, %globaltimer) in the rank-local area,
// located from the region-A pointer every kernel receives: [0] pass 1 start,
// [1] score done (select = [1]-[0]), finalize end - [1] = compute
__device__ __forceinline__ unsigned long long* ws_stamps(const int64_t* A) {
    return reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(const_cast<int64_t*>(A)) - OFF_A + OFF_LOCAL + LIST_SLOTS * 4);
}
// cp.async.bulk.prefetch.L2 needs a 16-byte aligned address (and size); a
// view of a vector may be only 8-byte aligned, so prefetch from the 16-byte
// granule holding p (inside the same allocation).  A hint: the 8 bytes this
// drops at the end of the range do not matter.
__device__ __forceinline__ const void* bulk_aligned(const void* p) {
    return reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(p) & ~static_cast<uintptr_t>(15));
}

// programmatic dependent launch (the kernels of one call are launched with
// programmatic stream serialization): a kernel may start while its
// predecessor drains, and waits here before touching the workspace
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// cold-element list: (x, y) of every element pass 1 did not accumulate in a
// private window, so that pass 2 (when it is needed only for such keys) reads
// this list instead of streaming both vectors again
constexpr int64_t LIST_CAP = 1 << 22;                             // entries (64 MiB)
constexpr int64_t LIST_PER_SLOT = LIST_CAP / LIST_SLOTS;
constexpr int64_t OFF_LIST = ((OFF_BINS + BYTES_BINS + 255) / 256) * 256;
constexpr int64_t WS_BYTES = OFF_LIST + LIST_CAP * 16;

static_assert(sizeof(ScoreMeta) <= 256, "meta");
static_assert(sizeof(qdot_result) <= 256, "result");
static_assert(sizeof(qdot_bin) == 56, "bin layout");

struct WsPtrs {
    int64_t* a;
    int64_t* b;
    uint32_t* list_fill;              // OFF_LOCAL: fill of each CTA slot
    double2* list;
    int32_t* lut_bin;
    uint32_t* lut_p2;
    ScoreMeta* meta;
    qdot_result* result;
    qdot_bin* bins;
};

inline WsPtrs ws_ptrs(void* ws) {
    char* p = static_cast<char*>(ws);
    WsPtrs w;
    w.a = reinterpret_cast<int64_t*>(p + OFF_A);
    w.b = reinterpret_cast<int64_t*>(p + OFF_B);
    w.list_fill = reinterpret_cast<uint32_t*>(p + OFF_LOCAL);
    w.list = reinterpret_cast<double2*>(p + OFF_LIST);
    w.lut_bin = reinterpret_cast<int32_t*>(p + OFF_LUT_BIN);
    w.lut_p2 = reinterpret_cast<uint32_t*>(p + OFF_LUT_P2);
    w.meta = reinterpret_cast<ScoreMeta*>(p + OFF_META);
    w.result = reinterpret_cast<qdot_result*>(p + OFF_RESULT);
    w.bins = reinterpret_cast<qdot_bin*>(p + OFF_BINS);
    return w;
}

// ---- bit helpers -------------------------------------------------------------
QD_HD uint64_t dbits(double v) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(v);
#else
    uint64_t b; std::memcpy(&b, &v, 8); return b;
#endif
}
QD_HD double bitsd(uint64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double v; std::memcpy(&v, &b, 8); return v;
#endif
}
QD_HD int clz64(uint64_t v) {
#ifdef __CUDA_ARCH__
    return __clzll((long long)v);
#else
    return v ? __builtin_clzll(v) : 64;
#endif
}

// floor(log2|x|) of a nonzero finite double from its bits (floatbits.py:17-27):
// exponent field - 1023, subnormals via the leading mantissa bit.
QD_HD int flexp_bits(uint64_t b) {
    int f = (int)((b >> 52) & 0x7FF);
    if (f) return f - 1023;
    uint64_t m = b & ((1ull << 52) - 1);
    return (63 - clz64(m)) - 1074;
}

// |x| * 2^-flexp(x) in [1, 2) as raw double bits (exact), x nonzero finite
QD_HD uint64_t mant_bits(uint64_t b) {
    int f = (int)((b >> 52) & 0x7FF);
    uint64_t m = b & ((1ull << 52) - 1);
    if (!f) {                      // subnormal: normalise the leading 1 to bit 52
        int sh = clz64(m) - 11;
        m = (m << sh) & ((1ull << 52) - 1);
    }
    return m | (1023ull << 52);
}

// DOUBLE quantum exponent of key e (see header comment)
QD_HD int qd_double(int e) { return e - 52 > -1074 ? e - 52 : -1074; }

// fl(x*y) (finite) as an exact integer multiple of 2^qd(e); sign applied
QD_HD int64_t double_units(uint64_t pb, int e) {
    int f = (int)((pb >> 52) & 0x7FF);
    uint64_t m = pb & ((1ull << 52) - 1);
    if (f) m |= 1ull << 52; else f = 1;
    int sh = (f - 1075) - qd_double(e);    // 0..2 (product exponent - key)
    int64_t k = (int64_t)(m << sh);
    return (pb >> 63) ? -k : k;
}

// ---- exact rounding -----------------------------------------------------------
// m * 2^qq for a nonzero m < 2^54 whose value is exactly representable with
// exponent <= 1023 (qq >= -1074): built from bits, no libm
QD_HD double exact_scale(uint64_t m, int qq) {
    const int tm = 63 - clz64(m);
    const int E = tm + qq;                          // exponent of the leading bit
    if (E >= -1022) {
        const uint64_t frac = tm <= 52 ? (m << (52 - tm)) : (m >> (tm - 52));
        return bitsd(((uint64_t)(E + 1023) << 52) | (frac & ((1ull << 52) - 1)));
    }
    return bitsd(m << (qq + 1074));                 // subnormal: exact since qq >= -1074
}

// 2^k as a double (0 below 2^-1074, inf above 2^1023), exact
QD_HD double pow2d(int k) {
    if (k >= -1022) return k > 1023 ? bitsd(0x7FF0000000000000ull) : bitsd((uint64_t)(k + 1023) << 52);
    return k >= -1074 ? bitsd(1ull << (k + 1074)) : 0.0;
}

// Round (top + frac) * 2^q, frac in [0,1) nonzero iff `sticky`, to the binary
// format with `mu` fraction bits and minimum normal exponent `emin`, maximum
// exponent `emax`: round-to-nearest-even, gradual underflow, overflow -> inf.
// Returns the rounded value as a double (exact for fp64 and fp32 targets).
QD_HD double round_scaled(uint64_t top, int q, bool sticky, bool neg, int mu, int emin, int emax,
                          int* overflow) {
    if (top == 0) return neg ? -0.0 : 0.0;   // (sticky without top never occurs)
    int t = 63 - clz64(top);
    int T = t + q;                              // exponent of the leading bit
    int qq = (T - mu > emin - mu) ? T - mu : emin - mu;   // quantum exponent
    int sh = qq - q;
    uint64_t m;
    if (sh <= 0) {
        m = top << (-sh);                        // t <= mu here: exact
    } else {
        bool rb, st = sticky;
        if (sh >= 65) { m = 0; rb = false; st = st || top; }
        else if (sh == 64) { m = 0; rb = (top >> 63) & 1; st = st || (top & ~(1ull << 63)); }
        else {
            m = top >> sh;
            rb = (top >> (sh - 1)) & 1;
            st = st || (top & ((1ull << (sh - 1)) - 1));
        }
        if (rb && (st || (m & 1))) m += 1;
    }
    if (m == 0) return neg ? -0.0 : 0.0;
    int tm = 63 - clz64(m);
    if (tm + qq > emax) { if (overflow) *overflow = 1; return neg ? -INFINITY : INFINITY; }
    double r = exact_scale(m, qq);               // exact: m <= 2^(mu+1), qq >= -1074
    return neg ? -r : r;
}

// math.ldexp(acc, u) semantics: correctly rounded, range error flagged
QD_HD double ldexp_rn(double acc, int64_t u, int* overflow) {
    if (acc == 0.0 || !(acc - acc == 0.0)) return acc;   // zero / inf / nan unchanged
    uint64_t b = dbits(acc);
    bool neg = b >> 63;
    int f = (int)((b >> 52) & 0x7FF);
    if (f && u > -1022 && u < 1023 && f + (int)u > 0 && f + (int)u < 0x7FF)   // normal in, normal out: exact
        return bitsd(b + ((uint64_t)(int64_t)u << 52));
    uint64_t m = b & ((1ull << 52) - 1);
    int q;
    if (f) { m |= 1ull << 52; q = f - 1075; } else { q = -1074; }
    if (u > 4000) u = 4000;
    if (u < -4000) u = -4000;
    return round_scaled(m, q + (int)u, false, neg, 52, -1022, 1023, overflow);
}

// Exact signed big integer in 32-bit digits held in int64 (carry-save), value
// = sum d[i] * 2^(32 i + lsb).  Used by finalize for per-bin exact sums.
template <int ND>
struct BigSum {
    int64_t d[ND];
    int lsb;
    int nd;
    QD_HD void init(int lsb_, int ndigits) {
        lsb = lsb_;
        nd = ndigits > ND ? ND : ndigits;
        for (int i = 0; i < nd; ++i) d[i] = 0;
    }
    // add v * 2^exp, v a signed 128-bit integer, exp >= lsb
    QD_HD void add(__int128 v, int exp) {
        if (v == 0) return;
        bool neg = v < 0;
        unsigned __int128 a = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
        int pos = exp - lsb;
        int di = pos >> 5, off = pos & 31;
        // a << off spans <= 160 bits -> 5 digits
        unsigned __int128 lo = a << off;
        uint64_t hi = off ? (uint64_t)(a >> (128 - off)) : 0;
        uint32_t dg[5] = {(uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)(lo >> 64),
                          (uint32_t)(lo >> 96), (uint32_t)hi};
        for (int k = 0; k < 5; ++k) {
            if (di + k >= nd) break;
            if (neg) d[di + k] -= dg[k]; else d[di + k] += dg[k];
        }
    }
    // normalise, then round to the target format
    QD_HD double round(int mu, int emin, int emax, int* overflow) {
        int64_t carry = 0;
        for (int i = 0; i < nd; ++i) {
            int64_t v = d[i] + carry;
            int64_t lo = v & 0xFFFFFFFFll;
            carry = (v - lo) >> 32;
            d[i] = lo;
        }
        bool neg = carry < 0;   // value = digits + carry * 2^(32 nd)
        if (neg) {              // two's complement negate digits (carry == -1)
            int64_t br = 0;
            for (int i = 0; i < nd; ++i) {
                int64_t v = -d[i] - br;
                if (v < 0) { v += 4294967296ll; br = 1; } else br = 0;
                d[i] = v;
            }
        }
        int top = nd - 1;
        while (top >= 0 && d[top] == 0) --top;
        if (top < 0) return 0.0;
        // gather the top 64 bits below and including the leading digit
        uint64_t t64 = 0;
        int got = 0, i = top;
        bool sticky = false;
        // leading digit bit length
        uint32_t lead = (uint32_t)d[top];
        int lb = 32 - (lead ? clz64((uint64_t)lead) - 32 : 32);
        t64 = lead;
        got = lb;
        --i;
        while (i >= 0 && got + 32 <= 64) { t64 = (t64 << 32) | (uint32_t)d[i]; got += 32; --i; }
        int q;
        if (i >= 0 && got < 64) {          // take the high (64-got) bits of the next digit
            int take = 64 - got;
            uint32_t nx = (uint32_t)d[i];
            t64 = (t64 << take) | (nx >> (32 - take));
            sticky = (nx & ((1u << (32 - take)) - 1)) != 0;
            q = lsb + 32 * i + (32 - take);
            --i;
        } else {
            q = lsb + 32 * (i + 1);
        }
        while (i >= 0 && !sticky) { sticky = d[i] != 0; --i; }
        return round_scaled(t64, q, sticky, neg, mu, emin, emax, overflow);
    }
};

}  // namespace qd
