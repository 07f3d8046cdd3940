// qdot_batched.cuh -- many independent qdots (rows of X, Y), one warp per row,
// one HBM pass (included into namespace qd of qdot_kernels.cu).
//
// Per row the warp runs the whole pipeline of kernel.qdot (kernel.py:179-240)
// for ExactBinning (and early termination at input_mu 52): exponent sums,
// exact per-key DOUBLE / SINGLE / HALF partial sums (the "full" variants of
// pass 1, accumulated in per-lane shared-memory slots for a 16-key window
// and per-warp 32-bit limb tables for a 64-key window), then per-row scoring
// (scoring.py:96-216), per-bin rounding (emulate.py:116-154) and the Neumaier
// fold (emulate.py:157-163) -- all inside the warp, no inter-row traffic.
//
// Ranged and split strategies (b_row_general): the partition, scores and
// precisions come from the same per-key counts; a HALF / SINGLE bin whose
// upper exceeds a member's key needs that member's partition-dependent
// product, so the warp streams its row a second time for those keys only
// (k_pass2's scaled_units), then rounds every bin like bin_value.
//
// Rows the kernel cannot finish exactly are flagged BS_GENERAL and re-run by
// the host through the single-vector pipeline: keys spread beyond the 64-key
// window, DOUBLE product overflow, early termination below input_mu 52, rows
// longer than 2^16.
//
// Per-row bin tables (optional, qdot_b200_batched_bins): row r's bins at
// bins[r * QDOT_BATCH_MAX_BINS ...], info[4r] of them.

constexpr int BW = 16;            // per-lane private window (keys)
constexpr int BCW = 64;           // per-warp limb table window (keys)
constexpr int B_WARPS = 4;        // warps (rows in flight) per CTA
constexpr int B_MAXLEN = 1 << 16;
constexpr int B_CHUNK = 512;      // L2 prefetch granule (elements; 4 warp iterations)
constexpr int B_PFC = 2;          // prefetch distance in chunks

// per-row status bits (qdot_b200_batched info[4*r + 3])
constexpr int BS_NONFINITE = 1;
constexpr int BS_OVERFLOW = 2;
constexpr int BS_EPS = 4;
constexpr int BS_GENERAL = 8;
constexpr int BS_EARLY = 16;
constexpr int BS_HALF_ORDER = 32;

struct __align__(16) BWarp {
    ulonglong2 priv[BW * 32];     // per-lane {D units, packed S|H|count}
    uint32_t c[8][BCW];           // limb table: cnt, d0, d1, d2, d3 (signed), s0, s1 (signed), h (signed)
};

struct BParams {
    double epsilon;
    int32_t split;
    int32_t input_mu;
    int32_t strategy;
    int32_t norm;
    int64_t strategy_param;      // ranged width / split levels
};
static_assert(BCW == QDOT_BATCH_MAX_BINS, "bin table stride");

// flush per-lane slots into the warp's limb table (all lanes, warp-synchronous).
// Transposed: lane L sums key (L & 15) over lanes 16*(L >> 4) .. +15 (staggered
// so each 8-lane LDS.128 phase touches 8 distinct bank groups), one xor-16
// shuffle merges the halves, lanes 0..15 update the table.
__device__ __forceinline__ void b_flush(BWarp& W, int lane, int base_rel) {
    __syncwarp();
    const int k = lane & 15, half = lane >> 4;
    uint64_t dlo = 0;
    int64_t dhi = 0;
    long long s = 0, h = 0, c = 0;
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
        const int idx = k * 32 + half * 16 + ((j + k) & 15);
        const ulonglong2 v = W.priv[idx];
        W.priv[idx] = make_ulonglong2(0ull, 0ull);
        const int64_t d = (int64_t)v.x;
        const uint64_t nl = dlo + (uint64_t)d;
        dhi += (d >> 63) + (nl < dlo ? 1 : 0);
        dlo = nl;
        const long long w = (long long)v.y;
        const long long cc = w & 0xFF;
        const long long w1 = (w - cc) >> 8;
        const long long hh = ((w1 & 0x1FFFFF) ^ 0x100000) - 0x100000;
        c += cc;
        h += hh;
        s += (w1 - hh) >> 21;
    }
    {
        const uint64_t olo = __shfl_xor_sync(0xffffffffu, dlo, 16);
        const int64_t ohi = __shfl_xor_sync(0xffffffffu, dhi, 16);
        const uint64_t nl = dlo + olo;
        dhi += ohi + (nl < dlo ? 1 : 0);
        dlo = nl;
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        h += __shfl_xor_sync(0xffffffffu, h, 16);
        c += __shfl_xor_sync(0xffffffffu, c, 16);
    }
    if (half == 0 && c) {
        const int t = base_rel + k;                          // index into the limb table
        const __int128 D = ((__int128)dhi << 64) | (__int128)dlo;
        W.c[0][t] += (uint32_t)c;
        W.c[1][t] += (uint32_t)((uint64_t)D & 0x3FFFu);
        W.c[2][t] += (uint32_t)(((uint64_t)D >> 14) & 0x3FFFu);
        W.c[3][t] += (uint32_t)(((uint64_t)D >> 28) & 0x3FFFu);
        W.c[4][t] += (uint32_t)(int32_t)(long long)(D >> 42);
        W.c[5][t] += (uint32_t)(s & 0x3FFF);
        W.c[6][t] += (uint32_t)(int32_t)(s >> 14);
        W.c[7][t] += (uint32_t)(int32_t)h;
    }
    __syncwarp();
}

// key - cbase from key - base: base = KOFF - 2046 - kbias
__device__ __forceinline__ int kbias_to_c(int kbias, int cbase) { return (KOFF - 2046 - kbias) - cbase; }

__device__ __forceinline__ void b_cold_add(BWarp& W, int c, int64_t kd, int32_t ks, int32_t kh) {
    uint64_t u = (uint64_t)kd;
    atomicAdd(&W.c[0][c], 1u);
    atomicAdd(&W.c[1][c], (uint32_t)(u & 0x3FFFu));
    atomicAdd(&W.c[2][c], (uint32_t)((u >> 14) & 0x3FFFu));
    atomicAdd(&W.c[3][c], (uint32_t)((u >> 28) & 0x3FFFu));
    atomicAdd(&W.c[4][c], (uint32_t)(int32_t)(kd >> 42));
    atomicAdd(&W.c[5][c], (uint32_t)ks & 0x3FFFu);
    atomicAdd(&W.c[6][c], (uint32_t)(ks >> 14));
    atomicAdd(&W.c[7][c], (uint32_t)kh);
}

// everything outside the private window: limb-table keys, zero / subnormal /
// non-finite / extreme elements (limb table or a row flag).  Returns the row
// status bits it raises, plus 256 for a zero product.
__device__ __noinline__ uint32_t b_cold(BWarp& W, int cbase, double xv, double yv) {
    uint64_t bx = dbits(xv), by = dbits(yv);
    if (((bx >> 52) & 0x7FF) == 0x7FF || ((by >> 52) & 0x7FF) == 0x7FF) return BS_NONFINITE;
    if (xv == 0.0 || yv == 0.0) return 256u;
    int e = flexp_bits(bx) + flexp_bits(by);
    int c = e + KOFF - cbase;
    if ((unsigned)c >= (unsigned)BCW) return BS_GENERAL;
    uint64_t pb = dbits(__dmul_rn(xv, yv));
    if (((pb >> 52) & 0x7FF) == 0x7FF) return BS_GENERAL;     // DOUBLE overflow: rare, general path
    int64_t kd = double_units(pb, e);
    int32_t ks, kh;
    exact_variants(bitsd(mant_bits(bx)), bitsd(mant_bits(by)), ks, kh);
    int32_t sg = -(int32_t)((bx ^ by) >> 63);
    ks = (ks ^ sg) - sg;
    kh = (kh ^ sg) - sg;
    b_cold_add(W, c, kd, ks, kh);
    return 0u;
}

// NE elements of one lane.  Private-window keys (both factors normal; the
// window lies in e in [-971, 1021], so 2^(52-e) is representable and fl(x*y)
// normal) update their slot inline; the rest go through b_cold (rare).
// ok: element in range (ragged tail).
template <int NE>
__device__ __forceinline__ void b_elems(BWarp& W, ulonglong2* __restrict__ my, int kbias, int cbase,
                                        const double (&xv)[NE], const double (&yv)[NE], const bool (&ok)[NE],
                                        uint32_t& zc, uint32_t& st) {
#pragma unroll
    for (int j = 0; j < NE; ++j) {
        const uint32_t hx = (uint32_t)(dbits(xv[j]) >> 32), hy = (uint32_t)(dbits(yv[j]) >> 32);
        const uint32_t fx = (hx >> 20) & 0x7FFu, fy = (hy >> 20) & 0x7FFu;
        const uint32_t esum = fx + fy;
        const int rel = (int)esum + kbias;
        if (((unsigned)rel < (unsigned)BW) & (max(fx - 1u, fy - 1u) < 0x7FEu) & ok[j]) {
            const double scale = __hiloint2double((int)((3121u - esum) << 20), 0);   // 2^(52-e)
            const long long kd = __double2ll_rn(__dmul_rn(__dmul_rn(xv[j], yv[j]), scale));
            const uint64_t bx = dbits(xv[j]), by = dbits(yv[j]);
            int32_t ks, kh;
            exact_variants_signed(bitsd((bx & 0x800FFFFFFFFFFFFFull) | 0x3FF0000000000000ull),
                                  bitsd((by & 0x800FFFFFFFFFFFFFull) | 0x3FF0000000000000ull), ks, kh);
            ulonglong2* slot = my + rel * 32;
            ulonglong2 v = *slot;
            v.x += (unsigned long long)kd;
            v.y += (unsigned long long)(((long long)ks << 29) + ((long long)kh << 8) + 1);
            *slot = v;
        } else if (ok[j]) {
            const uint32_t r = b_cold(W, cbase, xv[j], yv[j]);
            zc += r >> 8;
            st |= r & 0xFFu;
        }
    }
}

// exact sum of D over the row's present keys, rounded to double (early-terminated DOUBLE bin)
__device__ double b_early_double(const int64_t* kd_lo, int kmin_c, int kmax_c, int cbase, int lane,
                                 __int128 D0, __int128 D1, uint32_t cnt0, uint32_t cnt1, int* ovf) {
    BigSum<104> acc;
    int lsb = qd_double(cbase + kmin_c - KOFF);
    acc.init(lsb, (qd_double(cbase + kmax_c - KOFF) - lsb + 160) / 32 + 2);
    for (int j = kmin_c; j <= kmax_c; ++j) {
        const int src = j & 31;
        const bool hi = j >= 32;
        uint64_t lo64 = __shfl_sync(0xffffffffu, (uint64_t)(hi ? D1 : D0), src);
        int64_t hi64 = __shfl_sync(0xffffffffu, (int64_t)((hi ? D1 : D0) >> 64), src);
        uint32_t c = __shfl_sync(0xffffffffu, hi ? cnt1 : cnt0, src);
        if (c) acc.add(((__int128)hi64 << 64) | (__int128)lo64, qd_double(cbase + j - KOFF));
    }
    (void)kd_lo; (void)lane;
    return acc.round(52, -1022, 1023, ovf);
}

// bulk L2 prefetch of chunk `c` (B_CHUNK elements) of the warp's stream, which
// continues into its next row; lane 0 only
__device__ __forceinline__ void b_prefetch(const double* xr, const double* yr, const double* xn, const double* yn,
                                           int64_t len, int64_t c, bool norm) {
    int64_t e0 = c * B_CHUNK;
    const double *px = xr, *py = yr;
    if (e0 >= len) {
        if (!xn) return;
        e0 -= len;
        px = xn;
        py = yn;
    }
    if (e0 + B_CHUNK > len) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(bulk_aligned(px + e0)), "r"(B_CHUNK * 8) : "memory");
    if (!norm) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(bulk_aligned(py + e0)), "r"(B_CHUNK * 8) : "memory");
}

// warp iteration: 128 elements, lane holds {2l, 2l+1, 64+2l, 65+2l}
template <bool NORM>
__device__ __forceinline__ void b_load_full(const double* __restrict__ xr, const double* __restrict__ yr, int64_t i0,
                                            int lane, double (&xa)[4], double (&ya)[4]) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        const int64_t i = i0 + v * 64 + 2 * lane;
        const double2 a = __ldcs(reinterpret_cast<const double2*>(xr + i));
        xa[2 * v] = a.x;
        xa[2 * v + 1] = a.y;
        if (NORM) {
            ya[2 * v] = a.x;
            ya[2 * v + 1] = a.y;
        } else {
            const double2 b = __ldcs(reinterpret_cast<const double2*>(yr + i));
            ya[2 * v] = b.x;
            ya[2 * v + 1] = b.y;
        }
    }
}

template <bool NORM>
__device__ __forceinline__ void b_load_tail(const double* __restrict__ xr, const double* __restrict__ yr, int64_t i0,
                                            int64_t len, int lane, double (&xa)[4], double (&ya)[4], bool (&ok)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t i = i0 + (j >> 1) * 64 + 2 * lane + (j & 1);
        ok[j] = i < len;
        xa[j] = ok[j] ? xr[i] : 0.0;
        ya[j] = ok[j] ? (NORM ? xa[j] : yr[i]) : 0.0;
    }
}

// the per-key totals of the warp's limb table (table index j, key cbase + j)
__device__ __forceinline__ __int128 bw_d(const BWarp& W, int j) {
    return (__int128)W.c[1][j] + ((__int128)W.c[2][j] << 14) + ((__int128)W.c[3][j] << 28) +
           ((__int128)(int32_t)W.c[4][j] << 42);
}
__device__ __forceinline__ long long bw_s(const BWarp& W, int j) {
    return (long long)W.c[5][j] + ((long long)(int32_t)W.c[6][j] << 14);
}
__device__ __forceinline__ long long bw_h(const BWarp& W, int j) { return (long long)(int32_t)W.c[7][j]; }

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// scratch of b_row_general inside the warp's private slots (zero between rows;
// re-zeroed before it returns)
constexpr int BG_SLOTS = 16;      // pass-2 keys with per-lane accumulators (more: shared atomics)
struct BGenScratch {
    uint32_t off[BCW + 4];        // exclusive prefix of the key counts, off[BCW] = nnz
    uint32_t info[BCW];           // pass-2 descriptor per key (P2_NEED | P2_HALF | delta)
    uint32_t p2lo[BCW], p2hi[BCW];// pass-2 units of keys without a slot: lo 14 bits + signed rest
    long long p2[BCW];            // pass-2 sum per key
    double val[BCW];              // bin values in bin order (for the fold)
    int slot[BCW];                // per-lane accumulator slot of a pass-2 key, or -1
    long long pacc[BG_SLOTS][32]; // per-lane pass-2 accumulators (no atomics)
};
static_assert(sizeof(BGenScratch) <= sizeof(ulonglong2) * BW * 32, "scratch fits the private slots");

// Ranged / split rows (not early-terminated) of one warp: k_score's partition
// (binning.py:202-274), scores / precisions (scoring.py:96-123, 181-199),
// k_pass2's scaled products (emulate.py:137-147) for keys below their bin's
// upper, bin_value's rounding (emulate.py:116-154) and the Neumaier fold
// (emulate.py:157-163).  Lane-local results: cnt_p (summed by the caller).
template <bool NORM>
__device__ __noinline__ void b_row_general(BWarp& W, int lane, int cbase, const BParams& prm,
                                           const double* __restrict__ xr, const double* __restrict__ yr,
                                           int64_t len, uint32_t& st, double& value, long long (&cnt_p)[4],
                                           int& nbins, int& emin, int& emax, qdot_bin* __restrict__ bout) {
    BGenScratch& G = *reinterpret_cast<BGenScratch*>(W.priv);
    const uint32_t c0 = W.c[0][lane], c1 = W.c[0][lane + 32];
    const unsigned long long P = (unsigned long long)__ballot_sync(0xffffffffu, c0 != 0) |
                                 ((unsigned long long)__ballot_sync(0xffffffffu, c1 != 0) << 32);
    value = 0.0;
    nbins = 0;
    if (!P) return;
    const int jmin = __ffsll((long long)P) - 1, jmax = 63 - __clzll((long long)P);
    emin = cbase + jmin - KOFF;
    emax = cbase + jmax - KOFF;
    {
        const uint32_t i0 = warp_incl_scan(c0, lane), i1 = warp_incl_scan(c1, lane);
        const uint32_t t0 = __shfl_sync(0xffffffffu, i0, 31);
        G.off[lane] = i0 - c0;
        G.off[lane + 32] = t0 + i1 - c1;
        if (lane == 31) G.off[BCW] = t0 + i1;
        G.info[lane] = 0u;
        G.info[lane + 32] = 0u;
    }
    __syncwarp();
    const unsigned long long nnz = G.off[BCW];
    // ---- bin starts (binning.py:202-222 ranged, 224-274 split)
    unsigned long long S = 0ull;
    if (prm.strategy == QDOT_STRATEGY_RANGED) {
        const long long w = prm.strategy_param;
        bool f[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            f[h] = false;
            if ((P >> j) & 1ull) {
                const int gs = jmin + (int)(((long long)(j - jmin) / w) * w);
                const unsigned long long below = ((1ull << j) - 1ull) ^ ((1ull << gs) - 1ull);   // keys [gs, j)
                f[h] = (P & below) == 0ull;
            }
        }
        S = (unsigned long long)__ballot_sync(0xffffffffu, f[0]) |
            ((unsigned long long)__ballot_sync(0xffffffffu, f[1]) << 32);
    } else {
        long long levels = prm.strategy_param;
        const unsigned long long t = nnz > 1 ? nnz - 1 : 0;
        const int bl = t ? 64 - __clzll((long long)t) : 0;
        if (levels > bl) levels = bl;                                              // binning.py:235
        uint32_t nx[2] = {0u, 0u};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            if (!((P >> j) & 1ull)) continue;
            const unsigned long long a = G.off[j], b = a + W.c[0][j];
            if (b < nnz && split_boundary_in(nnz, (int)levels, a, b)) {             // cut after key j
                const unsigned long long rest = j == 63 ? 0ull : (P & ~((2ull << j) - 1ull));
                const int nj = __ffsll((long long)rest) - 1;                         // next present key
                nx[nj >> 5] |= 1u << (nj & 31);
            }
        }
        S = (unsigned long long)__reduce_or_sync(0xffffffffu, nx[0]) |
            ((unsigned long long)__reduce_or_sync(0xffffffffu, nx[1]) << 32) | (1ull << jmin);
    }
    nbins = __popcll(S);
    const double eps_eff = prm.split == 1 ? __ddiv_rn(prm.epsilon, (double)nbins) : prm.epsilon;   // scoring.py:192
    bool okf = true;
    const long long fl = floor_log2_d(eps_eff, &okf);
    if (!okf) { st |= BS_EPS; return; }
    // ---- per bin (the lane owning its first key): interval, score, precision; pass-2 keys
    long long bu[2] = {0, 0}, bl_[2] = {0, 0}, bm[2] = {0, 0}, bsc[2] = {0, 0};
    int bpr[2] = {0, 0}, bidx[2] = {-1, -1}, bl2[2] = {0, 0};
    bool need = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (!((S >> j) & 1ull)) continue;
        const int b = __popcll(S & ((1ull << j) - 1ull));
        const unsigned long long rest = j == 63 ? 0ull : (S & ~((2ull << j) - 1ull));
        const int nf = rest ? __ffsll((long long)rest) - 1 : BCW;
        const unsigned long long upto = nf == BCW ? ~0ull : ((1ull << nf) - 1ull);
        const int l = 63 - __clzll((long long)(P & upto));
        const long long M = (long long)(G.off[nf] - G.off[j]);
        long long upper, lower;
        if (prm.strategy == QDOT_STRATEGY_RANGED) {
            const long long w = prm.strategy_param;
            const long long g = (long long)(j - jmin) / w;
            upper = (long long)emin + (g + 1) * w - 1;
            lower = upper - w;
        } else {
            upper = cbase + l - KOFF;
            const unsigned long long pb = P & ((1ull << j) - 1ull);
            lower = pb ? (long long)(cbase + (63 - __clzll((long long)pb)) - KOFF) : (long long)emin - 1;
        }
        const unsigned long long mm = (unsigned long long)(M - 1);
        const long long score = (mm ? 64 - __clzll((long long)mm) : 0) + upper - emax - fl + 1;   // bin_score
        const int pr = precision_of(score, prm.input_mu);
        bu[h] = upper; bl_[h] = lower; bm[h] = M; bsc[h] = score; bpr[h] = pr; bidx[h] = b; bl2[h] = l;
        if (pr == QDOT_HALF || pr == QDOT_SINGLE) {
            for (int k = j; k <= l; ++k) {
                if (!((P >> k) & 1ull)) continue;
                const long long d = upper - (long long)(cbase + k - KOFF);
                if (d > 0) {
                    G.info[k] = P2_NEED | (pr == QDOT_HALF ? P2_HALF : 0u) | (uint32_t)(d > P2_DELTA_MAX ? P2_DELTA_MAX : d);
                    need = true;
                }
            }
        }
    }
    // ---- second pass over the row for the keys whose products depend on the partition
    if (__any_sync(0xffffffffu, need)) {
        const unsigned long long N = (unsigned long long)__ballot_sync(0xffffffffu, (G.info[lane] & P2_NEED) != 0) |
                                     ((unsigned long long)__ballot_sync(0xffffffffu, (G.info[lane + 32] & P2_NEED) != 0) << 32);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            const int sl = ((N >> j) & 1ull) ? __popcll(N & ((1ull << j) - 1ull)) : -1;
            G.slot[j] = sl < BG_SLOTS ? sl : -1;
            G.p2lo[j] = 0u;
            G.p2hi[j] = 0u;
        }
        for (int sl = 0; sl < BG_SLOTS; ++sl) G.pacc[sl][lane] = 0;
        __syncwarp();
        auto elem = [&](double a, double bb) {
            if (a == 0.0 || bb == 0.0) return;
            const uint64_t bx = dbits(a), by = dbits(bb);
            const int j = flexp_bits(bx) + flexp_bits(by) + KOFF - cbase;
            if ((unsigned)j >= (unsigned)BCW) return;
            const uint32_t inf = G.info[j];
            if (!(inf & P2_NEED)) return;
            long long k = scaled_units(bitsd(mant_bits(bx)), bitsd(mant_bits(by)), inf);
            if ((bx ^ by) >> 63) k = -k;
            const int sl = G.slot[j];
            if (sl >= 0) {
                G.pacc[sl][lane] += k;
            } else {
                atomicAdd(&G.p2lo[j], (uint32_t)((uint64_t)k & 0x3FFFu));
                atomicAdd(&G.p2hi[j], (uint32_t)(int32_t)(k >> 14));
            }
        };
        const bool vec = ((reinterpret_cast<uintptr_t>(xr) | reinterpret_cast<uintptr_t>(yr)) & 15u) == 0;
        int64_t i0 = 0;
        if (vec) {
            for (; i0 + 64 <= len; i0 += 64) {
                const double2 a = __ldcs(reinterpret_cast<const double2*>(xr + i0) + lane);
                const double2 bb = NORM ? a : __ldcs(reinterpret_cast<const double2*>(yr + i0) + lane);
                elem(a.x, bb.x);
                elem(a.y, bb.y);
            }
        }
        for (int64_t i = i0 + lane; i < len; i += 32) {
            const double a = xr[i];
            elem(a, NORM ? a : yr[i]);
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = lane + 32 * h;
            long long v = (long long)G.p2lo[j] + ((long long)(int32_t)G.p2hi[j] << 14);
            const int sl = G.slot[j];
            if (sl >= 0)
                for (int l2 = 0; l2 < 32; ++l2) v += G.pacc[sl][l2];
            G.p2[j] = v;
        }
        __syncwarp();
    }
    // ---- bin values (bin_value, emulate.py:116-154)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (bidx[h] < 0) continue;
        const int f = lane + 32 * h, l = bl2[h];
        const long long u = bu[h];
        const int pr = bpr[h];
        double val = 0.0;
        int o = 0, hf = 0;
        if (pr == QDOT_DOUBLE) {
            if (f == l) val = round_i128(bw_d(W, f), qd_double(cbase + f - KOFF), 52, -1022, 1023, &o);
            else {
                BigSum<104> acc;
                const int lsb = qd_double(cbase + f - KOFF);
                acc.init(lsb, (qd_double(cbase + l - KOFF) - lsb + 160) / 32 + 2);
                for (int k = f; k <= l; ++k)
                    if ((P >> k) & 1ull) acc.add(bw_d(W, k), qd_double(cbase + k - KOFF));
                val = acc.round(52, -1022, 1023, &o);
            }
        } else if (pr != QDOT_PERFORATE) {
            const bool half = pr == QDOT_HALF;
            const int mu = half ? 10 : 23;
            const int qmin_fmt = half ? -24 : -149;
            auto qs_of = [&](int k) {
                const long long d = u - (long long)(cbase + k - KOFF);
                const int dd = d > P2_DELTA_MAX ? P2_DELTA_MAX : (int)d;
                return -dd - mu > qmin_fmt ? -dd - mu : qmin_fmt;
            };
            auto keyval = [&](int k) -> long long {
                if (G.info[k] & P2_NEED) return G.p2[k];
                return half ? bw_h(W, k) : bw_s(W, k);
            };
            const int lsb = qs_of(f);
            double mass = 0.0;
            BigSum<16> acc;
            acc.init(lsb, (qs_of(l) - lsb + 128) / 32 + 2);
            for (int k = f; k <= l; ++k) {
                if (!((P >> k) & 1ull)) continue;
                const long long d = u - (long long)(cbase + k - KOFF);
                acc.add((__int128)keyval(k), qs_of(k));
                mass += (double)W.c[0][k] * pow2d(2 - (int)(d > 2000 ? 2000 : d));
            }
            const double a = half ? acc.round(23, -126, 127, &o) : acc.round(52, -1022, 1023, &o);
            val = ldexp_rn(a, u, &o);                                                  // emulate.py:154
            if (half && mass > pow2d(24 + lsb)) hf = 1;
        }
        if (o) st |= BS_OVERFLOW;
        if (hf) st |= BS_HALF_ORDER;
        G.val[bidx[h]] = val;
        cnt_p[pr] += bm[h];
        if (bout) {
            qdot_bin ob;
            ob.lower = bl_[h]; ob.upper = u; ob.cardinality = bm[h]; ob.score = bsc[h]; ob.precision = pr;
            ob.first_key = cbase + f; ob.last_key = cbase + l; ob.flags = hf; ob.value = val;
            bout[bidx[h]] = ob;
        }
    }
    __syncwarp();
    // ---- Neumaier fold in ascending upper order (emulate.py:157-163)
    if (lane == 0) {
        double sm = 0.0, c = 0.0;
        neumaier_fold(G.val, nbins, sm, c);
        value = (sm - sm == 0.0) ? __dadd_rn(sm, c) : sm;
    }
    value = __shfl_sync(0xffffffffu, value, 0);
    __syncwarp();
    // leave the private slots zero for the next row
    for (int i = lane; i < (int)(sizeof(BGenScratch) / 16); i += 32) W.priv[i] = make_ulonglong2(0ull, 0ull);
    __syncwarp();
}

// GEN: ranged / split strategies (b_row_general); the exact-binning
// instantiation keeps its epilogue in registers
template <bool NORM, bool VEC, bool GEN>
__global__ void __launch_bounds__(B_WARPS * 32, 5)
k_batched(const double* __restrict__ X, const double* __restrict__ Y, int64_t rows, int64_t len, int64_t ld,
          BParams prm, double* __restrict__ values, int64_t* __restrict__ counts, int32_t* __restrict__ info,
          qdot_bin* __restrict__ bins) {
    __shared__ BWarp warps[B_WARPS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    BWarp& W = warps[wid];
    ulonglong2* __restrict__ my = W.priv + lane;
    const int64_t rstride = (int64_t)gridDim.x * B_WARPS;
    const int64_t nfull = VEC ? len / 128 : 0;            // full warp iterations per row
    for (int i = lane; i < BW * 32; i += 32) W.priv[i] = make_ulonglong2(0ull, 0ull);   // flushes keep it zero
    for (int64_t r = (int64_t)blockIdx.x * B_WARPS + wid; r < rows; r += rstride) {
        const double* xr = X + r * ld;
        const double* yr = NORM ? xr : Y + r * ld;
        const bool has_next = r + rstride < rows;
        const double* xn = has_next ? X + (r + rstride) * ld : nullptr;
        const double* yn = has_next ? (NORM ? xn : Y + (r + rstride) * ld) : nullptr;
        uint32_t st = 0, zc = 0;
        if (len > B_MAXLEN) st |= BS_GENERAL;
        // ---- first warp iteration: doubles as the sample that places the windows
        double xa[4], ya[4], xb[4], yb[4];
        bool ok0[4] = {true, true, true, true};
        if (nfull > 0) b_load_full<NORM>(xr, yr, 0, lane, xa, ya);
        else b_load_tail<NORM>(xr, yr, 0, len, lane, xa, ya, ok0);
        if (VEC && lane == 0 && r == (int64_t)blockIdx.x * B_WARPS + wid)   // first row: warm its stream
            for (int64_t c = 1; c < B_PFC; ++c) b_prefetch(xr, yr, xn, yn, len, c, NORM);
        int base;
        {
            int k4[4];
            int kmx = -1;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t fx = (uint32_t)(dbits(xa[j]) >> 52) & 0x7FFu, fy = (uint32_t)(dbits(ya[j]) >> 52) & 0x7FFu;
                k4[j] = (ok0[j] && fx - 1u < 0x7FEu && fy - 1u < 0x7FEu) ? (int)(fx + fy) - 2046 + KOFF : -10000;
                kmx = max(kmx, k4[j]);
            }
            kmx = __reduce_max_sync(0xffffffffu, kmx);
            // window [kmax - W + 2, kmax + 1] when it holds >= 3/4 of the sample
            int cand = kmx - BW + 2, cov = 0, nv = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                cov += __popc(__ballot_sync(0xffffffffu, (unsigned)(k4[j] - cand) < (unsigned)BW));
                nv += __popc(__ballot_sync(0xffffffffu, k4[j] >= 0));
            }
            if (nv == 0) {
                base = KOFF - BW / 2;
            } else if (4 * cov >= 3 * nv) {
                base = cand;
            } else {
                // among windows anchored at sampled keys, the one covering most samples
                long long bestkey = -1;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int cd = k4[h] - BW + 3;
                    int cv = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        for (int src = 0; src < 32; ++src) {
                            const int a = __shfl_sync(0xffffffffu, k4[j], src);
                            cv += (unsigned)(a - cd) < (unsigned)BW;
                        }
                    const long long key = k4[h] < 0 ? -1ll : (((long long)cv << 32) | (uint32_t)(0x7FFFFFFF - cd));
                    bestkey = key > bestkey ? key : bestkey;
                }
                for (int o = 16; o; o >>= 1) {
                    const long long t = __shfl_xor_sync(0xffffffffu, bestkey, o);
                    bestkey = t > bestkey ? t : bestkey;
                }
                base = (int)(0x7FFFFFFF - (uint32_t)(bestkey & 0xFFFFFFFF));
            }
            base = base < KOFF - 971 ? KOFF - 971 : (base > KOFF + 1021 - BW + 1 ? KOFF + 1021 - BW + 1 : base);
        }
        int cbase = base - (BCW - BW) / 2;
        cbase = cbase < 0 ? 0 : (cbase + BCW > KEYS ? KEYS - BCW : cbase);
        const int kbias = KOFF - 2046 - base;
        // ---- clear this warp's limb table (the private slots are zero after every flush)
        for (int i = lane; i < 8 * BCW; i += 32) (&W.c[0][0])[i] = 0u;
        __syncwarp();
        // ---- stream the row (one HBM pass); trip counts are warp-uniform (b_flush is collective)
        if (!(st & BS_GENERAL)) {
            int since = 0;
            auto step = [&](int64_t it, double (&cx)[4], double (&cy)[4], double (&nx)[4], double (&ny)[4]) {
                if (it + 1 < nfull) b_load_full<NORM>(xr, yr, (it + 1) * 128, lane, nx, ny);
                if (lane == 0 && (it & (B_CHUNK / 128 - 1)) == 0)
                    b_prefetch(xr, yr, xn, yn, len, it / (B_CHUNK / 128) + B_PFC, NORM);
                const bool all[4] = {true, true, true, true};
                b_elems<4>(W, my, kbias, cbase, cx, cy, all, zc, st);
                if (++since == 62) { b_flush(W, lane, base - cbase); since = 0; }   // <= 248 elements per lane
            };
            int64_t it = 0;
            for (; it + 2 <= nfull; it += 2) {
                step(it, xa, ya, xb, yb);
                step(it + 1, xb, yb, xa, ya);
            }
            if (it < nfull) { step(it, xa, ya, xb, yb); ++it; }
            // ragged tail (and every iteration when the rows are not 16-byte aligned)
            for (int64_t i0 = it * 128; i0 < len; i0 += 128) {
                bool ok[4];
                b_load_tail<NORM>(xr, yr, i0, len, lane, xa, ya, ok);
                b_elems<4>(W, my, kbias, cbase, xa, ya, ok, zc, st);
                if (++since == 62) { b_flush(W, lane, base - cbase); since = 0; }
            }
            b_flush(W, lane, base - cbase);
        }
        // row-wide status and zero count
        st = __reduce_or_sync(0xffffffffu, st);          // row length <= B_MAXLEN: 32-bit counts
        zc = __reduce_add_sync(0xffffffffu, zc);
        double value = 0.0;
        long long cnt_p[4] = {0, 0, 0, 0};
        int nbins = 0, emin = 0, emax = 0;
        qdot_bin* __restrict__ bout = bins ? bins + r * (int64_t)BCW : nullptr;
        if (!(st & (BS_GENERAL | BS_NONFINITE))) {
            // ---- per-key totals: lane owns table entries j = lane and lane + 32
            uint32_t cnt[2];
            __int128 D[2];
            long long S[2], H[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = lane + 32 * h;
                cnt[h] = W.c[0][j];
                D[h] = (__int128)W.c[1][j] + ((__int128)W.c[2][j] << 14) + ((__int128)W.c[3][j] << 28) +
                       ((__int128)(int32_t)W.c[4][j] << 42);
                S[h] = (long long)W.c[5][j] + ((long long)(int32_t)W.c[6][j] << 14);
                H[h] = (long long)(int32_t)W.c[7][j];
            }
            const unsigned pres0 = __ballot_sync(0xffffffffu, cnt[0] != 0);
            const unsigned pres1 = __ballot_sync(0xffffffffu, cnt[1] != 0);
            nbins = __popc(pres0) + __popc(pres1);
            if (nbins) {
                const int jmin = pres0 ? __ffs(pres0) - 1 : 32 + __ffs(pres1) - 1;
                const int jmax = pres1 ? 63 - __clz(pres1) : 31 - __clz(pres0);
                emin = cbase + jmin - KOFF;
                emax = cbase + jmax - KOFF;
                bool okf = true;
                const long long fle = flexp_bits(dbits(prm.epsilon));
                const int mu_hat = prm.input_mu == 52 ? 23 : (prm.input_mu == 23 ? 10 : 0);
                const bool early = (long long)(emax - emin) <= (-fle - mu_hat);           // scoring.py:126-136
                long long nnz = 0;
#pragma unroll
                for (int h = 0; h < 2; ++h) nnz += cnt[h];
                nnz = __reduce_add_sync(0xffffffffu, (unsigned)nnz);
                if (early) {
                    st |= BS_EARLY;
                    if (prm.input_mu != 52) st |= BS_GENERAL;
                    nbins = 1;
                    // single bin (e_min-1, e_max], M = nnz, eps_eff = eps (one bin)
                    long long mm = nnz - 1;
                    long long sc = (mm ? 64 - __clzll(mm) : 0) + 0 - fle + 1;
                    int pr = precision_of(sc, prm.input_mu);
                    int ovf = 0;
                    if (pr == QDOT_DOUBLE) value = b_early_double(nullptr, jmin, jmax, cbase, lane, D[0], D[1], cnt[0], cnt[1], &ovf);
                    else if (pr != QDOT_PERFORATE) st |= BS_GENERAL;
                    if (ovf) st |= BS_OVERFLOW;
                    if (lane == 0) cnt_p[pr] += nnz;
                    if (bout && lane == 0) {
                        qdot_bin ob;
                        ob.lower = emin - 1; ob.upper = emax; ob.cardinality = nnz; ob.score = sc; ob.precision = pr;
                        ob.first_key = cbase + jmin; ob.last_key = cbase + jmax; ob.flags = 0; ob.value = value;
                        bout[0] = ob;
                    }
                } else if (GEN) {
                    b_row_general<NORM>(W, lane, cbase, prm, xr, yr, len, st, value, cnt_p, nbins, emin, emax, bout);
                } else {
                    double eps_eff = prm.split == 1 ? __ddiv_rn(prm.epsilon, (double)nbins) : prm.epsilon;
                    long long fl = floor_log2_d(eps_eff, &okf);
                    if (!okf) st |= BS_EPS;
                    double val[2] = {0.0, 0.0};
                    int pr[2] = {0, 0};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (!cnt[h]) continue;
                        const int e = cbase + lane + 32 * h - KOFF;
                        unsigned long long mm = cnt[h] - 1;
                        long long sc = (mm ? 64 - __clzll((long long)mm) : 0) + e - emax - fl + 1;   // bin_score
                        pr[h] = precision_of(sc, prm.input_mu);
                        int ovf = 0, hf = 0;
                        if (pr[h] == QDOT_DOUBLE) {
                            val[h] = round_i128(D[h], qd_double(e), 52, -1022, 1023, &ovf);
                        } else if (pr[h] == QDOT_SINGLE) {
                            val[h] = ldexp_rn(round_i128((__int128)S[h], -23, 52, -1022, 1023, &ovf), e, &ovf);
                        } else if (pr[h] == QDOT_HALF) {
                            val[h] = ldexp_rn(round_i128((__int128)H[h], -10, 23, -126, 127, &ovf), e, &ovf);
                            if ((double)cnt[h] * 4.0 > 16384.0) { st |= BS_HALF_ORDER; hf = 1; }
                        }
                        if (ovf) st |= BS_OVERFLOW;
                        cnt_p[pr[h]] += cnt[h];
                        if (bout) {
                            const int b = h ? __popc(pres0) + __popc(pres1 & ((1u << lane) - 1u))
                                            : __popc(pres0 & ((1u << lane) - 1u));
                            qdot_bin ob;
                            ob.lower = e - 1; ob.upper = e; ob.cardinality = cnt[h]; ob.score = sc; ob.precision = pr[h];
                            ob.first_key = e + KOFF; ob.last_key = e + KOFF; ob.flags = hf; ob.value = val[h];
                            bout[b] = ob;
                        }
                    }
                    // Neumaier fold over bins in ascending key order (emulate.py:157-163)
                    double s = 0.0, c = 0.0;
                    unsigned rem0 = pres0, rem1 = pres1;
                    while (rem0 | rem1) {
                        int j;
                        if (rem0) { j = __ffs(rem0) - 1; rem0 &= rem0 - 1; }
                        else { j = 32 + __ffs(rem1) - 1; rem1 &= rem1 - 1; }
                        const double v = __shfl_sync(0xffffffffu, j < 32 ? val[0] : val[1], j & 31);
                        const double t = __dadd_rn(s, v);
                        if (fabs(s) >= fabs(v)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), v));
                        else c = __dadd_rn(c, __dadd_rn(__dsub_rn(v, t), s));
                        s = t;
                    }
                    value = (s - s == 0.0) ? __dadd_rn(s, c) : s;
                }
                for (int p = 0; p < 4; ++p) cnt_p[p] = __reduce_add_sync(0xffffffffu, (unsigned)cnt_p[p]);
                st = __reduce_or_sync(0xffffffffu, st);
            }
        }
        if (lane == 0) {
            values[r] = value;
            counts[4 * r + 0] = cnt_p[0] + zc;
            counts[4 * r + 1] = cnt_p[1];
            counts[4 * r + 2] = cnt_p[2];
            counts[4 * r + 3] = cnt_p[3];
            info[4 * r + 0] = nbins;
            info[4 * r + 1] = emin;
            info[4 * r + 2] = emax;
            info[4 * r + 3] = (int32_t)st;
        }
        __syncwarp();
    }
}
