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
// Rows the fast kernel cannot finish exactly are flagged BS_GENERAL and
// re-run by the host through the single-vector pipeline: strategies other
// than exact binning, keys spread beyond the 64-key window, DOUBLE product
// overflow, early termination below input_mu 52, rows longer than 2^16.

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
};

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

template <bool NORM, bool VEC>
__global__ void __launch_bounds__(B_WARPS * 32, 5)
k_batched(const double* __restrict__ X, const double* __restrict__ Y, int64_t rows, int64_t len, int64_t ld,
          BParams prm, double* __restrict__ values, int64_t* __restrict__ counts, int32_t* __restrict__ info) {
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
        if (prm.strategy != QDOT_STRATEGY_EXACT || len > B_MAXLEN) st |= BS_GENERAL;
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
                    if (lane == 0) cnt_p[pr] += nnz;
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
                        int ovf = 0;
                        if (pr[h] == QDOT_DOUBLE) {
                            val[h] = round_i128(D[h], qd_double(e), 52, -1022, 1023, &ovf);
                        } else if (pr[h] == QDOT_SINGLE) {
                            val[h] = ldexp_rn(round_i128((__int128)S[h], -23, 52, -1022, 1023, &ovf), e, &ovf);
                        } else if (pr[h] == QDOT_HALF) {
                            val[h] = ldexp_rn(round_i128((__int128)H[h], -10, 23, -126, 127, &ovf), e, &ovf);
                            if ((double)cnt[h] * 4.0 > 16384.0) st |= BS_HALF_ORDER;
                        }
                        if (ovf) st |= BS_OVERFLOW;
                        cnt_p[pr[h]] += cnt[h];
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
