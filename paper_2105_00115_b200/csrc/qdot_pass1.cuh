// qdot_pass1.cuh -- the streaming pass (included into namespace qd of qdot_kernels.cu).
//
// Per element (floatbits.py:57-93 + emulate.py:133-146):
//   key  = flexp(x) + flexp(y) + 2148        exponent-sum histogram bin
//   D    = fl(x*y) in units of 2^(e-52)      exact DOUBLE partial  (|D| <= 2^54)
//   S0,H0 = exact-binning SINGLE / HALF products of the scaled mantissas in
//          units of 2^-23 / 2^-10 (always for cold keys, for private-window
//          keys only in full mode)
//
// Accumulation (all integer, order independent):
//   * private window: P1_W consecutive keys chosen per CTA from a sample of
//     its first tile; one 16-byte slot per (key, thread) in shared memory,
//     updated with plain LDS/STS (no atomics);
//   * cold window: P1_CW keys around it, per-CTA shared-memory tables of
//     32-bit limbs updated with native 32-bit shared atomics;
//   * anything else: global atomics.
//   Both shared tables are flushed (private -> per-CTA totals, cold -> global)
//   every <= 255 (full) / 511 (lean) elements per thread, which bounds every
//   per-thread int64 and per-CTA 32-bit limb sum.
//   Zero / subnormal / non-finite / extreme-exponent elements take a separate
//   non-inlined path.
//
// Lean vs full: the exact HALF/SINGLE variants are only needed for bins that
// end up HALF or SINGLE.  Each CTA predicts from its sample (estimated bin
// cardinality, exponent distance to the sampled maximum, epsilon) whether any
// key of its private window can score in [0, 23); if not it runs the lean
// loop (count + DOUBLE units only) and flags its window keys in A[A_HOT].
// The score kernel sends flagged keys that did become HALF/SINGLE to pass 2,
// so the prediction only affects speed, never results.

// The file is included twice (qdot_kernels.cu): with the defaults below for
// x . y, and inside namespace p1n with QDOT_P1_W 11 / QDOT_P1_WW 17 /
// QDOT_P1_MINB 4 for norm mode -- 11 private slots per thread instead of 16
// fit four CTAs per SM instead of three (norm mode is latency-bound, x . y
// HBM-bound).
#ifndef QDOT_P1_W
#define QDOT_P1_W 16
#endif
#ifndef QDOT_P1_WW
#define QDOT_P1_WW 24
#endif
#ifndef QDOT_P1_MINB
#define QDOT_P1_MINB 3
#endif
constexpr int P1_T = 256;                    // threads per CTA
constexpr int P1_W = QDOT_P1_W;              // keys with per-thread private slots
constexpr int P1_WW = QDOT_P1_WW;            // wide lean window: {D int64, count u16} per (key, thread)
static_assert(P1_WW * P1_T * 10 <= P1_W * P1_T * 16, "wide layout fits the private slots");
static_assert(4224 * 8 + 4224 * 2 <= P1_W * P1_T * 16, "sampling scratch fits the private slots");
constexpr int P1_CW = 128;                   // keys with per-CTA 32-bit limb tables
// private window keys keep e in [-971, 1021]: fl(x*y) normal and finite and
// 2^(52-e) representable
constexpr int P1_SAFE_LO = KOFF - 971;
constexpr int P1_SAFE_HI = KOFF + 1021 - P1_W + 1;
constexpr int P1_SAFE_HI_W = KOFF + 1021 - P1_WW + 1;

struct __align__(16) P1Shared {
    ulonglong2 priv[P1_W * P1_T];            // lean: {D, count}; full: {D, packed S|H|count}
    __int128 t_d[P1_WW];                     // CTA totals of the private window
    long long t_s[P1_WW], t_h[P1_WW], t_c[P1_WW];
    // cold window, 32-bit limbs: D = d0 + d1 2^14 + d2 2^28 + d3 2^42 (d3 signed),
    // S = s0 + s1 2^14 (s1 signed), H (signed)
    uint32_t c_cnt[P1_CW], c_d0[P1_CW], c_d1[P1_CW], c_d2[P1_CW], c_d3[P1_CW];
    uint32_t c_s0[P1_CW], c_s1[P1_CW], c_h[P1_CW];
    unsigned long long red[2 * (P1_T / 32)];
    double2 q[P1_T / 32][32];                // per-warp queue of cold elements (queue mode)
    int base;                                // first key of the private window
    int cbase;                               // first key of the cold window
    double2* list;                           // this CTA's slot of the cold-element list
    uint32_t list_fill;                      // entries used in it (across launches)
    int collect;                             // append cold elements to the list
    int full;                                // this CTA runs the full-variant loop
    int wide;                                // lean loop over the 24-key window
    int queue;                               // this CTA compacts cold elements through the warp queue
    int kmax;                                // largest sampled key
    int norm_lean;                           // x . x: exponent-indexed lean loop (window keys base + 2r)
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

// the same from SIGNED mantissas (|mx|, |my| in [1,2), signs of x and y): the
// format products carry the sign (RNE is sign-symmetric) and one scaled
// float->int conversion yields the signed units -- no bit extraction, no
// separate sign fix
__device__ __forceinline__ void exact_variants_signed(double sx, double sy, int32_t& ks, int32_t& kh) {
    const float ps = __fmul_rn(__double2float_rn(sx), __double2float_rn(sy));          // |ps| in [1, 4]
    ks = __float2int_rn(__fmul_rn(ps, 8388608.0f));                                    // exact: units of 2^-23
    const float ph = __half2float(__hmul(__double2half(sx), __double2half(sy)));       // exact widening
    kh = __float2int_rn(__fmul_rn(ph, 1024.0f));                                       // units of 2^-10
}

// append (x, y) to this CTA's slot of the cold-element list (shared counter;
// no global atomics); an overfull slot is flagged when the CTA ends
__device__ __forceinline__ void p1_list_append(P1Shared& S, int64_t* __restrict__ A, double xv, double yv) {
    const uint32_t pos = atomicAdd(&S.list_fill, 1u);
    if (pos < (uint32_t)LIST_PER_SLOT) S.list[pos] = make_double2(xv, yv);
}

// cold key: variants from the mantissa bits (mbx, mby = raw bits of mx, my),
// then the per-CTA limb table or, outside it, global atomics; the element
// itself goes to the cold-element list for a possible pass 2
__device__ __forceinline__ void p1_cold(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B, int key,
                                        int64_t kd, uint64_t mbx, uint64_t mby, int32_t sg, double xv, double yv) {
    if (S.collect) p1_list_append(S, A, xv, yv);
    int32_t ks, kh;
    exact_variants(bitsd(mbx), bitsd(mby), ks, kh);
    ks = (ks ^ sg) - sg;
    kh = (kh ^ sg) - sg;
    int c = key - S.cbase;
    if ((unsigned)c < (unsigned)P1_CW) {
        uint64_t u = (uint64_t)kd;
        atomicAdd(&S.c_cnt[c], 1u);
        atomicAdd(&S.c_d0[c], (uint32_t)(u & 0x3FFFu));
        atomicAdd(&S.c_d1[c], (uint32_t)((u >> 14) & 0x3FFFu));
        atomicAdd(&S.c_d2[c], (uint32_t)((u >> 28) & 0x3FFFu));
        atomicAdd(&S.c_d3[c], (uint32_t)(int32_t)(kd >> 42));
        atomicAdd(&S.c_s0[c], (uint32_t)ks & 0x3FFFu);
        atomicAdd(&S.c_s1[c], (uint32_t)(ks >> 14));
        atomicAdd(&S.c_h[c], (uint32_t)kh);
    } else {
        push_key(A, B, key, 1ull, (__int128)kd, ks, kh);
    }
}

// zero / subnormal / non-finite / extreme-exponent elements
__device__ __noinline__ void p1_special(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B,
                                        double xv, double yv, uint32_t* zc, uint32_t* nf) {
    uint64_t bx = dbits(xv), by = dbits(yv);
    if (((bx >> 52) & 0x7FF) == 0x7FF || ((by >> 52) & 0x7FF) == 0x7FF) { (*nf)++; return; }
    if (xv == 0.0 || yv == 0.0) { (*zc)++; return; }                   // floatbits.py:74
    int e = flexp_bits(bx) + flexp_bits(by);
    int key = e + KOFF;
    uint64_t pb = dbits(__dmul_rn(xv, yv));
    int64_t kd = 0;
    if (((pb >> 52) & 0x7FF) == 0x7FF) {                               // DOUBLE product overflow
        atomicAdd(reinterpret_cast<unsigned long long*>(B + ((pb >> 63) ? B_INFN : B_INFP) + key), 1ull);
    } else {
        kd = double_units(pb, e);
    }
    p1_cold(S, A, B, key, kd, mant_bits(bx), mant_bits(by), -(int32_t)((bx ^ by) >> 63), xv, yv);
}

// one element.  Private-window elements (both factors normal, key in the
// window, which lies inside e in [-971, 1021]): fl(x*y) * 2^(52-e) is an exact
// integer in [2^52, 2^54] -> one conversion gives the signed DOUBLE units.
// QUEUE: elements outside the private window are not handled here; the
// return value flags them for the warp queue.
// WW == P1_WW: the wide lean layout (FULL is false): per (key, thread) an
// int64 DOUBLE sum in priv[0 .. 24*256) as long long and a u16 count after it.
template <bool FULL, bool QUEUE, int WW = P1_W>
__device__ __forceinline__ bool p1_elem(P1Shared& S, ulonglong2* __restrict__ my, int kbias,
                                        int64_t* __restrict__ A, int64_t* __restrict__ B, double xv, double yv,
                                        uint32_t* zc, uint32_t* nf) {
    const uint32_t hx = (uint32_t)(dbits(xv) >> 32), hy = (uint32_t)(dbits(yv) >> 32);
    const uint32_t fx = (hx >> 20) & 0x7FFu, fy = (hy >> 20) & 0x7FFu;
    const uint32_t esum = fx + fy;                                      // e + 2046
    const int rel = (int)esum + kbias;                                  // key - base
    const bool hot = (max(fx - 1u, fy - 1u) < 0x7FEu) & ((unsigned)rel < (unsigned)WW);
    if (WW == P1_WW && hot) {
        const double scale = __hiloint2double((int)((3121u - esum) << 20), 0);   // 2^(52-e)
        const long long kd = __double2ll_rn(__dmul_rn(__dmul_rn(xv, yv), scale));
        long long* wd = reinterpret_cast<long long*>(S.priv) + threadIdx.x;
        uint16_t* wc = reinterpret_cast<uint16_t*>(reinterpret_cast<long long*>(S.priv) + P1_WW * P1_T) + threadIdx.x;
        wd[rel * P1_T] += kd;
        wc[rel * P1_T] += 1;
    } else if (hot) {
        // DOUBLE (emulate.py:133): fl(x*y) in units of 2^(e-52)
        const double scale = __hiloint2double((int)((3121u - esum) << 20), 0);   // 2^(52-e)
        const long long kd = __double2ll_rn(__dmul_rn(__dmul_rn(xv, yv), scale));
        ulonglong2* slot = my + rel * P1_T;
        ulonglong2 v = *slot;
        v.x += (unsigned long long)kd;
        if (FULL) {
            const uint64_t bx = dbits(xv), by = dbits(yv);
            int32_t ks, kh;
            exact_variants_signed(bitsd((bx & 0x800FFFFFFFFFFFFFull) | 0x3FF0000000000000ull),
                                  bitsd((by & 0x800FFFFFFFFFFFFFull) | 0x3FF0000000000000ull), ks, kh);
            v.y += (unsigned long long)(((long long)ks << 29) + ((long long)kh << 8) + 1);
        } else {
            v.y = (unsigned long long)((uint32_t)v.y + 1u);   // count < 2^32 between flushes
        }
        *slot = v;
    } else if (QUEUE) {
        return true;
    } else if ((max(fx - 1u, fy - 1u) < 0x7FEu) & (esum - 1024u < 2044u)) {  // normal, e in [-1022, 1021]
        const uint64_t bx = dbits(xv), by = dbits(yv);
        const int e = (int)esum - 2046;
        const int64_t kd = double_units(dbits(__dmul_rn(xv, yv)), e);
        p1_cold(S, A, B, e + KOFF, kd, (bx & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull,
                (by & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull, (int32_t)(hx ^ hy) >> 31, xv, yv);
    } else {
        p1_special(S, A, B, xv, yv, zc, nf);
    }
    return false;
}

// an element outside the private window (also the queue drain)
__device__ __forceinline__ void p1_outside(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B,
                                           double xv, double yv, uint32_t* zc, uint32_t* nf) {
    const uint32_t hx = (uint32_t)(dbits(xv) >> 32), hy = (uint32_t)(dbits(yv) >> 32);
    const uint32_t fx = (hx >> 20) & 0x7FFu, fy = (hy >> 20) & 0x7FFu;
    const uint32_t esum = fx + fy;
    if ((max(fx - 1u, fy - 1u) < 0x7FEu) & (esum - 1024u < 2044u)) {
        const uint64_t bx = dbits(xv), by = dbits(yv);
        const int e = (int)esum - 2046;
        const int64_t kd = double_units(dbits(__dmul_rn(xv, yv)), e);
        p1_cold(S, A, B, e + KOFF, kd, (bx & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull,
                (by & 0xFFFFFFFFFFFFFull) | 0x3FF0000000000000ull, (int32_t)(hx ^ hy) >> 31, xv, yv);
    } else {
        p1_special(S, A, B, xv, yv, zc, nf);
    }
}

// process the warp's queued cold elements, one per lane (warp-collective)
__device__ __forceinline__ void p1_drain(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B, int warp,
                                         int lane, uint32_t& qn, uint32_t* zc, uint32_t* nf) {
    __syncwarp();
    if ((uint32_t)lane < qn) {
        const double2 e = S.q[warp][lane];
        p1_outside(S, A, B, e.x, e.y, zc, nf);
    }
    qn = 0;
    __syncwarp();
}

// append this slot's cold elements (flag c per lane) to the warp queue,
// draining whenever 32 entries would be exceeded (warp-collective)
__device__ __forceinline__ void p1_enqueue(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B, int warp,
                                           int lane, uint32_t& qn, bool c, double xv, double yv, uint32_t* zc,
                                           uint32_t* nf) {
    const unsigned m = __ballot_sync(0xffffffffu, c);
    if (m) {
        const uint32_t k = __popc(m);
        if (qn + k > 32) p1_drain(S, A, B, warp, lane, qn, zc, nf);
        if (c) S.q[warp][qn + __popc(m & ((1u << lane) - 1u))] = make_double2(xv, yv);
        qn += k;
    }
}

// reduce the private slots into the CTA totals, push the cold table to the
// global tables, clear both (all threads of the CTA)
template <bool FULL, int WW = P1_W>
__device__ __forceinline__ void p1_flush(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B, int tid) {
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = warp; r < WW; r += P1_T / 32) {
        uint64_t dlo = 0;
        int64_t dhi = 0;
        long long ss = 0, hs = 0, cs = 0;
        if (WW == P1_WW) {
            long long* wd = reinterpret_cast<long long*>(S.priv);
            uint16_t* wc = reinterpret_cast<uint16_t*>(wd + P1_WW * P1_T);
            for (int i = lane; i < P1_T; i += 32) {
                const int64_t d = wd[r * P1_T + i];
                wd[r * P1_T + i] = 0;
                const uint64_t nl = dlo + (uint64_t)d;
                dhi += (d >> 63) + (nl < dlo ? 1 : 0);
                dlo = nl;
                cs += wc[r * P1_T + i];
                wc[r * P1_T + i] = 0;
            }
        } else
        for (int i = lane; i < P1_T; i += 32) {
            ulonglong2 v = S.priv[r * P1_T + i];
            S.priv[r * P1_T + i] = make_ulonglong2(0ull, 0ull);
            int64_t d = (int64_t)v.x;
            uint64_t nl = dlo + (uint64_t)d;
            dhi += (d >> 63) + (nl < dlo ? 1 : 0);
            dlo = nl;
            if (FULL) {
                long long w = (long long)v.y;
                long long c = w & 0xFF;
                long long w1 = (w - c) >> 8;
                long long h = ((w1 & 0x1FFFFF) ^ 0x100000) - 0x100000;
                long long s = (w1 - h) >> 21;
                cs += c; hs += h; ss += s;
            } else {
                cs += (long long)(uint32_t)v.y;
            }
        }
        for (int o = 16; o; o >>= 1) {
            uint64_t olo = __shfl_xor_sync(0xffffffffu, dlo, o);
            int64_t ohi = __shfl_xor_sync(0xffffffffu, dhi, o);
            uint64_t nl = dlo + olo;
            dhi += ohi + (nl < dlo ? 1 : 0);
            dlo = nl;
            cs += __shfl_xor_sync(0xffffffffu, cs, o);
            if (FULL) {
                ss += __shfl_xor_sync(0xffffffffu, ss, o);
                hs += __shfl_xor_sync(0xffffffffu, hs, o);
            }
        }
        if (lane == 0) {
            S.t_d[r] += ((__int128)dhi << 64) | (__int128)dlo;
            S.t_s[r] += ss;
            S.t_h[r] += hs;
            S.t_c[r] += cs;
        }
    }
    for (int c = tid; c < P1_CW; c += P1_T) {
        uint32_t cnt = S.c_cnt[c];
        if (cnt) {
            __int128 d = (__int128)S.c_d0[c] + ((__int128)S.c_d1[c] << 14) + ((__int128)S.c_d2[c] << 28) +
                         ((__int128)(int32_t)S.c_d3[c] << 42);
            long long s = (long long)S.c_s0[c] + ((long long)(int32_t)S.c_s1[c] << 14);
            push_key(A, B, S.cbase + c, cnt, d, s, (long long)(int32_t)S.c_h[c]);
            S.c_cnt[c] = 0u; S.c_d0[c] = 0u; S.c_d1[c] = 0u; S.c_d2[c] = 0u; S.c_d3[c] = 0u;
            S.c_s0[c] = 0u; S.c_s1[c] = 0u; S.c_h[c] = 0u;
        }
    }
    __syncthreads();
}

template <bool NORM, bool VEC, int V>
__device__ __forceinline__ void p1_load(const double* __restrict__ x, const double* __restrict__ y,
                                        int64_t n, int64_t tile, int tid, double (&xv)[2 * V],
                                        double (&yv)[2 * V], bool& full) {
    constexpr int TILE = P1_T * 2 * V;
    const int64_t e0 = tile * TILE;
    full = e0 + TILE <= n;
    if (VEC && full) {
        const double2* x2 = reinterpret_cast<const double2*>(x + e0);
        const double2* y2 = reinterpret_cast<const double2*>(y + e0);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            double2 a = __ldcs(x2 + v * P1_T + tid);
            xv[2 * v] = a.x; xv[2 * v + 1] = a.y;
            if (!NORM) {
                double2 b = __ldcs(y2 + v * P1_T + tid);
                yv[2 * v] = b.x; yv[2 * v + 1] = b.y;
            }
        }
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
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
        for (int j = 0; j < 2 * V; ++j) yv[j] = xv[j];
    }
}

template <bool FULL, bool QUEUE, int V, int WW = P1_W>
__device__ __forceinline__ void p1_tile(P1Shared& S, ulonglong2* __restrict__ my, int kbias,
                                        int64_t* __restrict__ A, int64_t* __restrict__ B,
                                        const double (&xv)[2 * V], const double (&yv)[2 * V], int64_t e0,
                                        int64_t n, bool fulltile, int tid, uint32_t& qn, uint32_t* zc, uint32_t* nf) {
    if (fulltile) {
#pragma unroll
        for (int j = 0; j < 2 * V; ++j) {
            const bool c = p1_elem<FULL, QUEUE, WW>(S, my, kbias, A, B, xv[j], yv[j], zc, nf);
            if (QUEUE) p1_enqueue(S, A, B, tid >> 5, tid & 31, qn, c, xv[j], yv[j], zc, nf);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 2 * V; ++j) {
            bool c = false;
            if (e0 + 2 * ((int64_t)(j >> 1) * P1_T + tid) + (j & 1) < n)
                c = p1_elem<FULL, QUEUE, WW>(S, my, kbias, A, B, xv[j], yv[j], zc, nf);
            if (QUEUE) p1_enqueue(S, A, B, tid >> 5, tid & 31, qn, c, xv[j], yv[j], zc, nf);
        }
    }
}

// bulk prefetch of one tile of x (and y) into L2 (TMA, no registers / smem):
// the demand loads of that tile later hit L2
template <bool NORM>
__device__ __forceinline__ void p1_prefetch_l2(const double* x, const double* y, int64_t n, int64_t tile, int TILE) {
    const int64_t e0 = tile * TILE;
    if (e0 + TILE > n) return;
    // evict-first: the streamed lines go before the workspace tables and the
    // code of the kernels that follow (score / finalize run cold otherwise)
    uint64_t pol;
#ifdef QDOT_P1_EVICT_NORMAL
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" :: "l"(bulk_aligned(x + e0)), "r"(TILE * 8), "l"(pol)
                 : "memory");
    if (!NORM)
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" :: "l"(bulk_aligned(y + e0)), "r"(TILE * 8),
                     "l"(pol) : "memory");
}

// persistent loop over tiles.  PF: register double buffering (the loads of
// the CTA's next tile are in flight while the current one is processed).
// L2D > 0: one thread per CTA bulk-prefetches the tile L2D+1 iterations ahead into L2.
template <bool NORM, bool VEC, bool FULL, bool QUEUE, int V, bool PF, int L2D, int WW = P1_W>
__device__ __forceinline__ void p1_main(P1Shared& S, const double* __restrict__ x, const double* __restrict__ y,
                                        int64_t n, int64_t* __restrict__ A, int64_t* __restrict__ B, int tid,
                                        uint32_t* zc, uint32_t* nf) {
    constexpr int EPT = 2 * V;
    constexpr int TILE = P1_T * EPT;
    constexpr int FLUSH = (FULL ? 255 : 511) / EPT;   // tiles between flushes
    const int64_t ntiles = (n + TILE - 1) / TILE;
    const int64_t stride = gridDim.x;
    const int kbias = KOFF - 2046 - S.base;
    ulonglong2* __restrict__ my = S.priv + tid;
    int since = 0;
    uint32_t qn = 0;                                   // warp queue fill (warp-uniform)
    auto flush = [&]() {
        if (QUEUE) p1_drain(S, A, B, tid >> 5, tid & 31, qn, zc, nf);
        p1_flush<FULL, WW>(S, A, B, tid);
    };
    if (!PF) {
        if (L2D > 0 && tid == 0) {   // warm the first prefetch window
            for (int d = 1; d <= L2D; ++d) p1_prefetch_l2<NORM>(x, y, n, blockIdx.x + d * stride, TILE);
        }
        for (int64_t t = blockIdx.x; t < ntiles; t += stride) {
            double xv[EPT], yv[EPT];
            bool f;
            if (L2D > 0 && tid == 0) p1_prefetch_l2<NORM>(x, y, n, t + (L2D + 1) * stride, TILE);
            p1_load<NORM, VEC, V>(x, y, n, t, tid, xv, yv, f);
            p1_tile<FULL, QUEUE, V, WW>(S, my, kbias, A, B, xv, yv, t * TILE, n, f, tid, qn, zc, nf);
            if (++since == FLUSH) { flush(); since = 0; }
        }
    } else {
        double xa[EPT], ya[EPT], xb[EPT], yb[EPT];
        bool fa = false, fb = false;
        int64_t t = blockIdx.x;
        if (L2D > 0 && tid == 0) {
            for (int d = 2; d <= L2D + 1; ++d) p1_prefetch_l2<NORM>(x, y, n, blockIdx.x + d * stride, TILE);
        }
        if (t < ntiles) p1_load<NORM, VEC, V>(x, y, n, t, tid, xa, ya, fa);
        while (t < ntiles) {
            const int64_t tb = t + stride;
            if (L2D > 0 && tid == 0) {
                p1_prefetch_l2<NORM>(x, y, n, t + (L2D + 2) * stride, TILE);
                p1_prefetch_l2<NORM>(x, y, n, t + (L2D + 3) * stride, TILE);
            }
            if (tb < ntiles) p1_load<NORM, VEC, V>(x, y, n, tb, tid, xb, yb, fb);
            p1_tile<FULL, QUEUE, V, WW>(S, my, kbias, A, B, xa, ya, t * TILE, n, fa, tid, qn, zc, nf);
            if (++since == FLUSH) { flush(); since = 0; }
            if (tb >= ntiles) break;
            const int64_t ta = tb + stride;
            if (ta < ntiles) p1_load<NORM, VEC, V>(x, y, n, ta, tid, xa, ya, fa);
            p1_tile<FULL, QUEUE, V, WW>(S, my, kbias, A, B, xb, yb, tb * TILE, n, fb, tid, qn, zc, nf);
            if (++since == FLUSH) { flush(); since = 0; }
            t = ta;
        }
    }
    flush();
}

// ---- norm mode (x . x), lean: every key is 2 ex + KOFF (even), so the P1_W
// private slots are indexed by the exponent of x (slot r <-> key base + 2r),
// and a window element needs no exponent sum, no sign and no scale: with
// m26 = |x| 2^(26 - ex) (x's mantissa bits under the biased exponent 1049),
// fl(m26 * m26) = fl(x * x) 2^(52 - 2 ex) exactly, so one DMUL and one
// conversion give the DOUBLE units (emulate.py:133).  Window keys lie in the
// safe range, so rel < P1_W also excludes zero / subnormal / non-finite x.
// Returns the tile's cold elements (bit j: xv[j] outside the window).
// L2 prefetch of one norm tile with an explicit cache policy (pol from createpolicy)
__device__ __forceinline__ void p1_prefetch_norm(const double* x, int64_t n, int64_t tile, int TILE, uint64_t pol) {
    const int64_t e0 = tile * TILE;
    if (e0 + TILE > n) return;
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" :: "l"(bulk_aligned(x + e0)),
                 "r"(TILE * 8), "l"(pol) : "memory");
}

// WIDE: P1_WW exponents in the wide layout (int64 D at slot * P1_T * 8 + tid * 8,
// u16 count after all D words) -- more exponents in the same bytes, for CTAs
// whose sampled exponents spread beyond the P1_W-slot window (mys: the D base,
// mysc: the count base of this thread)
template <int V, bool FULLT>
__device__ __forceinline__ uint32_t p1_tile_norm_wide(uint32_t mys, uint32_t mysc, uint32_t ebase,
                                                      const double (&xv)[2 * V], int64_t e0, int64_t n, int tid) {
    uint32_t cold = 0;
#pragma unroll
    for (int j = 0; j < 2 * V; ++j) {
        const uint32_t hi = (uint32_t)__double2hiint(xv[j]);
        const uint32_t d = (hi & 0x7FF00000u) - ebase;
        const bool ok = FULLT || e0 + 2 * ((int64_t)(j >> 1) * P1_T + tid) + (j & 1) < n;
        uint32_t mh;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(mh) : "r"(hi), "r"(0x000FFFFFu), "r"(0x41900000u));
        const double m26 = __hiloint2double((int)mh, __double2loint(xv[j]));
        const long long kd = __double2ll_rn(__dmul_rn(m26, m26));
        const bool hot = d < ((uint32_t)P1_WW << 20);
        const uint32_t r = min(d, ((uint32_t)P1_WW - 1u) << 20) >> 20;
        asm volatile("{\n\t.reg .pred p;\n\t.reg .u64 a;\n\t.reg .u16 c;\n\t"
                     "setp.ne.u32 p, %3, 0;\n\t"
                     "ld.shared.u64 a, [%0];\n\t"
                     "add.s64 a, a, %2;\n\t"
                     "@p st.shared.u64 [%0], a;\n\t"
                     "ld.shared.u16 c, [%1];\n\t"
                     "add.u16 c, c, 1;\n\t"
                     "@p st.shared.u16 [%1], c;\n\t}"
                     :: "r"(mys + r * (P1_T * 8)), "r"(mysc + r * (P1_T * 2)), "l"(kd), "r"((uint32_t)(hot && ok)));
        if (!hot && ok) cold |= 1u << j;
    }
    return cold;
}

template <int V, bool FULLT>
__device__ __forceinline__ uint32_t p1_tile_norm(uint32_t mys, uint32_t ebase, const double (&xv)[2 * V],
                                                 int64_t e0, int64_t n, int tid) {
    uint32_t cold = 0;
#pragma unroll
    for (int j = 0; j < 2 * V; ++j) {
        const uint32_t hi = (uint32_t)__double2hiint(xv[j]);
        const uint32_t d = (hi & 0x7FF00000u) - ebase;          // (slot of x's exponent) << 20
        const bool ok = FULLT || e0 + 2 * ((int64_t)(j >> 1) * P1_T + tid) + (j & 1) < n;
        uint32_t mh;                                             // (hi & 0xFFFFF) | 0x41900000 in one LOP3
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(mh) : "r"(hi), "r"(0x000FFFFFu), "r"(0x41900000u));
        const double m26 = __hiloint2double((int)mh, __double2loint(xv[j]));
        const long long kd = __double2ll_rn(__dmul_rn(m26, m26));
        const bool hot = d < ((uint32_t)P1_W << 20);
        // slot {D lo, D hi, count, 0} at mys + slot * P1_T * 16 bytes.  Straight-line code
        // (no per-element branch / reconvergence): every element loads a slot (a cold one
        // reads slot min(d, P1_W - 1), harmlessly) and only a window element stores it back
        asm volatile("{\n\t.reg .pred p;\n\t.reg .u32 a, b, c, w;\n\t"
                     "setp.ne.u32 p, %3, 0;\n\t"
                     "ld.shared.v4.u32 {a, b, c, w}, [%0];\n\t"
                     "add.cc.u32 a, a, %1;\n\t"
                     "addc.u32 b, b, %2;\n\t"
                     "add.u32 c, c, 1;\n\t"
                     "@p st.shared.v4.u32 [%0], {a, b, c, w};\n\t}"
                     :: "r"(mys + (min(d, ((uint32_t)P1_W - 1u) << 20) >> 8)), "r"((uint32_t)kd),
                        "r"((uint32_t)((unsigned long long)kd >> 32)), "r"((uint32_t)(hot && ok)));
        // (no memory clobber: it would force the tile's registers into local memory; the
        // slots are touched by C++ code only across __syncthreads, and volatile asm keeps
        // its order)
        if (!hot && ok) cold |= 1u << j;
    }
    return cold;
}

// one norm tile: window elements into the private slots, cold ones through the
// warp queue, the flush every FLUSH tiles
template <int V, bool WIDE>
__device__ __forceinline__ void p1_norm_tile(P1Shared& S, int64_t* __restrict__ A, int64_t* __restrict__ B,
                                             uint32_t mys, uint32_t mysc, uint32_t ebase, const double (&xv)[2 * V],
                                             int64_t t, bool f, int64_t n, int tid, uint32_t& qn, int& since,
                                             uint32_t* zc, uint32_t* nf) {
    constexpr int EPT = 2 * V;
    constexpr int FLUSH = 511 / EPT;                   // D < 511 * 2^54 per slot between flushes
    const int warp = tid >> 5, lane = tid & 31;
    uint32_t cold;
    if (WIDE) cold = f ? p1_tile_norm_wide<V, true>(mys, mysc, ebase, xv, t * (P1_T * EPT), n, tid)
                       : p1_tile_norm_wide<V, false>(mys, mysc, ebase, xv, t * (P1_T * EPT), n, tid);
    else cold = f ? p1_tile_norm<V, true>(mys, ebase, xv, t * (P1_T * EPT), n, tid)
                  : p1_tile_norm<V, false>(mys, ebase, xv, t * (P1_T * EPT), n, tid);
    const uint32_t wm = __reduce_or_sync(0xffffffffu, cold);     // positions with a cold element in the warp
    if (wm) {
#pragma unroll
        for (int j = 0; j < EPT; ++j)
            if ((wm >> j) & 1u) p1_enqueue(S, A, B, warp, lane, qn, (cold >> j) & 1u, xv[j], xv[j], zc, nf);
    }
    if (++since == FLUSH) {
        p1_drain(S, A, B, warp, lane, qn, zc, nf);
        p1_flush<false, WIDE ? P1_WW : P1_W>(S, A, B, tid);
        since = 0;
    }
}

// (register double buffering -- the next tile's loads issued before the current
// tile is accumulated -- and two tiles per iteration both measured slower:
// 0.60 / 0.49 vs 0.45 ms at 2^28, profiles/r2_norm_experiments.md)
template <bool VEC, int V, bool WIDE>
__device__ __forceinline__ void p1_main_norm(P1Shared& S, const double* __restrict__ x, int64_t n,
                                             int64_t* __restrict__ A, int64_t* __restrict__ B, int tid,
                                             uint32_t* zc, uint32_t* nf, int L2D, int pmode) {
    constexpr int EPT = 2 * V;
    constexpr int TILE = P1_T * EPT;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    const int64_t stride = gridDim.x;
    // slot r holds key base + 2r, i.e. biased exponent fx = r + (base - KOFF) / 2 + 1023
    const uint32_t ebase = (uint32_t)((S.base - KOFF) / 2 + 1023) << 20;
    const uint32_t pbase = (uint32_t)__cvta_generic_to_shared(S.priv);
    const uint32_t mys = WIDE ? pbase + tid * 8 : pbase + tid * 16;
    const uint32_t mysc = pbase + P1_WW * P1_T * 8 + tid * 2;      // wide layout's u16 counts
    int since = 0;
    uint32_t qn = 0;
    // prefetched lines: evict-first (0), evict-normal (1) or evict-last (2); the demand
    // loads stream with evict-first either way
    uint64_t pol = 0;
    if (tid == 0) {
        if (pmode == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        else if (pmode == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    }
    if (L2D > 0 && tid == 0) {
        for (int d = 1; d <= L2D; ++d) p1_prefetch_norm(x, n, blockIdx.x + d * stride, TILE, pol);
    }
    for (int64_t t = blockIdx.x; t < ntiles; t += stride) {
        double xv[EPT], yv[EPT];
        bool f;
        if (L2D > 0 && tid == 0) p1_prefetch_norm(x, n, t + (L2D + 1) * stride, TILE, pol);
        p1_load<true, VEC, V>(x, x, n, t, tid, xv, yv, f);
        p1_norm_tile<V, WIDE>(S, A, B, mys, mysc, ebase, xv, t, f, n, tid, qn, since, zc, nf);
    }
    const int warp = tid >> 5, lane = tid & 31;
    p1_drain(S, A, B, warp, lane, qn, zc, nf);
    p1_flush<false, WIDE ? P1_WW : P1_W>(S, A, B, tid);
}

// SMALL: the variant for short inputs (a few tiles per CTA), where the fixed
// per-CTA cost dominates: one main loop (full variants, no queue, no L2
// prefetch) keeps the code a CTA must fetch small.
template <bool NORM, bool VEC, int V, bool PF, int L2D, bool SMALL>
__global__ void __launch_bounds__(P1_T, QDOT_P1_MINB)
k_pass1(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
        int64_t* __restrict__ A, int64_t* __restrict__ B, P1Params prm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    P1Shared& S = *reinterpret_cast<P1Shared*>(smem_raw);
    const int tid = threadIdx.x;
    constexpr int TILE = P1_T * 2 * V;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    pdl_trigger();   // score may be scheduled as SMs drain; it waits for this grid

    if (SMALL) {
        // short inputs: the window only has to be reasonable -- [kmax - W + 3,
        // kmax + 2] around the largest key of the first tile (no histogram)
        int kmx = -1;
        if ((int64_t)blockIdx.x < ntiles) {
            double xv[2 * V], yv[2 * V];
            bool full;
            p1_load<NORM, VEC, V>(x, y, n, blockIdx.x, tid, xv, yv, full);
            const int64_t e0 = (int64_t)blockIdx.x * TILE;
#pragma unroll
            for (int j = 0; j < 2 * V; ++j) {
                const int64_t i = e0 + 2 * ((int64_t)(j >> 1) * P1_T + tid) + (j & 1);
                const uint32_t fx = (uint32_t)(dbits(xv[j]) >> 52) & 0x7FFu, fy = (uint32_t)(dbits(yv[j]) >> 52) & 0x7FFu;
                if (i < n && fx - 1u < 0x7FEu && fy - 1u < 0x7FEu) kmx = max(kmx, (int)(fx + fy) - 2046 + KOFF);
            }
        }
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        if ((tid & 31) == 0) S.red[tid >> 5] = (unsigned long long)(long long)kmx;
        pdl_wait();      // the sampling above reads only x, y; the workspace comes next
        if (blockIdx.x == 0 && tid == 0) atomicCAS(ws_stamps(A), 0ull, global_ns());   // first launch only
        __syncthreads();
        if (tid == 0) {
            int m = -1;
            for (int w = 0; w < P1_T / 32; ++w) m = max(m, (int)(long long)S.red[w]);
            int b = m < 0 ? KOFF - 8 : m - P1_W + 3;
            b = b < P1_SAFE_LO ? P1_SAFE_LO : (b > P1_SAFE_HI ? P1_SAFE_HI : b);
            S.kmax = m;
            S.base = b;
            int cb = b - (P1_CW - P1_W) / 2;
            cb = cb < 0 ? 0 : cb;
            S.cbase = cb + P1_CW > KEYS ? KEYS - P1_CW : cb;
            S.full = 1;
            S.wide = 0;
            S.queue = 0;
            S.norm_lean = 0;
            const bool slot_ok = blockIdx.x < (unsigned)LIST_SLOTS;
            S.list = prm.list + (int64_t)(slot_ok ? blockIdx.x : 0) * LIST_PER_SLOT;
            S.list_fill = slot_ok ? prm.list_fill[blockIdx.x] : (uint32_t)LIST_PER_SLOT;
            S.collect = prm.collect;
        }
        __syncthreads();
    } else {
        // ---- sample this CTA's first tile: histogram of keys (reusing priv)
        uint32_t* hist = reinterpret_cast<uint32_t*>(S.priv);           // KEYS u32
        uint32_t* pref = hist + 4224;                                   // KEYS+1 u32
        for (int k = tid; k < 4224 * 2; k += P1_T) hist[k] = 0u;
        __syncthreads();
        if ((int64_t)blockIdx.x < ntiles) {
            double xv[2 * V], yv[2 * V];
            bool full;
            p1_load<NORM, VEC, V>(x, y, n, blockIdx.x, tid, xv, yv, full);
            const int64_t e0 = (int64_t)blockIdx.x * TILE;
    #pragma unroll
            for (int j = 0; j < 2 * V; ++j) {
                int64_t i = e0 + 2 * ((int64_t)(j >> 1) * P1_T + tid) + (j & 1);
                if (i >= n) continue;
                uint64_t bx = dbits(xv[j]), by = dbits(yv[j]);
                uint32_t fx = (uint32_t)(bx >> 52) & 0x7FFu, fy = (uint32_t)(by >> 52) & 0x7FFu;
                if (fx - 1u < 0x7FEu && fy - 1u < 0x7FEu) atomicAdd(&hist[(int)(fx + fy) - 2046 + KOFF], 1u);
            }
        }
        pdl_wait();      // the sampling above reads only x, y; the workspace comes next
        if (blockIdx.x == 0 && tid == 0) atomicCAS(ws_stamps(A), 0ull, global_ns());   // first launch only
        __syncthreads();
        {   // inclusive prefix over KEYS (17 keys per thread) + largest sampled key
            constexpr int PER = (KEYS + P1_T - 1) / P1_T;
            uint32_t loc[PER];
            uint32_t run = 0;
            int kmx = -1;
    #pragma unroll
            for (int i = 0; i < PER; ++i) {
                int k = tid * PER + i;
                uint32_t h = k < KEYS ? hist[k] : 0u;
                if (h) kmx = k;
                run += h;
                loc[i] = run;
            }
            const int lane = tid & 31, warp = tid >> 5;
            uint32_t incl = run;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            for (int o = 16; o; o >>= 1) kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
            if (lane == 31) S.red[warp] = incl;
            if (lane == 0) S.red[P1_T / 32 + warp] = (unsigned long long)(long long)kmx;
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
            if (tid == 0) {
                int m = -1;
                for (int w = 0; w < P1_T / 32; ++w) m = max(m, (int)(long long)S.red[P1_T / 32 + w]);
                S.kmax = m;
            }
        }
        __syncthreads();
        {   // private window: argmax over starts b of pref[b+W] - pref[b], inside the safe
            // range, for the 16-key window and the 24-key wide lean window
            unsigned long long best = 0ull, best24 = 0ull;
            for (int b = P1_SAFE_LO + tid; b <= P1_SAFE_HI; b += P1_T) {
                uint32_t s = pref[b + P1_W] - pref[b];
                unsigned long long cand = ((unsigned long long)s << 32) | (uint32_t)(0xFFFFFFFFu - b);
                best = cand > best ? cand : best;
                if (b <= P1_SAFE_HI_W) {
                    const uint32_t s24 = pref[b + P1_WW] - pref[b];
                    const unsigned long long c24 = ((unsigned long long)s24 << 32) | (uint32_t)(0xFFFFFFFFu - b);
                    best24 = c24 > best24 ? c24 : best24;
                }
            }
            for (int o = 16; o; o >>= 1) {
                unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
                best = t > best ? t : best;
                t = __shfl_xor_sync(0xffffffffu, best24, o);
                best24 = t > best24 ? t : best24;
            }
            __syncthreads();
            if ((tid & 31) == 0) { S.red[tid >> 5] = best; S.red[P1_T / 32 + (tid >> 5)] = best24; }
            __syncthreads();
            if (tid == 0) {
                unsigned long long m = 0ull, m24 = 0ull;
                for (int w = 0; w < P1_T / 32; ++w) {
                    m = S.red[w] > m ? S.red[w] : m;
                    m24 = S.red[P1_T / 32 + w] > m24 ? S.red[P1_T / 32 + w] : m24;
                }
                int b = (m >> 32) ? (int)(0xFFFFFFFFu - (uint32_t)m) : (KOFF - 8);   // default near e = 0
                // lean / full decision (see header); only speed depends on it
                int full = 0;
                if (SMALL || (prm.mode & 3) == 2 || prm.input_mu != 52) full = 1;
                else if ((prm.mode & 3) == 0) {
                    const uint32_t ns = pref[KEYS];
                    const int fl = flexp_bits(dbits(prm.epsilon));
                    for (int r = 0; r < P1_W && ns; ++r) {
                        uint32_t c = hist[b + r];
                        if (!c) continue;
                        double mest = (double)c * (double)prm.n_total / (double)ns;
                        int lg = mest >= 1.0 ? flexp_bits(dbits(mest)) : 0;
                        int score = lg - 2 + (b + r - S.kmax) - fl + 1;
                        if (score > -6 && score < 27) full = 1;
                    }
                }
                S.full = full;
                // wide lean window (24 keys): a lean CTA whose 16-key window misses more
                // than 3% of its sample switches to the best 24-key window when that
                // covers more and none of its keys can plausibly score below 27
                int wide = 0, ww = P1_W;
                if (!full && (m24 >> 32) && ((prm.mode & 16) || ((prm.mode & 3) == 0 && (prm.mode & 12) == 0))) {
                    const uint32_t ns = pref[KEYS];
                    const int b24 = (int)(0xFFFFFFFFu - (uint32_t)m24);
                    const uint32_t cov16 = pref[b + P1_W] - pref[b], cov24 = pref[b24 + P1_WW] - pref[b24];
                    bool ok = (prm.mode & 16) != 0;
                    if (!ok && (uint64_t)cov16 * 100u < (uint64_t)ns * 97u && cov24 > cov16) {
                        ok = true;
                        const int fl = flexp_bits(dbits(prm.epsilon));
                        for (int r = 0; r < P1_WW; ++r) {
                            const uint32_t c = hist[b24 + r];
                            if (!c) continue;
                            const double mest = (double)c * (double)prm.n_total / (double)ns;
                            const int lg = mest >= 1.0 ? flexp_bits(dbits(mest)) : 0;
                            const int score = lg - 2 + (b24 + r - S.kmax) - fl + 1;
                            if (score > -6 && score < 27) ok = false;
                        }
                    }
                    if (ok) { wide = 1; ww = P1_WW; b = b24; }
                }
                S.wide = wide;
                S.base = b;
                int cb = b - (P1_CW - ww) / 2;
                cb = cb < 0 ? 0 : cb;
                cb = cb + P1_CW > KEYS ? KEYS - P1_CW : cb;
                S.cbase = cb;
                const bool slot_ok = blockIdx.x < (unsigned)LIST_SLOTS;
                S.list = prm.list + (int64_t)(slot_ok ? blockIdx.x : 0) * LIST_PER_SLOT;
                S.list_fill = slot_ok ? prm.list_fill[blockIdx.x] : (uint32_t)LIST_PER_SLOT;   // no slot: never write
                S.collect = prm.collect;
                // queue mode when more than 1/128 of the sample lies outside the private window
                const uint32_t ns = pref[KEYS], cov = pref[b + ww] - pref[b];
                const int qm = (prm.mode >> 2) & 3;
                S.queue = qm == 1 ? 1 : (qm == 2 ? 0 : ((ns - cov) * 128u > ns));
                S.norm_lean = 0;
            }
        }
        __syncthreads();
        if (NORM && (prm.mode & 32) == 0 && (prm.mode & 3) != 2 && prm.input_mu == 52) {
            // norm lean window: P1_W exponents (keys b, b + 2, .., b + 2 P1_W - 2), the
            // start maximising the sampled coverage among windows holding no sampled key
            // whose estimated score could reach HALF / SINGLE (those stay in the cold
            // path, which computes the exact variants).  eps_eff is bounded with the
            // number of sampled keys under per-bin splitting (n_bins >= that number).
            constexpr int PER = (KEYS + P1_T - 1) / P1_T;
            constexpr int SPAN = 2 * P1_W - 1;
            uint16_t* upref = reinterpret_cast<uint16_t*>(hist + 8448);    // KEYS+1 u16 (<= 2048)
            const int lane = tid & 31, warp = tid >> 5;
            const uint32_t ns = pref[KEYS];
            uint32_t nk = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int k = tid * PER + i;
                nk += (k < KEYS && hist[k]) ? 1u : 0u;
            }
            nk = __reduce_add_sync(0xffffffffu, nk);
            if (lane == 0) S.red[warp] = nk;
            __syncthreads();
            uint32_t nkeys = 0;
            for (int w = 0; w < P1_T / 32; ++w) nkeys += (uint32_t)S.red[w];
            const double eps_e = prm.per_bin && nkeys > 1 ? prm.epsilon / (double)nkeys : prm.epsilon;
            const int fl = flexp_bits(dbits(eps_e));
            const bool check = (prm.mode & 3) == 0;
            uint32_t loc[PER];
            uint32_t run = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int k = tid * PER + i;
                const uint32_t c = k < KEYS ? hist[k] : 0u;
                uint32_t u = 0;
                if (c && check) {
                    const double mest = (double)c * (double)prm.n_total / (double)ns;
                    const int lg = mest >= 1.0 ? flexp_bits(dbits(mest)) : 0;
                    // the sampled kmax undershoots e_max and the sampled key count n_bins
                    // (score overestimated / underestimated by about as much), so the
                    // margin to 23 (SINGLE) covers the count's sampling noise
                    const int score = lg - 2 + (k - S.kmax) - fl + 1;
                    u = (score > -6 && score < 25) ? 1u : 0u;
                }
                run += u;
                loc[i] = run;
            }
            uint32_t incl = run;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            __syncthreads();
            if (lane == 31) S.red[warp] = incl;
            __syncthreads();
            uint32_t pre = incl - run;
            for (int w = 0; w < warp; ++w) pre += (uint32_t)S.red[w];
            if (tid == 0) upref[0] = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int k = tid * PER + i;
                if (k < KEYS) upref[k + 1] = (uint16_t)(pre + loc[i]);
            }
            __syncthreads();
            // best lean-safe window of P1_W exponents (16-byte slots) and of P1_WW
            // exponents (the wide 10-byte layout)
            constexpr int SPANW = 2 * P1_WW - 1;
            unsigned long long best = 0ull, bestw = 0ull;
            const int lo = P1_SAFE_LO + ((P1_SAFE_LO - KOFF) & 1);           // keys of x . x have KOFF's parity
            for (int b = lo + 2 * tid; b + SPAN - 1 <= KOFF + 1021; b += 2 * P1_T) {
                if (upref[b + SPAN] != upref[b]) continue;
                const uint32_t cov = pref[b + SPAN] - pref[b];
                const unsigned long long cand = ((unsigned long long)cov << 32) | (uint32_t)b;   // ties: larger b
                best = cand > best ? cand : best;
                if (b + SPANW - 1 <= KOFF + 1021 && upref[b + SPANW] == upref[b]) {
                    const uint32_t cw = pref[b + SPANW] - pref[b];
                    const unsigned long long cd = ((unsigned long long)cw << 32) | (uint32_t)b;
                    bestw = cd > bestw ? cd : bestw;
                }
            }
            for (int o = 16; o; o >>= 1) {
                unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
                best = t > best ? t : best;
                t = __shfl_xor_sync(0xffffffffu, bestw, o);
                bestw = t > bestw ? t : bestw;
            }
            __syncthreads();
            if (lane == 0) { S.red[warp] = best; S.red[P1_T / 32 + warp] = bestw; }
            __syncthreads();
            if (tid == 0) {
                unsigned long long m = 0ull, mw = 0ull;
                for (int w = 0; w < P1_T / 32; ++w) {
                    m = S.red[w] > m ? S.red[w] : m;
                    mw = S.red[P1_T / 32 + w] > mw ? S.red[P1_T / 32 + w] : mw;
                }
                const uint32_t cov = (uint32_t)(m >> 32), covw = (uint32_t)(mw >> 32);
                // the 16-byte slots when they hold >= 99% of the sample, else the wide
                // layout when it holds >= 7/8 (the rest goes through the cold-element queue)
                int b = -1, wide = 0;
                if (ns && (uint64_t)cov * 100u >= (uint64_t)ns * 99u) b = (int)(uint32_t)m;
                else if (ns && covw > cov && (uint64_t)covw * 8u >= (uint64_t)ns * 7u) { b = (int)(uint32_t)mw; wide = 1; }
                else if (ns && (uint64_t)cov * 8u >= (uint64_t)ns * 7u) b = (int)(uint32_t)m;
                if (b >= 0) {
                    const int span = wide ? SPANW : SPAN;
                    S.norm_lean = 1;
                    S.full = 0;
                    S.wide = wide;
                    S.queue = 1;
                    S.base = b;
                    int cb = b - (P1_CW - span) / 2;
                    cb = cb < 0 ? 0 : cb;
                    S.cbase = cb + P1_CW > KEYS ? KEYS - P1_CW : cb;
                }
            }
            __syncthreads();
        }
    }
    // ---- clear private slots, cold table and totals
    for (int k = tid; k < P1_W * P1_T; k += P1_T) S.priv[k] = make_ulonglong2(0ull, 0ull);
    for (int k = tid; k < P1_CW; k += P1_T) {
        S.c_cnt[k] = 0u; S.c_d0[k] = 0u; S.c_d1[k] = 0u; S.c_d2[k] = 0u; S.c_d3[k] = 0u;
        S.c_s0[k] = 0u; S.c_s1[k] = 0u; S.c_h[k] = 0u;
    }
    if (tid < P1_WW) { S.t_d[tid] = 0; S.t_s[tid] = 0; S.t_h[tid] = 0; S.t_c[tid] = 0; }
    __syncthreads();

    // ---- main streaming loop (persistent grid over tiles)
    uint32_t zc = 0, nf = 0;
    const bool fullmode = SMALL || S.full != 0;
    if (SMALL) {
        p1_main<NORM, VEC, true, false, V, false, 0>(S, x, y, n, A, B, tid, &zc, &nf);
    } else if (NORM && S.norm_lean) {
        // L2 prefetch distance in tiles (a norm tile is half the bytes of an x . y tile);
        // mode bits 6-7 select it for tuning: 0 -> L2D, 1 -> 2 L2D + 1, 2 -> none, 3 -> 1
        const int sel = (prm.mode >> 6) & 3;
        const int l2d = L2D == 0 ? 0 : (sel == 0 ? L2D : (sel == 1 ? 2 * L2D + 1 : (sel == 2 ? 0 : 1)));
        if (S.wide) p1_main_norm<VEC, V, true>(S, x, n, A, B, tid, &zc, &nf, l2d, (prm.mode >> 8) & 3);
        else p1_main_norm<VEC, V, false>(S, x, n, A, B, tid, &zc, &nf, l2d, (prm.mode >> 8) & 3);
    } else if (S.wide) {
        if (S.queue) p1_main<NORM, VEC, false, true, V, PF, L2D, P1_WW>(S, x, y, n, A, B, tid, &zc, &nf);
        else p1_main<NORM, VEC, false, false, V, PF, L2D, P1_WW>(S, x, y, n, A, B, tid, &zc, &nf);
    } else if (S.queue) {
        if (fullmode) p1_main<NORM, VEC, true, true, V, PF, L2D>(S, x, y, n, A, B, tid, &zc, &nf);
        else p1_main<NORM, VEC, false, true, V, PF, L2D>(S, x, y, n, A, B, tid, &zc, &nf);
    } else {
        if (fullmode) p1_main<NORM, VEC, true, false, V, PF, L2D>(S, x, y, n, A, B, tid, &zc, &nf);
        else p1_main<NORM, VEC, false, false, V, PF, L2D>(S, x, y, n, A, B, tid, &zc, &nf);
    }

    // ---- publish CTA partials (the cold table was pushed by the last flush)
    const int kstep = (NORM && S.norm_lean) ? 2 : 1;
    for (int r = tid; r < (S.wide ? P1_WW : P1_W); r += P1_T) {
        if (S.t_c[r]) {
            const int key = S.base + kstep * r;
            push_key(A, B, key, (unsigned long long)S.t_c[r], S.t_d[r], S.t_s[r], S.t_h[r]);
            atomicAdd(reinterpret_cast<unsigned long long*>(A + A_PRIV + key), (unsigned long long)S.t_c[r]);
            if (!fullmode) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_HOT + key),
                                     (unsigned long long)S.t_c[r]);
        }
    }
    __syncthreads();
    if (tid == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(A + (fullmode ? A_FULLCTAS : A_LEANCTAS)), 1ull);
        const uint32_t f = S.list_fill;
        if (blockIdx.x < (unsigned)LIST_SLOTS) {
            const uint32_t before = prm.list_fill[blockIdx.x];
            prm.list_fill[blockIdx.x] = f;
            if (f > (uint32_t)LIST_PER_SLOT && before <= (uint32_t)LIST_PER_SLOT)   // flag each slot once
                atomicAdd(reinterpret_cast<unsigned long long*>(A + A_LISTOVF), 1ull);
        } else if (f > (uint32_t)LIST_PER_SLOT) {
            atomicAdd(reinterpret_cast<unsigned long long*>(A + A_LISTOVF), 1ull);
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
