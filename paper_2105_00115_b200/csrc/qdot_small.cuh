// qdot_small.cuh -- a whole single-device qdot of a short vector in ONE launch:
// a thread-block cluster (included into namespace qd of qdot_kernels.cu).
//
// The multi-CTA pipeline (begin, pass 1, score, pass 2) costs four dependent
// launches and a 400 KB workspace reset -- at the solvers' sizes (n ~ 1e3 ..
// 6e4, apps.py:178-229, 275-325) that is the whole call.  Here the CL CTAs
// of one cluster keep every exact per-key partial in shared memory:
//
//   1. window: each CTA reads the same first 2 SM_T elements (its own first
//      pair already in flight); the largest
//      exponent-sum key kmx places the private window [kmx - 13, kmx + 2]
//      (per-thread slots, full DOUBLE / SINGLE / HALF variants as in pass 1's
//      full loop) inside a 64-key table [kmx - 61, kmx + 2] (per-CTA 32-bit
//      limb counters, shared atomics);
//   2. every element goes to its slot or table key (exact integers, order
//      independent: emulate.py:133-146 restated as in pass 1);
//   3. per-CTA totals, then CTA 0 sums the cluster's totals through
//      distributed shared memory (no global traffic, no workspace reset);
//   4. CTA 0's first warp scores, rounds, folds and writes the result header,
//      bins and LUTs exactly as score_warp does for the global regions
//      (kernel.py:179-240 via scoring.py / emulate.py).
//
// Anything outside that shape -- a key outside the 64-key table, a DOUBLE
// product overflow, a sample without a normal element, a window clamped at the
// exponent range's ends, no nonzero product -- is handed over: the cluster
// zeroes the exchange regions, CTA 0 adds the in-table totals, every CTA adds
// its out-of-table elements with global atomics (pass 1's global path) and
// A[A_SMALL] = 2 lets the k_score / k_pass2 launches that follow finish the
// call as usual.  In the common case they see A[A_SMALL] = 1 / meta->done and
// return at once.

// (cooperative_groups.h is included at the top of qdot_kernels.cu, outside namespace qd)

constexpr int SM_CL = 16;                        // CTAs per cluster, at most (16: non-portable, B200 runs it)
constexpr int SM_CL_SMALL = 8;                   // n <= SM_CL_SPLIT: the portable 8
constexpr int SM_T = 256;                        // threads per CTA
constexpr int SM_K = 64;                         // table keys (= score_warp's span)
constexpr int SM_EPT = 32;                       // elements per thread at the size limit (<= 255: slot count)
constexpr int64_t SM_MAX = (int64_t)SM_CL * SM_T * SM_EPT;   // 131072
constexpr int64_t SM_CL_SPLIT = 16384;
static_assert(SM_K == SW_KEYS, "score_warp scores the table");

struct __align__(16) SmShared {
    ulonglong2 priv[P1_W * SM_T];                // per-thread {D, packed S | H | count} (pass 1's full layout)
    __int128 td[SM_K];                           // per-key totals of this CTA (CTA 0: of the cluster)
    long long tsum[SM_K], thalf[SM_K];
    unsigned long long tcnt[SM_K];
    // CTA 0 only: every CTA's totals, pushed through distributed shared memory
    __int128 rd[SM_CL][SM_K];
    long long rs[SM_CL][SM_K], rh[SM_CL][SM_K];
    unsigned long long rc[SM_CL][SM_K];
    unsigned long long rzc[SM_CL], rnf[SM_CL];
    int roor[SM_CL];
    uint32_t c[8][SM_K];                         // limb table: cnt, d0, d1, d2, d3 (signed), s0, s1 (signed), h
    double sval[SM_K + 1];                       // score_warp scratch
    long long bup[SM_K + 1];
    signed char bprec[SM_K + 1];
    unsigned long long zc, nf;                   // zero / non-finite products of this CTA (CTA 0: cluster)
    int oor;                                     // an element this path cannot keep (hand over)
    int kmx;
    int decision;                                // CTA 0: 1 finish here, 2 hand over (read by every CTA)
    int post;                                    // CTA 0: score_warp asked for a pass 2 (hand over after all)
    int kmin, kmax;
};

size_t small_smem_bytes() { return sizeof(SmShared); }

// score_warp's view of the cluster totals (CTA 0's shared memory)
struct SmallKeys {
    const SmShared* S;
    int cbase;
    __device__ __forceinline__ long long d(int i, int k) const {
        const __int128 D = S->td[k - cbase];
        return i < 3 ? (long long)(uint32_t)(uint64_t)(D >> (32 * i)) : (long long)(D >> 96);
    }
    __device__ __forceinline__ long long infp(int) const { return 0; }
    __device__ __forceinline__ long long infn(int) const { return 0; }
    __device__ __forceinline__ long long cnt(int k) const { return (long long)S->tcnt[k - cbase]; }
    __device__ __forceinline__ long long keyval(int k, bool half) const {
        return half ? S->thalf[k - cbase] : S->tsum[k - cbase];
    }
};
struct SmallSrc {
    const SmShared* S;
    int cbase;
    __device__ __forceinline__ long long cnt(int k) const { return (long long)S->tcnt[k - cbase]; }
    __device__ __forceinline__ long long hot(int) const { return 0; }       // every variant is exact here
    __device__ __forceinline__ long long priv(int) const { return 0; }
    __device__ __forceinline__ SmallKeys keys() const { return SmallKeys{S, cbase}; }
};

// element outside the private window: the table key's limbs (shared atomics),
// a zero / non-finite count, or "cannot keep" (returns true)
__device__ __forceinline__ bool sm_cold(SmShared& S, int cbase, double xv, double yv, uint32_t& zc, uint32_t& nf) {
    const uint64_t bx = dbits(xv), by = dbits(yv);
    if (((bx >> 52) & 0x7FF) == 0x7FF || ((by >> 52) & 0x7FF) == 0x7FF) { ++nf; return false; }
    if (xv == 0.0 || yv == 0.0) { ++zc; return false; }                  // floatbits.py:74
    const int e = flexp_bits(bx) + flexp_bits(by);
    const int c = e + KOFF - cbase;
    if ((unsigned)c >= (unsigned)SM_K) return true;
    const uint64_t pb = dbits(__dmul_rn(xv, yv));
    if (((pb >> 52) & 0x7FF) == 0x7FF) return true;                     // DOUBLE overflow
    const int64_t kd = double_units(pb, e);
    int32_t ks, kh;
    exact_variants(bitsd(mant_bits(bx)), bitsd(mant_bits(by)), ks, kh);
    const int32_t sg = -(int32_t)((bx ^ by) >> 63);
    ks = (ks ^ sg) - sg;
    kh = (kh ^ sg) - sg;
    const uint64_t u = (uint64_t)kd;
    atomicAdd(&S.c[0][c], 1u);
    atomicAdd(&S.c[1][c], (uint32_t)(u & 0x3FFFu));
    atomicAdd(&S.c[2][c], (uint32_t)((u >> 14) & 0x3FFFu));
    atomicAdd(&S.c[3][c], (uint32_t)((u >> 28) & 0x3FFFu));
    atomicAdd(&S.c[4][c], (uint32_t)(int32_t)(kd >> 42));
    atomicAdd(&S.c[5][c], (uint32_t)ks & 0x3FFFu);
    atomicAdd(&S.c[6][c], (uint32_t)(ks >> 14));
    atomicAdd(&S.c[7][c], (uint32_t)kh);
    return false;
}

// hand-over path of one element: pass 1's global accumulation (regions A / B)
__device__ __forceinline__ void sm_global(int64_t* __restrict__ A, int64_t* __restrict__ B, double xv, double yv,
                                          bool count_special, uint32_t& zc, uint32_t& nf) {
    const uint64_t bx = dbits(xv), by = dbits(yv);
    if (((bx >> 52) & 0x7FF) == 0x7FF || ((by >> 52) & 0x7FF) == 0x7FF) { if (count_special) ++nf; return; }
    if (xv == 0.0 || yv == 0.0) { if (count_special) ++zc; return; }
    const int e = flexp_bits(bx) + flexp_bits(by);
    const int key = e + KOFF;
    const uint64_t pb = dbits(__dmul_rn(xv, yv));
    int64_t kd = 0;
    if (((pb >> 52) & 0x7FF) == 0x7FF)
        atomicAdd(reinterpret_cast<unsigned long long*>(B + ((pb >> 63) ? B_INFN : B_INFP) + key), 1ull);
    else
        kd = double_units(pb, e);
    int32_t ks, kh;
    exact_variants(bitsd(mant_bits(bx)), bitsd(mant_bits(by)), ks, kh);
    const int32_t sg = -(int32_t)((bx ^ by) >> 63);
    ks = (ks ^ sg) - sg;
    kh = (kh ^ sg) - sg;
    push_key(A, B, key, 1ull, (__int128)kd, ks, kh);
}

template <bool NORM, bool VEC>
__device__ __forceinline__ void sm_load2(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                                         int64_t i, double (&xv)[2], double (&yv)[2], bool (&ok)[2]) {
    if (VEC && i + 1 < n) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(x + i));
        xv[0] = a.x; xv[1] = a.y;
        if (NORM) { yv[0] = a.x; yv[1] = a.y; }
        else { const double2 b = __ldcs(reinterpret_cast<const double2*>(y + i)); yv[0] = b.x; yv[1] = b.y; }
        ok[0] = ok[1] = true;
    } else {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            ok[k] = i + k < n;
            xv[k] = ok[k] ? x[i + k] : 0.0;
            yv[k] = ok[k] ? (NORM ? xv[k] : y[i + k]) : 0.0;
        }
    }
}

// CL CTAs per cluster (launched with a cluster-dimension attribute)
template <bool NORM, bool VEC, int CL>
__global__ void __launch_bounds__(SM_T, 1)
k_small(const double* __restrict__ x, const double* __restrict__ y, int64_t n, int64_t* __restrict__ A,
        int64_t* __restrict__ B, int32_t* __restrict__ lut_bin, uint32_t* __restrict__ lut_p2,
        ScoreMeta* __restrict__ meta, qdot_result* __restrict__ res, qdot_bin* __restrict__ bins, qdot_config cfg) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmShared& S = *reinterpret_cast<SmShared*>(smem_raw);
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned long long ts0 = global_ns();
    pdl_trigger();                               // k_score may be scheduled; it waits for this grid
    // split cluster barrier: every CTA has started (its shared memory exists)
    // before any distributed-shared-memory access; the wait is just before the push
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    // phase clocks of CTA 0 (SM cycles since entry) in A[A_SMALL + 1 ..]: diagnostics
    const long long c0 = clock64();
    auto phase = [&](int i) {
        if (rank == 0 && tid == 0) A[A_SMALL + i] = clock64() - c0;
    };

    const int64_t stride = 2 * (int64_t)SM_T * CL;
    const int64_t i0 = 2 * ((int64_t)rank * SM_T + tid);
    double cx[2] = {0.0, 0.0}, cy[2] = {0.0, 0.0};          // this thread's first pair, in flight
    bool cok[2] = {false, false};                           // during the sample's reduction
    if (i0 < n) sm_load2<NORM, VEC>(x, y, n, i0, cx, cy, cok);
    // ---- clear, and the common sample: elements [0, 2 SM_T) -> largest key
    for (int i = tid; i < P1_W * SM_T; i += SM_T) S.priv[i] = make_ulonglong2(0ull, 0ull);
    for (int i = tid; i < 8 * SM_K; i += SM_T) (&S.c[0][0])[i] = 0u;
    if (tid == 0) { S.zc = 0; S.nf = 0; S.oor = 0; S.kmx = -1; S.decision = 0; S.post = 0; }
    __syncthreads();
    {
        double xv[2], yv[2];
        bool ok[2];
        sm_load2<NORM, VEC>(x, y, n, 2 * (int64_t)tid, xv, yv, ok);
        int kmx = -1;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t fx = (uint32_t)(dbits(xv[k]) >> 52) & 0x7FFu, fy = (uint32_t)(dbits(yv[k]) >> 52) & 0x7FFu;
            if (ok[k] && fx - 1u < 0x7FEu && fy - 1u < 0x7FEu) kmx = max(kmx, (int)(fx + fy) - 2046 + KOFF);
        }
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        if (lane == 0 && kmx >= 0) atomicMax(&S.kmx, kmx);
    }
    __syncthreads();
    phase(1);
    const int kmx = S.kmx;
    const int base = kmx - P1_W + 3;             // window [kmx - 13, kmx + 2]
    const int cbase = kmx + 3 - SM_K;            // table  [kmx - 61, kmx + 2]
    // the window must sit in pass 1's safe range (fl(x*y) normal, 2^(52-e) finite)
    // and the table inside the key range; otherwise everything is handed over
    const bool bad = kmx < 0 || base < P1_SAFE_LO || base > P1_SAFE_HI || cbase < 0 || cbase + SM_K > KEYS;
    const int kbias = KOFF - 2046 - base;
    ulonglong2* __restrict__ my = S.priv + tid;

    // ---- every element of this thread into its slot or table key
    uint32_t zc = 0, nf = 0;
    bool oor = false;
    if (!bad) {
        for (int64_t i = i0; i < n; i += stride) {
            double xv[2] = {cx[0], cx[1]}, yv[2] = {cy[0], cy[1]};
            const bool ok[2] = {cok[0], cok[1]};
            cok[0] = cok[1] = false;
            if (i + stride < n) sm_load2<NORM, VEC>(x, y, n, i + stride, cx, cy, cok);   // next pair in flight
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (!ok[k]) continue;
                const uint32_t hx = (uint32_t)(dbits(xv[k]) >> 32), hy = (uint32_t)(dbits(yv[k]) >> 32);
                const uint32_t fx = (hx >> 20) & 0x7FFu, fy = (hy >> 20) & 0x7FFu;
                const uint32_t esum = fx + fy;
                const int rel = (int)esum + kbias;
                if ((max(fx - 1u, fy - 1u) < 0x7FEu) & ((unsigned)rel < (unsigned)P1_W)) {
                    // DOUBLE units fl(x*y) 2^(52-e) and the exact SINGLE / HALF units (pass 1's full loop)
                    const double scale = __hiloint2double((int)((3121u - esum) << 20), 0);
                    const long long kd = __double2ll_rn(__dmul_rn(__dmul_rn(xv[k], yv[k]), scale));
                    const uint64_t bx = dbits(xv[k]), by = dbits(yv[k]);
                    int32_t ks, kh;
                    exact_variants_signed(bitsd((bx & 0x800FFFFFFFFFFFFFull) | 0x3FF0000000000000ull),
                                          bitsd((by & 0x800FFFFFFFFFFFFFull) | 0x3FF0000000000000ull), ks, kh);
                    ulonglong2* slot = my + rel * SM_T;
                    ulonglong2 v = *slot;
                    v.x += (unsigned long long)kd;
                    v.y += (unsigned long long)(((long long)ks << 29) + ((long long)kh << 8) + 1);
                    *slot = v;                   // <= 32 elements per thread: the 8-bit count never wraps
                } else {
                    oor |= sm_cold(S, cbase, xv[k], yv[k], zc, nf);
                }
            }
        }
    }
    {
        const unsigned long long z = __reduce_add_sync(0xffffffffu, zc), f = __reduce_add_sync(0xffffffffu, nf);
        const bool o = __any_sync(0xffffffffu, oor);
        if (lane == 0) {
            if (z) atomicAdd(&S.zc, z);
            if (f) atomicAdd(&S.nf, f);
            if (o) S.oor = 1;
        }
    }
    __syncthreads();
    phase(2);
    // ---- this CTA's per-key totals: table limbs, plus the window slots (one warp per window key)
    if (tid < SM_K) {
        const int j = tid;
        S.tcnt[j] = S.c[0][j];
        S.td[j] = (__int128)S.c[1][j] + ((__int128)S.c[2][j] << 14) + ((__int128)S.c[3][j] << 28) +
                  ((__int128)(int32_t)S.c[4][j] << 42);
        S.tsum[j] = (long long)S.c[5][j] + ((long long)(int32_t)S.c[6][j] << 14);
        S.thalf[j] = (long long)(int32_t)S.c[7][j];
    }
    __syncthreads();
    {
        // slot D < 32 * 2^54 per thread: its low 32 bits and its signed rest summed
        // apart (no carry chain), D = hi 2^32 + lo once at the end
        static_assert(P1_W % (SM_T / 32) == 0, "window keys per warp");
#pragma unroll 1
        for (int r = tid >> 5; r < P1_W; r += SM_T / 32) {   // warp w sums window keys w, w + 8
        unsigned long long dlo = 0;
        long long dhi = 0, ss = 0, hs = 0, cs = 0;
#pragma unroll 4
        for (int i = lane; i < SM_T; i += 32) {
            const ulonglong2 v = S.priv[r * SM_T + i];
            dlo += v.x & 0xFFFFFFFFull;
            dhi += (long long)v.x >> 32;
            const long long w = (long long)v.y;
            const long long c = w & 0xFF;
            const long long w1 = (w - c) >> 8;
            const long long h = ((w1 & 0x1FFFFF) ^ 0x100000) - 0x100000;
            cs += c; hs += h; ss += (w1 - h) >> 21;
        }
        for (int o = 16; o; o >>= 1) {
            dlo += __shfl_xor_sync(0xffffffffu, dlo, o);      // < 256 * 8 * 2^32: no wrap
            dhi += __shfl_xor_sync(0xffffffffu, dhi, o);
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
            hs += __shfl_xor_sync(0xffffffffu, hs, o);
        }
        cs = __reduce_add_sync(0xffffffffu, (unsigned)cs);
        const int j = base + r - cbase;          // the window lies inside the table
        if (lane == 0 && !bad && cs) {
            S.tcnt[j] += (unsigned long long)cs;
            S.td[j] += ((__int128)dhi << 32) + (__int128)dlo;
            S.tsum[j] += ss;
            S.thalf[j] += hs;
        }
        }
    }
    // ---- every CTA pushes its totals into CTA 0 (distributed shared memory stores,
    // no round trips), CTA 0 sums them and decides
    __syncthreads();
    phase(3);
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    {
        SmShared* R0 = cl.map_shared_rank(&S, 0);
        if (tid < SM_K) {
            const int j = tid;
            R0->rd[rank][j] = S.td[j];
            R0->rs[rank][j] = S.tsum[j];
            R0->rh[rank][j] = S.thalf[j];
            R0->rc[rank][j] = S.tcnt[j];
        } else if (tid == SM_K) {
            R0->rzc[rank] = S.zc;
            R0->rnf[rank] = S.nf;
            R0->roor[rank] = S.oor;
        }
    }
    cl.sync();
    if (rank == 0) {
        if (tid < SM_K) {
            const int j = tid;
            __int128 d = 0;
            long long a = 0, h = 0;
            unsigned long long c = 0;
#pragma unroll
            for (int q = 0; q < CL; ++q) { d += S.rd[q][j]; a += S.rs[q][j]; h += S.rh[q][j]; c += S.rc[q][j]; }
            S.td[j] = d; S.tsum[j] = a; S.thalf[j] = h; S.tcnt[j] = c;
        } else if (tid == SM_K) {
            unsigned long long z = 0, f = 0;
            int o = 0;
#pragma unroll
            for (int q = 0; q < CL; ++q) { z += S.rzc[q]; f += S.rnf[q]; o |= S.roor[q]; }
            S.zc = z; S.nf = f; S.oor = o;
        }
        __syncthreads();
        if (tid < 32) {
            const bool p0 = S.tcnt[lane] != 0, p1 = S.tcnt[lane + 32] != 0;
            const unsigned long long P = (unsigned long long)__ballot_sync(0xffffffffu, p0) |
                                         ((unsigned long long)__ballot_sync(0xffffffffu, p1) << 32);
            if (lane == 0) {
                S.kmin = P ? cbase + __ffsll((long long)P) - 1 : 0;
                S.kmax = P ? cbase + 63 - __clzll((long long)P) : -1;
                S.decision = (bad || S.oor || !P) ? 2 : 1;
            }
        }
        __syncthreads();
    }
    phase(4);
    cl.sync();
    const int decision = cl.map_shared_rank(&S, 0)->decision;
    phase(5);
    if (decision == 1) {
        // ---- common case: CTA 0's first warp scores and finalizes (score_warp over shared memory)
        if (rank == 0) {
            if (tid < 32) {
                const int need = score_warp(SmallSrc{&S, cbase}, A, lut_bin, lut_p2, meta, res, bins, n, cfg, S.kmin,
                                            S.kmax, ts0, (long long)S.nf, (long long)S.zc, 0ll, S.sval, S.bup,
                                            S.bprec);
                if (lane == 0) S.post = need;                        // a pass 2 reads the global regions
            }
            __syncthreads();
            if (S.post) {
                // (early termination below input_mu 52: HALF / SINGLE products of keys under
                // the bin's upper) -- hand the totals to k_score / k_pass2 through regions A / B
                ulonglong2* z = reinterpret_cast<ulonglong2*>(A);
                const int64_t n16 = (BYTES_A + BYTES_B + BYTES_LOCAL) / 16;
                for (int64_t i = tid; i < n16; i += SM_T) z[i] = make_ulonglong2(0ull, 0ull);
                __syncthreads();
                if (tid < SM_K && S.tcnt[tid]) push_key(A, B, cbase + tid, S.tcnt[tid], S.td[tid], S.tsum[tid], S.thalf[tid]);
                if (tid == SM_K) {
                    if (S.zc) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_ZERO), S.zc);
                    if (S.nf) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_NONFINITE), S.nf);
                    ws_stamps(A)[0] = ts0;
                }
                __syncthreads();
                if (tid == 0) A[A_SMALL] = 2;
            } else if (tid == 0) {
                A[A_SMALL] = 1;
            }
            phase(6);
        }
    } else {
        // ---- hand over: zero the exchange regions, add what this path kept, push the rest
        ulonglong2* z = reinterpret_cast<ulonglong2*>(A);     // regions A, B, local are contiguous
        const int64_t n16 = (BYTES_A + BYTES_B + BYTES_LOCAL) / 16;
        for (int64_t i = (int64_t)rank * SM_T + tid; i < n16; i += (int64_t)CL * SM_T)
            z[i] = make_ulonglong2(0ull, 0ull);
        __threadfence();
        cl.sync();
        if (rank == 0 && !bad) {
            if (tid < SM_K && S.tcnt[tid]) {
                const int j = tid;
                const __int128 D = S.td[j];
                push_key(A, B, cbase + j, S.tcnt[j], D, S.tsum[j], S.thalf[j]);
            }
            if (tid == SM_K) {
                if (S.zc) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_ZERO), S.zc);
                if (S.nf) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_NONFINITE), S.nf);
            }
        }
        // out-of-table elements (all of them when nothing was kept), with pass 1's global path
        uint32_t zc2 = 0, nf2 = 0;
        for (int64_t i = i0; i < n; i += stride) {
            double xv[2], yv[2];
            bool ok[2];
            sm_load2<NORM, VEC>(x, y, n, i, xv, yv, ok);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (!ok[k]) continue;
                bool take = bad;
                if (!bad) {
                    const uint64_t bx = dbits(xv[k]), by = dbits(yv[k]);
                    const bool special = ((bx >> 52) & 0x7FF) == 0x7FF || ((by >> 52) & 0x7FF) == 0x7FF ||
                                         xv[k] == 0.0 || yv[k] == 0.0;
                    if (!special) {
                        const int e = flexp_bits(bx) + flexp_bits(by);
                        const uint64_t pb = dbits(__dmul_rn(xv[k], yv[k]));
                        take = (unsigned)(e + KOFF - cbase) >= (unsigned)SM_K || ((pb >> 52) & 0x7FF) == 0x7FF;
                    }
                }
                if (take) sm_global(A, B, xv[k], yv[k], bad, zc2, nf2);
            }
        }
        const unsigned long long z2 = __reduce_add_sync(0xffffffffu, zc2), f2 = __reduce_add_sync(0xffffffffu, nf2);
        if (lane == 0) {
            if (z2) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_ZERO), z2);
            if (f2) atomicAdd(reinterpret_cast<unsigned long long*>(A + A_NONFINITE), f2);
        }
        if (rank == 0 && tid == 0) {
            A[A_SMALL] = 2;
            ws_stamps(A)[0] = ts0;
        }
    }
    cl.sync();                                   // CTA 0's shared memory stays readable until everyone is done
    phase(7);
}
