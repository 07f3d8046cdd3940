// qdot_order.cu -- member order of the bins on the device.
//
// 1. Stable counting-sort scatter (binning.py:46-55, 88-116, 197, 218, 270).
//    The reference materialises `order` = nonzero indices sorted by (exponent
//    sum, index) and slices it per bin; ranged / split bins np.sort their
//    slice, so every Bin.indices is ascending in index, zero_idx too
//    (floatbits.py:74-76).  Here each element gets a slot -- 0 for an exact-zero
//    product, 1 + bin id otherwise (the score kernel's key -> bin LUT) -- and
//    the elements of each wanted slot are written in index order:
//      k_ord_count   warp per segment: per-slot counts of the segment
//                    (match_any groups, a per-warp shared-memory table)
//      k_ord_scan    CTA per slot: exclusive scan over the segments
//      k_ord_base    1 CTA: slot bases (exclusive scan of the slot totals)
//      k_ord_scatter warp per segment: cursor table = base + segment prefix,
//                    rank inside the 32-element step from the match mask
//    Counts live in int64[slots][segments] (slot-major: the scan reads it
//    coalesced); the segment length grows with the slot count so the table
//    stays under ORD_TABLE_MAX entries.
//
// 2. Ordered HALF sums (emulate.py:150-151).  The reference sums a HALF bin's
//    fp16 products sequentially in fp32, in ascending index order.  The main
//    pipeline rounds the exact sum once, which equals that sequential sum
//    unless partial sums can leave fp32's exact range -- finalize flags such
//    bins (qdot_bin.flags bit 0).  For them, k_half_seq replays the fp32 chain
//    in index order from the member list above (a warp per bin; a 32-element
//    step is taken in one go when every exact partial sum of the step is an
//    fp32 number, else element by element), and k_half_apply rescales those
//    bins (math.ldexp semantics) and re-folds the result (emulate.py:157-163).
//    The chain carries an fp32 start value per bin, so contiguous shards on
//    several ranks run it one after another (dist.py).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "qdot_common.cuh"

namespace qd {
int report_cuda_error(cudaError_t e, const char* where);
}

using namespace qd;

namespace {

constexpr int ORD_WARPS = 4;                          // warps per CTA (count / scatter)
constexpr int64_t ORD_TABLE_MAX = 1ll << 25;           // count-table entries (int64)
constexpr int ORD_SEG_MIN = 4096;                      // elements per segment, at least
constexpr int ORD_SCAN_T = 1024;
constexpr size_t ORD_SMEM_OPTIN = (size_t)ORD_WARPS * (QDOT_KEYS + 1) * 8;   // 134 KB

struct OrdGeom {
    int64_t seg_len, nseg;
    int slots;
};

OrdGeom ord_geom(int64_t n, int32_t n_bins) {
    OrdGeom g;
    g.slots = n_bins + 1;
    int64_t want = (n * (int64_t)g.slots + ORD_TABLE_MAX - 1) / ORD_TABLE_MAX;
    int64_t sl = want > ORD_SEG_MIN ? want : ORD_SEG_MIN;
    g.seg_len = (sl + 31) / 32 * 32;
    g.nseg = n > 0 ? (n + g.seg_len - 1) / g.seg_len : 0;
    return g;
}

// scratch: want[slots] (uint8, 16-aligned) | totals[slots] | base[slots+1] | counts[slots * nseg]
struct OrdScratch {
    uint8_t* want;
    int64_t* totals;
    int64_t* base;
    int64_t* counts;
    size_t bytes;
};

inline size_t al16(size_t b) { return (b + 15) / 16 * 16; }

OrdScratch ord_scratch(void* p, const OrdGeom& g) {
    OrdScratch s;
    char* c = static_cast<char*>(p);
    size_t off = 0;
    s.want = reinterpret_cast<uint8_t*>(c + off); off += al16((size_t)g.slots);
    s.totals = reinterpret_cast<int64_t*>(c + off); off += al16(8 * (size_t)g.slots);
    s.base = reinterpret_cast<int64_t*>(c + off); off += al16(8 * (size_t)(g.slots + 1));
    s.counts = reinterpret_cast<int64_t*>(c + off); off += 8 * (size_t)g.slots * (size_t)g.nseg;
    s.bytes = off;
    return s;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// slot of element i: 0 for an exact-zero product, 1 + bin id, or -1 (unwanted / past n)
template <bool NORM>
__device__ __forceinline__ int elem_slot(const double* __restrict__ x, const double* __restrict__ y, int64_t i,
                                         int64_t n, const int32_t* __restrict__ lut_bin,
                                         const uint8_t* __restrict__ want) {
    if (i >= n) return -1;
    const double a = x[i];
    const double b = NORM ? a : y[i];
    int s = 0;
    if (a != 0.0 && b != 0.0) s = 1 + lut_bin[flexp_bits(dbits(a)) + flexp_bits(dbits(b)) + KOFF];
    return (want == nullptr || want[s]) ? s : -1;
}

template <bool NORM>
__global__ void __launch_bounds__(ORD_WARPS * 32)
k_ord_count(const double* __restrict__ x, const double* __restrict__ y, int64_t n, const int32_t* __restrict__ lut_bin,
            const uint8_t* __restrict__ want, int slots, int64_t seg_len, int64_t nseg, int64_t* __restrict__ counts) {
    extern __shared__ long long ord_tbl[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long* tbl = ord_tbl + (size_t)w * slots;
    const int64_t gw = (int64_t)blockIdx.x * ORD_WARPS + w, nw = (int64_t)gridDim.x * ORD_WARPS;
    for (int64_t seg = gw; seg < nseg; seg += nw) {
        for (int s = lane; s < slots; s += 32) tbl[s] = 0;
        __syncwarp();
        const int64_t lo = seg * seg_len, hi = lo + seg_len < n ? lo + seg_len : n;
        for (int64_t i0 = lo; i0 < hi; i0 += 32) {
            const int s = elem_slot<NORM>(x, y, i0 + lane, hi, lut_bin, want);
            const unsigned grp = __match_any_sync(0xffffffffu, s);
            if (s >= 0 && (grp & lanemask_lt()) == 0) tbl[s] += __popc(grp);   // group leader
            __syncwarp();
        }
        for (int s = lane; s < slots; s += 32) counts[(int64_t)s * nseg + seg] = tbl[s];
        __syncwarp();
    }
}

// CTA per slot: exclusive scan over its segments in place, slot total out
__global__ void __launch_bounds__(ORD_SCAN_T)
k_ord_scan(int64_t* __restrict__ counts, int64_t nseg, int64_t* __restrict__ totals) {
    __shared__ long long warp_sum[ORD_SCAN_T / 32];
    __shared__ long long carry;
    int64_t* row = counts + (int64_t)blockIdx.x * nseg;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nseg; b0 += ORD_SCAN_T) {
        const int64_t i = b0 + tid;
        const long long v = i < nseg ? row[i] : 0;
        long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) warp_sum[w] = inc;
        __syncthreads();
        if (w == 0) {
            long long ws = warp_sum[lane];
            long long wi = ws;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            warp_sum[lane] = wi - ws;                 // exclusive prefix of the warp totals
        }
        __syncthreads();
        const long long c0 = carry;
        if (i < nseg) row[i] = c0 + warp_sum[w] + inc - v;
        __syncthreads();
        if (tid == ORD_SCAN_T - 1) carry = c0 + warp_sum[w] + inc;
        __syncthreads();
    }
    if (tid == 0) totals[blockIdx.x] = carry;
}

// 1 CTA: base[s] = exclusive prefix of totals, base[slots] = total
__global__ void __launch_bounds__(ORD_SCAN_T)
k_ord_base(const int64_t* __restrict__ totals, int slots, int64_t* __restrict__ base) {
    __shared__ long long warp_sum[ORD_SCAN_T / 32];
    __shared__ long long carry;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int b0 = 0; b0 < slots; b0 += ORD_SCAN_T) {
        const int i = b0 + tid;
        const long long v = i < slots ? totals[i] : 0;
        long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) warp_sum[w] = inc;
        __syncthreads();
        if (w == 0) {
            long long ws = warp_sum[lane];
            long long wi = ws;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            warp_sum[lane] = wi - ws;
        }
        __syncthreads();
        const long long c0 = carry;
        if (i < slots) base[i] = c0 + warp_sum[w] + inc - v;
        __syncthreads();
        if (tid == ORD_SCAN_T - 1) carry = c0 + warp_sum[w] + inc;
        __syncthreads();
    }
    if (tid == 0) base[slots] = carry;
}

template <bool NORM>
__global__ void __launch_bounds__(ORD_WARPS * 32)
k_ord_scatter(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
              const int32_t* __restrict__ lut_bin, const uint8_t* __restrict__ want, int slots, int64_t seg_len,
              int64_t nseg, const int64_t* __restrict__ counts, const int64_t* __restrict__ base,
              int64_t* __restrict__ order) {
    extern __shared__ long long ord_tbl[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long* tbl = ord_tbl + (size_t)w * slots;
    const int64_t gw = (int64_t)blockIdx.x * ORD_WARPS + w, nw = (int64_t)gridDim.x * ORD_WARPS;
    for (int64_t seg = gw; seg < nseg; seg += nw) {
        for (int s = lane; s < slots; s += 32) tbl[s] = base[s] + counts[(int64_t)s * nseg + seg];
        __syncwarp();
        const int64_t lo = seg * seg_len, hi = lo + seg_len < n ? lo + seg_len : n;
        for (int64_t i0 = lo; i0 < hi; i0 += 32) {
            const int64_t i = i0 + lane;
            const int s = elem_slot<NORM>(x, y, i, hi, lut_bin, want);
            const unsigned grp = __match_any_sync(0xffffffffu, s);
            const unsigned below = grp & lanemask_lt();
            if (s >= 0) order[tbl[s] + __popc(below)] = i;
            __syncwarp();
            if (s >= 0 && below == 0) tbl[s] += __popc(grp);
            __syncwarp();
        }
    }
}

// want[1 + b] = bin b is a HALF bin flagged order-sensitive (zero slot never)
__global__ void k_half_want(const qdot_bin* __restrict__ bins, int n_bins, uint8_t* __restrict__ want,
                            float* __restrict__ s_io) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s <= n_bins; s += gridDim.x * blockDim.x) {
        uint8_t w = 0;
        if (s > 0) {
            const qdot_bin& b = bins[s - 1];
            w = (b.precision == QDOT_HALF && (b.flags & 1)) ? 1 : 0;
            s_io[s - 1] = 0.0f;
        }
        want[s] = w;
    }
}

// emulate.py:137-146 for one HALF member of a bin with upper bound u: sx =
// x 2^-ex, sy = y 2^(ex-u) (= the mantissa of y times 2^(e-u)), both rounded
// to fp16, multiplied in fp16; returned as the fp32 value the sum adds
__device__ __forceinline__ float half_product(double a, double b, long long u) {
    const uint64_t bx = dbits(a), by = dbits(b);
    const long long e = (long long)flexp_bits(bx) + flexp_bits(by);
    long long d = u - e;                                      // >= 0 for a member
    if (d > 255) d = 255;                                     // fp16 of 2^-d y-mantissa is 0 past 2^-25 anyway
    double mx = bitsd(mant_bits(bx) | (bx & 0x8000000000000000ull));
    double sy = bitsd(mant_bits(by) | (by & 0x8000000000000000ull)) * bitsd((uint64_t)(1023 - d) << 52);
    const __half p = __hmul(__double2half(mx), __double2half(sy));
    return __half2float(p);
}

// exact fp32 representability of t * 2^-24 (t an integer, |t| < 2^62)
__device__ __forceinline__ bool f32_exact(long long t) {
    unsigned long long a = t < 0 ? (unsigned long long)(-t) : (unsigned long long)t;
    if (!a) return true;
    a >>= __ffsll((long long)a) - 1;
    return a < (1ull << 24);
}

// a warp per wanted bin: s = s_io[b]; for members in index order s = fp32(s + p)
template <bool NORM>
__global__ void __launch_bounds__(32)
k_half_seq(const double* __restrict__ x, const double* __restrict__ y, const qdot_bin* __restrict__ bins,
           const uint8_t* __restrict__ want, const int64_t* __restrict__ order, const int64_t* __restrict__ base,
           float* __restrict__ s_io) {
    const int b = blockIdx.x;                 // bin id; slot b + 1
    if (!want[b + 1]) return;
    const int lane = threadIdx.x;
    const long long u = bins[b].upper;
    const int64_t lo = base[b + 1], hi = base[b + 2];
    float s = s_io[b];
    // software pipeline: the next step's loads are issued before this step's chain
    double na = 0.0, nb = 0.0;
    if (lo + lane < hi) {
        const int64_t i = order[lo + lane];
        na = x[i];
        nb = NORM ? na : y[i];
    }
    for (int64_t j0 = lo; j0 < hi; j0 += 32) {
        const int cnt = hi - j0 < 32 ? (int)(hi - j0) : 32;
        const double a = na, bb = nb;
        if (j0 + 32 + lane < hi) {
            const int64_t i = order[j0 + 32 + lane];
            na = x[i];
            nb = NORM ? na : y[i];
        }
        const float p = lane < cnt ? half_product(a, bb, u) : 0.0f;
        // fast step: every exact partial sum an fp32 number -> no rounding anywhere
        bool fast = fabsf(s) < 0x1p37f;
        long long T = 0;
        if (fast) {
            long long k = (long long)((double)p * 0x1p24);     // p is a multiple of 2^-24, |p| < 2^16
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, k, o);
                if (lane >= o) k += t;
            }
            T = (long long)((double)s * 0x1p24) + k;
            fast = __all_sync(0xffffffffu, f32_exact(T));
        }
        if (fast) {
            const long long t_last = __shfl_sync(0xffffffffu, T, 31);
            s = (float)((double)t_last * 0x1p-24);
        } else {
            for (int j = 0; j < cnt; ++j) s = __fadd_rn(s, __shfl_sync(0xffffffffu, p, j));
        }
    }
    if (lane == 0) s_io[b] = s;
}

// rescale the re-summed bins (math.ldexp semantics, emulate.py:154) and
// re-fold every bin value in ascending-upper order (emulate.py:157-163)
__global__ void __launch_bounds__(32)
k_half_apply(qdot_bin* __restrict__ bins, const uint8_t* __restrict__ want, const float* __restrict__ s_io,
             qdot_result* __restrict__ res) {
    if (threadIdx.x != 0) return;
    const int nb = res->n_bins;
    int ovf = 0;
    double sum = 0.0, c = 0.0;
    for (int b = 0; b < nb; ++b) {
        double v = bins[b].value;
        if (want[b + 1]) {
            int o = 0;
            v = ldexp_rn((double)s_io[b], bins[b].upper, &o);
            ovf |= o;
            bins[b].value = v;
            bins[b].flags |= 2;                    // re-summed in index order
        }
        const double t = __dadd_rn(sum, v);
        if (fabs(sum) >= fabs(v)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(sum, t), v));
        else c = __dadd_rn(c, __dadd_rn(__dsub_rn(v, t), sum));
        sum = t;
    }
    res->value = (sum - sum == 0.0) ? __dadd_rn(sum, c) : sum;
    if (ovf && res->status == QDOT_OK) res->status = QDOT_ERR_OVERFLOW;
    res->half_order_sensitive = 2;                 // resolved
}

int ord_grid(int64_t nseg) {
    const int64_t cap = (int64_t)device_sm_count() * 8;
    int64_t g = (nseg + ORD_WARPS - 1) / ORD_WARPS;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

int fail(cudaError_t e, const char* where) { return qd::report_cuda_error(e, where); }

template <bool NORM>
cudaError_t run_order(const double* x, const double* y, int64_t n, const int32_t* lut_bin, const uint8_t* want,
                      const OrdGeom& g, const OrdScratch& sc, int64_t* base, int64_t* order, cudaStream_t st) {
    const size_t smem = (size_t)ORD_WARPS * g.slots * sizeof(long long);
    // opt in once per device to the largest table (any slot count fits)
    static KernelDevCache c_cnt, c_sct;
    kernel_occupancy(k_ord_count<NORM>, ORD_WARPS * 32, ORD_SMEM_OPTIN, c_cnt);
    kernel_occupancy(k_ord_scatter<NORM>, ORD_WARPS * 32, ORD_SMEM_OPTIN, c_sct);
    const int grid = ord_grid(g.nseg);
    if (g.nseg > 0) {
        k_ord_count<NORM><<<grid, ORD_WARPS * 32, smem, st>>>(x, y, n, lut_bin, want, g.slots, g.seg_len, g.nseg,
                                                             sc.counts);
        k_ord_scan<<<g.slots, ORD_SCAN_T, 0, st>>>(sc.counts, g.nseg, sc.totals);
    } else {
        cudaMemsetAsync(sc.totals, 0, 8 * (size_t)g.slots, st);
    }
    k_ord_base<<<1, ORD_SCAN_T, 0, st>>>(sc.totals, g.slots, base);
    if (g.nseg > 0)
        k_ord_scatter<NORM><<<grid, ORD_WARPS * 32, smem, st>>>(x, y, n, lut_bin, want, g.slots, g.seg_len, g.nseg,
                                                               sc.counts, base, order);
    return cudaGetLastError();
}

}  // namespace

extern "C" {

size_t qdot_b200_order_scratch_bytes(int64_t n, int32_t n_bins) {
    if (n < 0 || n_bins < 0 || n_bins > QDOT_KEYS) return 0;
    const OrdGeom g = ord_geom(n, n_bins);
    return ord_scratch(nullptr, g).bytes;
}

int qdot_b200_bin_order(const double* x, const double* y, int64_t n, int norm, const int32_t* lut_bin,
                        int32_t n_bins, const uint8_t* want, int64_t* bin_start, int64_t* order, void* scratch,
                        size_t scratch_bytes, void* stream) {
    if (n < 0 || n_bins < 0 || n_bins > QDOT_KEYS || !bin_start || !scratch) return QDOT_ERR_ARG;
    if (n > 0 && (!x || (!norm && !y) || !lut_bin || !order)) return QDOT_ERR_ARG;
    const OrdGeom g = ord_geom(n, n_bins);
    const OrdScratch sc = ord_scratch(scratch, g);
    if (scratch_bytes < sc.bytes || (size_t)ORD_WARPS * g.slots * 8 > ORD_SMEM_OPTIN) return QDOT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = norm ? run_order<true>(x, x, n, lut_bin, want, g, sc, bin_start, order, st)
                         : run_order<false>(x, y, n, lut_bin, want, g, sc, bin_start, order, st);
    return e == cudaSuccess ? QDOT_OK : fail(e, "bin_order");
}

int qdot_b200_half_ordered(const double* x, const double* y, int64_t n, int norm, void* ws, int32_t n_bins,
                           int64_t* order, int64_t order_len, float* chain, void* scratch, size_t scratch_bytes,
                           int stage, void* stream) {
    if (n < 0 || n_bins < 0 || n_bins > QDOT_KEYS || !ws || !scratch || (n_bins > 0 && !chain)) return QDOT_ERR_ARG;
    if (n > 0 && (!x || (!norm && !y))) return QDOT_ERR_ARG;
    const OrdGeom g = ord_geom(n, n_bins);
    const OrdScratch sc = ord_scratch(scratch, g);
    if (scratch_bytes < sc.bytes) return QDOT_ERR_ARG;
    const WsPtrs w = ws_ptrs(ws);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    if (stage & 1) {    // want mask + member order of the flagged bins, s_io = 0
        k_half_want<<<(n_bins + 256) / 256, 256, 0, st>>>(w.bins, n_bins, sc.want, chain);
        e = norm ? run_order<true>(x, x, n, w.lut_bin, sc.want, g, sc, sc.base, order, st)
                 : run_order<false>(x, y, n, w.lut_bin, sc.want, g, sc, sc.base, order, st);
        if (e != cudaSuccess) return fail(e, "half_ordered/order");
    }
    (void)order_len;
    if ((stage & 2) && n_bins > 0) {   // the fp32 chains (start values in s_io)
        if (norm) k_half_seq<true><<<n_bins, 32, 0, st>>>(x, x, w.bins, sc.want, order, sc.base, chain);
        else k_half_seq<false><<<n_bins, 32, 0, st>>>(x, y, w.bins, sc.want, order, sc.base, chain);
    }
    if (stage & 4) k_half_apply<<<1, 32, 0, st>>>(w.bins, sc.want, chain, w.result);
    e = cudaGetLastError();
    return e == cudaSuccess ? QDOT_OK : fail(e, "half_ordered");
}

}  // extern "C"
