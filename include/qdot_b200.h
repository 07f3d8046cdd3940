/*
 * qdot_b200.h -- C ABI of the B200-native qdot hot path (sm_100a).
 *
 * The reference (qdot 0.1.0, /root/reference/pkg/src/qdot) has no FFI: its
 * hot path is the Python function
 *
 *     qdot(x, y, cfg: ToleranceConfig, strategy=None, reference=None) -> QdotReport
 *                                                              (kernel.py:179-240)
 *
 * whose internal seam is kernel.py:199-202 (select_parameters + the bin_dot
 * loop + qdot_accumulate).  Every entry point below replaces one stage of
 * that seam; the Python package paper_2105_00115_b200 (the host-side mirror
 * of the reference interface) drives them through ctypes, and any other host
 * language can bind the same symbols.
 *
 * Conventions
 *  - Plain pointers and sizes only.  `stream` is a cudaStream_t passed as
 *    void* (NULL = legacy default stream).  x, y are DEVICE pointers to
 *    float64 unless the function name ends in _host.
 *  - `ws` is a caller-owned device workspace of qdot_b200_workspace_bytes()
 *    bytes (256-byte aligned).  All calls are stream-ordered; only
 *    qdot_b200_fetch / qdot_b200_dot / qdot_b200_dot_host synchronise.
 *  - Return value: a qdot_status.  Device-detected conditions (non-finite
 *    input, HALF/SINGLE overflow, eps underflow) are reported in
 *    qdot_result.status after qdot_b200_fetch; the Python layer maps them to
 *    the reference's exception types (ValueError / OverflowError).
 *  - No CPU fallback exists: without a CUDA device every compute entry point
 *    returns QDOT_ERR_CUDA.
 */
#ifndef QDOT_B200_H
#define QDOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QDOT_B200_VERSION 1

/* Exponent sums of two finite doubles lie in [-2148, 2046] (floatbits.py:10-14). */
#define QDOT_KEYS 4195
#define QDOT_KEY_OFFSET 2148

typedef enum {
    QDOT_OK = 0,
    QDOT_ERR_NONFINITE = 1, /* floatbits.py:70-71  ValueError("inputs must be finite")          */
    QDOT_ERR_OVERFLOW = 2,  /* emulate.py:147-148 / math.ldexp in emulate.py:154 -> OverflowError */
    QDOT_ERR_ARG = 3,       /* bad config / strategy (scoring.py:72-79, binning.py:131,142)       */
    QDOT_ERR_CUDA = 4,      /* no device / launch failure                                         */
    QDOT_ERR_EPS = 5        /* scoring.py:84-85 floor_log2(eps_eff) of 0 -> ValueError            */
} qdot_status;

/* PrecisionLevel (scoring.py:15-41); values order coarse -> fine */
typedef enum { QDOT_PERFORATE = 0, QDOT_HALF = 1, QDOT_SINGLE = 2, QDOT_DOUBLE = 3 } qdot_precision;

/* ExactBinning / RangedBinning(width) / BinSplitting(levels)  (binning.py:119-144) */
typedef enum { QDOT_STRATEGY_EXACT = 0, QDOT_STRATEGY_RANGED = 1, QDOT_STRATEGY_SPLIT = 2 } qdot_strategy;

/* ToleranceConfig (scoring.py:59-79) + the strategy argument of qdot() */
typedef struct {
    double epsilon;          /* (0, 2^60]                                      */
    int32_t split;           /* 0 = SplitMode.NONE, 1 = SplitMode.PER_BIN       */
    int32_t input_mu;        /* 52, 23 or 10                                    */
    int32_t strategy;        /* qdot_strategy                                   */
    int32_t reserved;        /* pass-1 speed knob: see qdot_b200_pass1          */
    int64_t strategy_param;  /* width (ranged, >= 1) or levels (split, >= 0)    */
} qdot_config;

/* One scored bin: Bin (binning.py:168-177) + its bin_dot value (emulate.py:116-154) */
typedef struct {
    int64_t lower;       /* bin is the exponent-sum interval (lower, upper]        */
    int64_t upper;
    int64_t cardinality; /* M: number of nonzero products in the bin               */
    int64_t score;       /* bin_score (scoring.py:96-105)                          */
    int32_t precision;   /* qdot_precision (precision_of, scoring.py:108-123)      */
    int32_t first_key;   /* first / last present exponent-sum key (e + 2148)       */
    int32_t last_key;
    int32_t flags;       /* bit0: HALF bin whose fp32 sequential sum in the
                            reference is not provably exact (its order matters);
                            bit1: that sum was replayed in index order by
                            qdot_b200_half_ordered (value bit-exact again)        */
    double value;        /* per-bin value (already scaled by 2^upper)              */
} qdot_bin;

/* Everything QdotReport (kernel.py:136-168) needs besides the host-side fsum bounds */
typedef struct {
    double value;            /* qdot_accumulate over bins (emulate.py:157-163)   */
    double eps_eff;          /* scoring.py:193                                    */
    int64_t n;               /* elements processed                                */
    int64_t nnz;             /* nonzero products                                  */
    int64_t zero_count;      /* exact-zero products (ParameterSet.zero_idx.size)  */
    int64_t counts[4];       /* component counts by precision, zeros -> PERFORATE */
    int32_t status;          /* qdot_status detected on the device                */
    int32_t n_bins;
    int32_t e_min, e_max;    /* 0, 0 when degenerate                              */
    int32_t early_terminated;
    int32_t pass2_needed;    /* a second streaming pass was required              */
    int32_t half_order_sensitive; /* 1: some bin has flags bit0 (value pending the
                                     ordered replay); 2: replayed, value final    */
    int32_t select_ns;       /* device time: pass 1 start -> scoring done         */
    int32_t compute_ns;      /* device time: scoring done -> finalize done        */
    int32_t reserved[3];
} qdot_result;

/* Workspace regions, in bytes from the start of ws.  Region A (int64[a_len],
 * exponent histogram + zero count + non-finite count) must be summed across
 * ranks between pass1 and score; region B (int64[b_len], exact per-key partial
 * sums) must be summed across ranks between pass2 and finalize.  Both are
 * integer sums, so any reduction order gives bit-identical results. */
typedef struct {
    int64_t total_bytes;
    int64_t a_offset, a_len;
    int64_t b_offset, b_len;
    int64_t result_offset, result_bytes;
} qdot_ws_layout;

/* --- introspection --------------------------------------------------------- */
int qdot_b200_version(void);
const char* qdot_b200_status_string(int status);
/* message of the last CUDA failure on this host thread */
const char* qdot_b200_last_error(void);
size_t qdot_b200_workspace_bytes(void);
int qdot_b200_workspace_layout(qdot_ws_layout* out);
/* 0 on success; fills SM count and compute capability of the current device */
int qdot_b200_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* --- staged path (the seam kernel.py:199-202) -------------------------------- */
/* zero regions A and B: start of one qdot (per rank) */
int qdot_b200_begin(void* ws, void* stream);
/* pass 1 over n elements (accumulates; may be called per chunk/shard):
 * exponent preprocessing + exact exponent-sum histogram + exact per-key
 * DOUBLE partials and exact-binning HALF/SINGLE partials.
 * Replaces floatbits.exponent_preprocess (floatbits.py:57-93),
 * binning.sorted_bin_init's histogram (binning.py:102-106) and, for every
 * bin whose products do not depend on the partition, emulate.bin_dot.
 * cfg (may be NULL) and n_total (elements over all ranks) only steer the
 * per-CTA lean/full and cold-queue choices (speed, never results);
 * cfg->reserved bits 0-1: 0 auto, 1 lean, 2 full; bits 2-3: cold-element warp
 * queue 0 auto, 4 on, 8 off; bit 4 (16): force the 24-key wide lean window;
 * bit 5 (32): norm mode without its exponent-indexed lean loop; bits 6-7: that
 * loop's L2 prefetch distance, bits 8-9 its cache policy (tuning). */
int qdot_b200_pass1(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg,
                    int64_t n_total, void* ws, void* stream);
/* the whole single-device pipeline of one qdot on `stream` (no sync): for
 * 1 <= n <= 16384 with the exact strategy and cfg->reserved 0,
 * one thread-block-cluster launch that keeps every exact per-key partial in
 * distributed shared memory and scores / finalizes in place (qdot_b200_small),
 * then score_finalize and pass2_finalize, which return at once unless it
 * handed the call over; otherwise begin, pass1, score_finalize,
 * pass2_finalize.  Replaces kernel.qdot's body (kernel.py:179-240). */
int qdot_b200_enqueue(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                      void* stream);
int qdot_b200_small(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                    void* stream);
/* qdot_b200_enqueue for a workspace whose exchange regions are already zero
 * (no begin launch on the four-launch path) */
int qdot_b200_enqueue_zeroed(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg, void* ws,
                             void* stream);
int64_t qdot_b200_small_max(void);   /* qdot_b200_small's limit (131072) */
/* one-CTA scoring on the (reduced) histogram: partition, scores, precisions.
 * Replaces kernel.select_parameters' partition + scoring (kernel.py:59-72,
 * binning.py:191-284, scoring.py:126-216).  n_total = elements over all ranks. */
int qdot_b200_score(void* ws, int64_t n_total, const qdot_config* cfg, void* stream);
/* single-device form of qdot_b200_score: when no pass 2 is needed (the common
 * case) the same launch also runs finalize, and the later qdot_b200_pass2 /
 * qdot_b200_finalize calls return on the device at once.  Not for multi-rank
 * runs, whose finalize must follow the allreduce of region B. */
int qdot_b200_score_finalize(void* ws, int64_t n_total, const qdot_config* cfg, void* stream);
/* pass 2 (exits on the device unless score flagged it): scaled HALF/SINGLE
 * products for bins whose upper bound differs from the element's exponent
 * sum (ranged / split / early-terminated bins; emulate.py:137-153). */
int qdot_b200_pass2(const double* x, const double* y, int64_t n, int norm, void* ws, void* stream);
/* single-device form of pass 2 + finalize in one launch: pass 2 when score
 * flagged it, then the last CTA to finish finalizes (unless
 * qdot_b200_score_finalize already did).  Not for multi-rank runs. */
int qdot_b200_pass2_finalize(const double* x, const double* y, int64_t n, int norm, void* ws, void* stream);
/* per-bin values + ascending-upper Neumaier fold (emulate.py:154-163) */
int qdot_b200_finalize(void* ws, void* stream);
/* copy the result (and up to max_bins bins) to host memory; synchronises */
int qdot_b200_fetch(const void* ws, qdot_result* out, qdot_bin* bins, int32_t max_bins, void* stream);

/* --- one-call forms ----------------------------------------------------------- */
/* device-resident x, y: begin + pass1 + score + pass2 + finalize + fetch */
int qdot_b200_dot(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg,
                  void* ws, qdot_result* out, qdot_bin* bins, int32_t max_bins, void* stream);
/* pass 1 over HOST vectors (pageable or pinned): copies them into the caller's
 * device buffers dx, dy (n elements each) chunk by chunk while pass 1 consumes
 * each landed chunk on `stream`.  Pageable memory goes through the library's
 * pinned staging ring, filled by a pool of host threads (parallel memcpy)
 * while the DMA engine drains the previous buffer.  Returns when the host
 * memory has been read (pageable) / all copies are enqueued (pinned).
 * Replaces the np.ascontiguousarray hand-off of kernel.py:195-196 + pass 1. */
int qdot_b200_pass1_host(const double* hx, const double* hy, int64_t n, int norm, const qdot_config* cfg,
                         int64_t n_total, void* ws, double* dx, double* dy, void* stream);
/* host threads of the staging copy pool */
int qdot_b200_host_copy_threads(void);
/* host x, y: allocates device buffers, copies in, runs, copies the result out */
int qdot_b200_dot_host(const double* x, const double* y, int64_t n, int norm, const qdot_config* cfg,
                       qdot_result* out, qdot_bin* bins, int32_t max_bins);

/* --- batched qdot (BASELINE configs[3]: many independent short dots) -------- */
/* Row-status bits in info[4*r+3]. */
#define QDOT_BATCH_NONFINITE 1   /* ValueError for that row                                  */
#define QDOT_BATCH_OVERFLOW 2    /* OverflowError for that row                               */
#define QDOT_BATCH_EPS 4         /* floor_log2(eps_eff) ValueError                           */
#define QDOT_BATCH_GENERAL 8     /* not finished by the fused kernel: recompute the row with
                                    the single-vector path (keys spread over > 64
                                    exponents, DOUBLE overflow, len > 65536, ...)            */
#define QDOT_BATCH_EARLY 16      /* early-terminated row                                     */
#define QDOT_BATCH_HALF_ORDER 32 /* a HALF bin the reference sums order-sensitively          */
#define QDOT_BATCH_MAX_BINS 64   /* row stride of the per-row bin tables                     */
/* rows x len row-major (row stride ld >= len elements), one warp per row, one
 * HBM pass.  Device outputs: values[rows]; counts[4*rows] (PERFORATE incl.
 * zeros, HALF, SINGLE, DOUBLE); info[4*rows] = {n_bins, e_min, e_max, status}.
 * Equivalent to qdot(X[r], Y[r], cfg) per row (kernel.py:179-240). */
int qdot_b200_batched(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld, int norm,
                      const qdot_config* cfg, double* values, int64_t* counts, int32_t* info, void* stream);
/* the same, also writing each row's bin table (the reference's
 * QdotReport.params.bins per row, kernel.py:62-72): row r's info[4r] bins at
 * bins[r * QDOT_BATCH_MAX_BINS ...] (device memory, rows * 64 entries); rows
 * flagged QDOT_BATCH_GENERAL / _HALF_ORDER have no table (the caller reruns them). */
int qdot_b200_batched_bins(const double* X, const double* Y, int64_t rows, int64_t len, int64_t ld, int norm,
                           const qdot_config* cfg, double* values, int64_t* counts, int32_t* info, qdot_bin* bins,
                           void* stream);

/* --- lazy Bin.indices support (binning.py:174) ------------------------------- */
/* write the bin id of every element (-1 for exact-zero products) given a
 * device LUT of QDOT_KEYS int32 entries mapping exponent-sum key -> bin id
 * (built by the caller from the bin table: keys first_key..last_key -> bin) */
int qdot_b200_bin_ids(const double* x, const double* y, int64_t n, int norm, const int32_t* lut_bin,
                      int32_t* bin_ids, void* stream);

/* Stable counting-sort scatter: the members of every bin in ascending index
 * order, i.e. the reference's `order` slices (binning.py:46-55, 88-116; the
 * np.sort of ranged / split members, binning.py:218, 270) and zero_idx
 * (floatbits.py:74-76).  Slot 0 = exact-zero products, slot 1 + b = bin b
 * (lut_bin: exponent-sum key -> bin id).  want[slot] != 0 selects the slots
 * written (NULL: all).  Outputs: bin_start[n_bins + 2] (device int64: start
 * of each slot in `order`, bin_start[n_bins + 1] = total) and the indices.
 * scratch: device memory of qdot_b200_order_scratch_bytes(n, n_bins). */
size_t qdot_b200_order_scratch_bytes(int64_t n, int32_t n_bins);
int qdot_b200_bin_order(const double* x, const double* y, int64_t n, int norm, const int32_t* lut_bin,
                        int32_t n_bins, const uint8_t* want, int64_t* bin_start, int64_t* order, void* scratch,
                        size_t scratch_bytes, void* stream);
/* HALF bins the finalize flagged order-sensitive (qdot_bin.flags bit 0):
 * replay the reference's sequential fp32 sum in index order (emulate.py:150-151)
 * after the pipeline, on the workspace of that call.  stage bits: 1 = member
 * order of the flagged bins into `order` (order_len >= their total
 * cardinality) and zero start values; 2 = the fp32 chains from the start
 * values; 4 = rescale those bins (math.ldexp semantics, bin flags |= 2) and
 * re-fold the result (emulate.py:154-163; result.half_order_sensitive = 2).
 * chain: device float[n_bins], the running fp32 sum per bin (stage 1 zeroes
 * it, stage 2 continues from it, stage 4 reads it).  One device: stage 7.
 * Contiguous shards: 1, then 2 on every rank in rank order with the previous
 * rank's chain copied in, then 4 everywhere with the last rank's chain. */
int qdot_b200_half_ordered(const double* x, const double* y, int64_t n, int norm, void* ws, int32_t n_bins,
                           int64_t* order, int64_t order_len, float* chain, void* scratch, size_t scratch_bytes,
                           int stage, void* stream);

/* --- solver callers (apps.py: acg / apm) -------------------------------------- */
/* y = A x for a CSR matrix (int64 indptr[n_rows+1], int32 or int64 column
 * indices: index_bytes 4 or 8).  Each row is summed sequentially from +0.0 in
 * CSR order with separately rounded products, bit-identical to scipy's
 * csr_matvec used by SparseMatrix.matvec (apps.py:57-58).  indices, data and x
 * are only read through the row extents (may be NULL for an empty matrix). */
int qdot_b200_csr_spmv(int64_t n_rows, const int64_t* indptr, const void* indices, int index_bytes,
                       const double* data, const double* x, double* y, void* stream);
/* the same product from a sliced-ELL copy of the matrix (slices of 32 rows;
 * entry j of row r at slice_off[r / 32] + 32 j + r % 32; row_len[r] entries;
 * int32 column indices): coalesced loads, identical per-row summation order,
 * hence identical results. */
int qdot_b200_sell_spmv(int64_t n_rows, const int64_t* slice_off, const int32_t* row_len, const int32_t* cols,
                        const double* vals, const double* x, double* y, void* stream);
/* elementwise vector updates of the solvers (apps.py:216-220, 306-308), each
 * bit-identical to the numpy expression: op 0 out = a + s*b, op 1 out = a - s*b
 * (s*b rounded first), op 2 out = a / s (b unused).  out may alias a or b. */
int qdot_b200_vec_update(int64_t n, int op, const double* a, double s, const double* b, double* out,
                         void* stream);

/* device-scalar forms for solver iterations captured in CUDA graphs:
 * vec_update_dev reads s from device memory; solver_scalar runs one scalar
 * step on the qdot result in `ws` (which 0: alpha = st[0] / d, st[4] = d;
 * 1: beta = value / st[0], st[0] = value, st[3] = sqrt(value); 2: st[0] =
 * value, st[3] = sqrt(value)); publish_iter copies the 256-byte result headers
 * of ws_a and ws_b and st[0..7] to device-visible pinned host memory (576
 * bytes) and then writes an incremented sequence word at host + 576. */
int qdot_b200_vec_update_dev(int64_t n, int op, const double* a, const double* s_dev, const double* b, double* out,
                             void* stream);
int qdot_b200_solver_scalar(int which, const void* ws, double* st, void* stream);
int qdot_b200_publish_iter(const void* ws_a, const void* ws_b, const double* st, void* host, uint32_t* dev_seq,
                           void* stream);

/* --- exact dot product (verification oracle) --------------------------------- */
/* Correctly rounded x.y computed exactly on the device: the device form of
 * kernel.reference_dot (kernel.py:98-133) for checking qdot at sizes the host
 * cannot hold.  Every product is an exact integer mx*my * 2^(qx+qy); the pass
 * sums them per exponent in integer limbs, finalize rounds once.  Sequence:
 *   exact_begin -> exact_accumulate (per chunk / shard) [-> allreduce(SUM) of
 *   the first qdot_b200_exact_region_words() int64 words of xws across ranks]
 *   -> exact_plain (optional, serial) -> exact_finalize -> exact_fetch. */
typedef struct {
    double value;           /* correctly rounded dot product                         */
    double plain;           /* left-to-right double sum of fl(x_i*y_i) (ReferenceResult.plain) */
    int64_t nonfinite;      /* non-finite input elements (-> ValueError)             */
    int32_t status;         /* QDOT_OK, QDOT_ERR_NONFINITE, QDOT_ERR_OVERFLOW        */
    int32_t flexp_e;        /* flexp(value) when value != 0                          */
    int32_t is_zero;        /* value == 0 (flexp_e undefined -> None)                */
    int32_t fallback;       /* the reference would take its Fraction path            */
    int32_t reserved[4];
} qdot_exact_result;
size_t qdot_b200_exact_workspace_bytes(void);
int64_t qdot_b200_exact_region_words(void);
int qdot_b200_exact_begin(void* xws, void* stream);
int qdot_b200_exact_accumulate(const double* x, const double* y, int64_t n, int norm, void* xws, void* stream);
/* one-thread sequential sum, chained across calls in element order; run after
 * every exact_accumulate of the same vectors (its start value depends on them) */
int qdot_b200_exact_plain(const double* x, const double* y, int64_t n, int norm, void* xws, void* stream);
int qdot_b200_exact_finalize(void* xws, void* stream);
int qdot_b200_exact_fetch(const void* xws, qdot_exact_result* out, void* stream);

/* --- synthetic inputs on the device (bench / harness at 2^28-2^31) ----------- */
/* x[i], y[i] (y may be NULL) for global indices offset..offset+n-1 of one
 * vector pair: a pure function of (law, param, seed, index), so shards of any
 * rank count concatenate to the unsharded vectors.  Laws: 0 standard normal
 * (SURVEY.md §8d C1/C2/C4/C5), 1 ill-conditioned pairs (C3), 2 / 3 harness
 * families A / B with spread param = t (harness.py:61-76).  Same laws as the
 * numpy generators, not their bytes. */
int qdot_b200_generate(int law, double param, uint64_t seed, int64_t offset, int64_t n, double* x, double* y,
                       void* stream);

/* --- measurement ------------------------------------------------------------- */
/* stream n doubles (16-byte aligned) once with pass 1's load pattern and
 * discard them: the HBM read ceiling bench.py reports next to the copy peak */
int qdot_b200_read_probe(const double* x, int64_t n, double* out, void* stream);

/* --- device-resident solver loop (apps.py:178-229 without a host round trip
 * per iteration): a CUDA graph whose single WHILE-conditional node runs a body
 * the caller captures on `stream` between _loop_create and _loop_finish (the
 * iteration's SpMV, qdot pipelines, scalar recurrence and vector updates),
 * ending with qdot_b200_acg_check: it records iteration k (both dots' result
 * headers and the scalar state st[0..7], 576 bytes) into rec[k] and clears
 * the condition once the host loop would stop (a dot's status, p.Ap not finite
 * or <= 0, r.r < 0, sqrt(r.r) <= tau = st[7], or k + 1 == cap).  counter =
 * {k, cap} (device int64[2]) is set by the caller before each launch. */
int qdot_b200_loop_create(void* stream, void** loop, unsigned long long* handle);
int qdot_b200_loop_finish(void* loop, void* stream);
int qdot_b200_loop_launch(void* loop, void* stream);
void qdot_b200_loop_destroy(void* loop);
int qdot_b200_acg_check(const void* ws_a, const void* ws_b, const double* st, void* rec, long long* counter,
                        unsigned long long handle, void* stream);
/* fused ACG iteration tail for the loop body (apps.py:212-223): cg_xr computes
 * alpha = st[0] / d (d = the p.Ap result in ws_pq), x += alpha p, r -= alpha q
 * (products rounded first, as numpy); cg_p_check computes beta = c_new / st[0]
 * (c_new = the r.r result in ws_rr), p = r + beta p, and then, in the last
 * CTA, advances st (c, beta, sqrt(c)) and does qdot_b200_acg_check's record and
 * condition.  counter = {k, cap, ticket} (device int64[3], ticket 0). */
int qdot_b200_cg_xr(int64_t n, const void* ws_pq, double* st, double* x, const double* p, double* r,
                    const double* q, void* ws_clear, void* stream);
int qdot_b200_cg_p_check(int64_t n, const void* ws_pq, const void* ws_rr, double* st, const double* r, double* p,
                         void* rec, long long* counter, unsigned long long handle, void* ws_clear, void* stream);
/* ws_clear (may be NULL): a qdot workspace whose exchange regions the kernel also
 * zeroes (what qdot_b200_begin does) -- the loop body then runs the next qdot
 * on it with qdot_b200_enqueue_zeroed (no begin launch) */
/* fused power-method iteration for the loop body (apps.py:302-315): pm_div:
 * x_next = z / sqrt(c) (c = the z.z result in ws_zz; st[0] = c, st[3] = sqrt c);
 * pm_check: x = x_next, then in the last CTA lam = (x . x_next) * st[3]
 * (st[4], st[5] = lam_prev, st[6] = 1), the record of iteration k and the
 * condition (both dots OK, z not all zero, z.z >= 0, not |lam - lam_prev| <=
 * tau = st[7] with st[6] set on entry, k + 1 < cap); counter = {k, cap, ticket}. */
int qdot_b200_pm_div(int64_t n, const void* ws_zz, double* st, const double* z, double* xn, void* stream);
int qdot_b200_pm_check(int64_t n, const void* ws_zz, const void* ws_lam, double* st, const double* xn, double* x,
                       void* rec, long long* counter, unsigned long long handle, void* stream);

/* --- host-side helpers (no GPU needed; exported for tests and bindings) ----- */
/* correctly rounded acc * 2^u with math.ldexp semantics; *overflow set on range error */
double qdot_b200_ldexp_rn(double acc, int64_t u, int* overflow);
/* the report's bound sums over a fetched bin table (scoring.py:171-199,
 * kernel.py:205-222): out[0] = math.fsum of M * ldexp(eps(precision),
 * upper - shift + 1) over the bins, out[1] = their left-to-right sum from 0.0.
 * shift = 0: abs_bound; e_max: rel_bound; reference.flexp_e: rel_bound_e.
 * QDOT_ERR_OVERFLOW where the reference raises OverflowError. */
int qdot_b200_bound_sums(const qdot_bin* bins, int32_t n_bins, int64_t shift, double* out);
/* both at once for shifts a then b (out[0..1], out[2..3]); the first failure is returned */
int qdot_b200_bound_sums2(const qdot_bin* bins, int32_t n_bins, int64_t shift_a, int64_t shift_b, double* out);

#ifdef __cplusplus
}
#endif

#endif /* QDOT_B200_H */
