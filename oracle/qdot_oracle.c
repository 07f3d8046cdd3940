/*
 * qdot CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference qdot path
 * (/root/reference/pkg/src/qdot, package version 0.1.0), used only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs as the CHECKER.  Nothing in paper_2105_00115_b200/ may
 * link, import or call this file.
 *
 * Every function follows the reference line by line (file:line cited), with
 * the same data structures: the exponent-sum array e, the stable counting
 * sort producing `order`, the per-bin member lists, Neumaier accumulation in
 * index order, fp16/fp32 round-to-nearest-even emulation and the Neumaier
 * fold in ascending-upper order.  It deliberately does NOT share code or
 * algorithms with the CUDA path (which derives everything from the
 * histogram and accumulates exactly).
 *
 * Pinning: tests/test_oracle_golden.py checks this restatement against the
 * golden vectors in tests/golden/ that tests/golden/make_golden.py generated
 * by importing the reference package itself (PYTHONPATH=/root/reference/pkg/src).
 *
 * Build: oracle/Makefile  (gcc -O2 -fopenmp -ffp-contract=off, no fast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_NONFINITE 1 /* floatbits.py:70-71  ValueError("inputs must be finite") */
#define OR_ERR_OVERFLOW 2  /* emulate.py:147-148 / math.ldexp range error / kernel.py:130 */
#define OR_ERR_ARG 3       /* bad strategy / mu (binning.py:157, scoring.py:78) */
#define OR_ERR_EPS 4       /* scoring.py:84-85 floor_log2 of non-positive eps_eff */
#define OR_ERR_NOMEM 5

#define OR_PERFORATE 0
#define OR_HALF 1
#define OR_SINGLE 2
#define OR_DOUBLE 3

#define OR_EXACT 0
#define OR_RANGED 1
#define OR_SPLIT 2

#define OR_KEYS 4195   /* exponent sums lie in [-2148, 2046]  (floatbits.py:10-14) */
#define OR_KEY_OFF 2148

typedef struct {
    int64_t lower, upper, cardinality, score;
    int32_t precision, pad;
    double value;          /* bin_dot(x, y, b)  (emulate.py:116-154) */
    int64_t member_start;  /* offset of this bin's ascending indices in `members` */
} or_bin;

typedef struct {
    double value;          /* qdot_accumulate(values)  (emulate.py:157-163) */
    double eps_eff;        /* scoring.py:193 */
    double rel_bound_plain;/* ParameterSet.rel_bound, plain left-to-right sum (scoring.py:195-199) */
    int64_t n, nnz, zero_count;
    int64_t e_min, e_max, n_bins;
    int64_t early_terminated;
    int64_t counts[4];     /* kernel.py:171-176 (zeros counted as PERFORATE) */
} or_result;

static int g_threads = 1;

void or_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int or_get_threads(void) { return g_threads; }

/* ------------------------------------------------------------------ */
/* floatbits.py:17-27  flexp(x) = frexp(|x|)[1] - 1                    */
static inline int64_t or_flexp(double v) {
    int e;
    frexp(fabs(v), &e);
    return (int64_t)e - 1;
}

int64_t or_flexp_export(double v) { return or_flexp(v); }

/* scoring.py:82-86 floor_log2; returns 0 and sets *ok=0 for non-positive/non-finite */
static inline int64_t or_floor_log2(double v, int* ok) {
    if (!(v > 0.0 && isfinite(v))) { *ok = 0; return 0; }
    int e;
    frexp(v, &e);
    *ok = 1;
    return (int64_t)e - 1;
}

/* scoring.py:89-93 ceil_log2(m) = (m-1).bit_length() */
static inline int64_t or_ceil_log2(int64_t m) {
    uint64_t v = (uint64_t)(m - 1);
    int64_t b = 0;
    while (v) { b++; v >>= 1; }
    return b;
}

/* scoring.py:108-123 precision_of */
static const int MU_OF[4] = {0, 10, 23, 52};
static int or_precision_of(int64_t score, int input_mu) {
    if (score < 0) return OR_PERFORATE;
    for (int lvl = OR_HALF; lvl <= OR_DOUBLE; ++lvl) {
        if (MU_OF[lvl] > input_mu) break;
        if (score < MU_OF[lvl]) return lvl;
    }
    return input_mu == 10 ? OR_HALF : (input_mu == 23 ? OR_SINGLE : OR_DOUBLE);
}

/* scoring.py:49 _MU_BELOW + scoring.py:126-136 early_termination */
static int or_early_termination(int64_t e_min, int64_t e_max, int input_mu, double eps, int* ok) {
    int64_t mu_hat = input_mu == 52 ? 23 : (input_mu == 23 ? 10 : 0);
    int64_t fl = or_floor_log2(eps, ok);
    return (e_max - e_min) <= (-fl - mu_hat);
}

/* ------------------------------------------------------------------ */
/* RNE rounding into a binary format by exact arithmetic, the same recipe
 * as the reference test oracle conftest.py:42-60 (quantum = 2^(max(e,
 * min_exp) - mant)), overflow to inf.  All steps are exact in double.     */
static double or_round_to_format(double v, int mant, int min_exp, int max_exp) {
    if (v == 0.0) return v;
    double a = fabs(v);
    int64_t e = or_flexp(a);
    int64_t q = (e > min_exp ? e : min_exp) - mant;
    double s = ldexp(a, (int)(-q));           /* exact: power-of-two scaling */
    double k = floor(s);
    double frac = s - k;                      /* exact */
    if (frac > 0.5 || (frac == 0.5 && fmod(k, 2.0) == 1.0)) k += 1.0;
    double r = ldexp(k, (int)q);
    double max_finite = ldexp(2.0 - ldexp(1.0, -mant), max_exp);
    if (r > max_finite) r = INFINITY;
    return v < 0 ? -r : r;
}

/* emulate.py:27-52 round_to / _round_array: numpy casts to float16/float32 */
double or_round_half(double v) { return or_round_to_format(v, 10, -14, 15); }
double or_round_single(double v) { return or_round_to_format(v, 23, -126, 127); }

/* ------------------------------------------------------------------ */
/* emulate.py:55-72 neumaier_sum / :77-89 _neumaier_kernel               */
typedef struct { double s, c; } or_neu;
static inline void or_neu_add(or_neu* a, double v) {
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
    else a->c += (v - t) + a->s;
    a->s = t;
}
static inline double or_neu_total(const or_neu* a) {
    if (!isfinite(a->s)) return a->s;
    return a->s + a->c;
}

double or_neumaier(const double* v, int64_t m) {
    or_neu a = {0.0, 0.0};
    for (int64_t i = 0; i < m; ++i) or_neu_add(&a, v[i]);
    return or_neu_total(&a);
}

/* math.ldexp semantics: correctly rounded, OverflowError on finite->inf */
static inline double or_py_ldexp(double acc, int64_t u, int* ovf) {
    if (acc == 0.0 || !isfinite(acc)) return ldexp(acc, 0);
    if (u > 100000) u = 100000;
    if (u < -100000) u = -100000;
    double r = ldexp(acc, (int)u);
    if (isinf(r)) *ovf = 1;
    return r;
}

/* np.ldexp semantics (no raise; inf on overflow, RNE on underflow) */
static inline double or_np_ldexp(double v, int64_t k) {
    if (k > 100000) k = 100000;
    if (k < -100000) k = -100000;
    return ldexp(v, (int)k);
}

/* ------------------------------------------------------------------ */
/* emulate.py:116-154 bin_dot over ascending member indices.            */
static double or_bin_dot(const double* x, const double* y, const int64_t* idx, int64_t m,
                         int prec, int64_t upper, int* ovf) {
    if (prec == OR_PERFORATE || m == 0) return 0.0;                  /* :128-129 */
    if (prec == OR_DOUBLE) {                                          /* :132-133 */
        or_neu a = {0.0, 0.0};
        for (int64_t j = 0; j < m; ++j) or_neu_add(&a, x[idx[j]] * y[idx[j]]);
        return or_neu_total(&a);
    }
    float acc32 = 0.0f;                                               /* :91-96 */
    or_neu a = {0.0, 0.0};
    for (int64_t j = 0; j < m; ++j) {
        double xs = x[idx[j]], ys = y[idx[j]];
        int64_t ex = or_flexp(xs);                                    /* :137 */
        double sx = or_np_ldexp(xs, -ex);                             /* :140 */
        double sy = or_np_ldexp(ys, ex - upper);                      /* :141 */
        double rx, ry, p;
        if (prec == OR_HALF) {
            rx = or_round_half(sx); ry = or_round_half(sy);           /* :142-143 */
            p = or_round_half(rx * ry);                               /* :146 */
        } else {
            rx = or_round_single(sx); ry = or_round_single(sy);
            p = or_round_single(rx * ry);
        }
        if (!isfinite(p)) { *ovf = 1; return NAN; }                   /* :147-148 */
        if (prec == OR_HALF) acc32 = (float)(acc32 + (float)p);       /* :150-151 */
        else or_neu_add(&a, p);                                       /* :152-153 */
    }
    double acc = prec == OR_HALF ? (double)acc32 : or_neu_total(&a);
    return or_py_ldexp(acc, upper, ovf);                              /* :154 */
}

/* ------------------------------------------------------------------ */
/* exponent histogram only (floatbits.py:57-93 + binning.py:102-103),   */
/* used by host-logic tests (multi-rank histogram exchange).            */
int or_hist(const double* x, const double* y, int64_t n, int64_t* counts /*[OR_KEYS]*/,
            int64_t* zero_count) {
    memset(counts, 0, sizeof(int64_t) * OR_KEYS);
    int64_t z = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(x[i]) || !isfinite(y[i])) return OR_ERR_NONFINITE;
    }
    for (int64_t i = 0; i < n; ++i) {
        if (x[i] == 0.0 || y[i] == 0.0) { z++; continue; }
        counts[or_flexp(x[i]) + or_flexp(y[i]) + OR_KEY_OFF]++;
    }
    *zero_count = z;
    return OR_OK;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* ------------------------------------------------------------------ */
/* The whole qdot path: kernel.py:179-240 minus report bounds (the Python
 * wrapper computes those with math.fsum exactly as kernel.py:205-206).
 * bins must hold >= min(nnz, OR_KEYS) + 1 entries (never more bins than
 * distinct keys); members, if non-NULL, must hold n entries.            */
int or_qdot(const double* x, const double* y, int64_t n,
            double eps, int split_per_bin, int input_mu, int strategy, int64_t param,
            or_result* res, or_bin* bins, int64_t max_bins, int64_t* members) {
    memset(res, 0, sizeof(*res));
    res->n = n;
    if (!(input_mu == 10 || input_mu == 23 || input_mu == 52)) return OR_ERR_ARG;
    if (strategy == OR_RANGED && param < 1) return OR_ERR_ARG;       /* binning.py:131 */
    if (strategy == OR_SPLIT && param < 0) return OR_ERR_ARG;        /* binning.py:142 */
    if (strategy < 0 || strategy > 2) return OR_ERR_ARG;

    /* ---- exponent_preprocess  floatbits.py:57-93 ---- */
    int bad = 0;
#pragma omp parallel for num_threads(g_threads) reduction(|:bad) schedule(static)
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(x[i]) || !isfinite(y[i])) bad |= 1;
    if (bad) return OR_ERR_NONFINITE;                                  /* :70-71 */

    int nt = g_threads;
    int64_t chunk = (n + nt - 1) / (nt > 0 ? nt : 1);
    if (chunk < 1) chunk = 1;
    int nchunks = (int)((n + chunk - 1) / chunk);
    int64_t* cnz = calloc((size_t)nchunks + 1, sizeof(int64_t));
    if (!cnz) return OR_ERR_NOMEM;
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int c = 0; c < nchunks; ++c) {
        int64_t lo = (int64_t)c * chunk, hi = lo + chunk < n ? lo + chunk : n, k = 0;
        for (int64_t i = lo; i < hi; ++i) k += !(x[i] == 0.0 || y[i] == 0.0);   /* :74 */
        cnz[c + 1] = k;
    }
    for (int c = 0; c < nchunks; ++c) cnz[c + 1] += cnz[c];
    int64_t nnz = cnz[nchunks];
    res->nnz = nnz;
    res->zero_count = n - nnz;

    int64_t* idx = malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    int16_t* e = malloc(sizeof(int16_t) * (size_t)(nnz > 0 ? nnz : 1));
    if (!idx || !e) { free(cnz); free(idx); free(e); return OR_ERR_NOMEM; }
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int c = 0; c < nchunks; ++c) {
        int64_t lo = (int64_t)c * chunk, hi = lo + chunk < n ? lo + chunk : n, w = cnz[c];
        for (int64_t i = lo; i < hi; ++i) {
            if (x[i] == 0.0 || y[i] == 0.0) continue;
            idx[w] = i;                                                          /* :76 */
            e[w] = (int16_t)(or_flexp(x[i]) + or_flexp(y[i]));                  /* :82-85 */
            w++;
        }
    }

    int status = OR_OK;
    int64_t* order = NULL;
    int64_t* counts = NULL;
    int64_t* offsets = NULL;

    res->eps_eff = eps;
    if (nnz == 0) {                                  /* kernel.py:51-57 degenerate */
        res->n_bins = 0;
        res->counts[OR_PERFORATE] = n;
        res->value = 0.0;                            /* neumaier_sum([]) */
        goto done;
    }
    int64_t e_min = 1 << 20, e_max = -(1 << 20);
    for (int64_t k = 0; k < nnz; ++k) {
        if (e[k] < e_min) e_min = e[k];
        if (e[k] > e_max) e_max = e[k];
    }
    res->e_min = e_min;
    res->e_max = e_max;

    int okf = 1;
    int early = or_early_termination(e_min, e_max, input_mu, eps, &okf);   /* kernel.py:59 */
    if (!okf) { status = OR_ERR_EPS; goto done; }

    int64_t nb = 0;
    if (early) {                                     /* kernel.py:60-67 */
        res->early_terminated = 1;
        if (max_bins < 1) { status = OR_ERR_ARG; goto done; }
        bins[0].lower = e_min - 1;
        bins[0].upper = e_max;
        bins[0].cardinality = nnz;
        bins[0].member_start = 0;
        nb = 1;
        order = idx;                                 /* indices=summary.idx (ascending) */
        idx = NULL;
    } else {
        /* ---- sorted_bin_init  binning.py:88-116 (counting sort) ---- */
        int64_t span = e_max - e_min + 1;
        counts = calloc((size_t)span, sizeof(int64_t));
        offsets = malloc(sizeof(int64_t) * (size_t)(span + 1));
        order = malloc(sizeof(int64_t) * (size_t)nnz);
        if (!counts || !offsets || !order) { status = OR_ERR_NOMEM; goto done; }
        /* per-chunk histograms so the stable scatter can run in parallel */
        int64_t* ch = calloc((size_t)nchunks * (size_t)span, sizeof(int64_t));
        if (!ch) { status = OR_ERR_NOMEM; goto done; }
        int64_t kchunk = (nnz + nchunks - 1) / nchunks;
#pragma omp parallel for num_threads(g_threads) schedule(static)
        for (int c = 0; c < nchunks; ++c) {
            int64_t lo = (int64_t)c * kchunk, hi = lo + kchunk < nnz ? lo + kchunk : nnz;
            for (int64_t k = lo; k < hi; ++k) ch[(int64_t)c * span + (e[k] - e_min)]++;
        }
        for (int64_t v = 0; v < span; ++v)
            for (int c = 0; c < nchunks; ++c) counts[v] += ch[(int64_t)c * span + v];   /* :103 bincount */
        offsets[0] = 0;
        for (int64_t v = 0; v < span; ++v) offsets[v + 1] = offsets[v] + counts[v];  /* :104-106 */
        /* write cursors: offsets[v] + earlier chunks' counts (stable order) */
        for (int64_t v = 0; v < span; ++v) {
            int64_t w = offsets[v];
            for (int c = 0; c < nchunks; ++c) {
                int64_t t = ch[(int64_t)c * span + v];
                ch[(int64_t)c * span + v] = w;
                w += t;
            }
        }
#pragma omp parallel for num_threads(g_threads) schedule(static)
        for (int c = 0; c < nchunks; ++c) {                                /* :46-55 scatter */
            int64_t lo = (int64_t)c * kchunk, hi = lo + kchunk < nnz ? lo + kchunk : nnz;
            int64_t* wr = ch + (int64_t)c * span;
            for (int64_t k = lo; k < hi; ++k) order[wr[e[k] - e_min]++] = idx[k];   /* :114 */
        }
        free(ch);

        /* ---- build_partition  binning.py:277-284 ---- */
        if (strategy == OR_EXACT) {                                        /* :191-200 */
            for (int64_t v = 0; v < span; ++v) {
                if (!counts[v]) continue;
                if (nb >= max_bins) { status = OR_ERR_ARG; goto done; }
                int64_t u = e_min + v;
                bins[nb].lower = u - 1;
                bins[nb].upper = u;
                bins[nb].cardinality = counts[v];
                bins[nb].member_start = offsets[v];
                nb++;
            }
        } else if (strategy == OR_RANGED) {                                /* :203-220 */
            int64_t w = param;
            int64_t n_int = (span + w - 1) / w;
            for (int64_t k = 1; k <= n_int; ++k) {
                int64_t u = e_min + k * w - 1;
                int64_t lo_key = (k - 1) * w;
                int64_t hi_key = k * w < span ? k * w : span;
                int64_t m = offsets[hi_key] - offsets[lo_key];
                if (m == 0) continue;
                if (nb >= max_bins) { status = OR_ERR_ARG; goto done; }
                qsort(order + offsets[lo_key], (size_t)m, sizeof(int64_t), cmp_i64);   /* np.sort */
                bins[nb].lower = u - w;
                bins[nb].upper = u;
                bins[nb].cardinality = m;
                bins[nb].member_start = offsets[lo_key];
                nb++;
            }
        } else {                                                           /* :223-274 */
            int64_t levels = param;
            int64_t nz = nnz;
            uint64_t t = (uint64_t)(nz - 1 > 0 ? nz - 1 : 0);
            int64_t bl = 0;
            while (t) { bl++; t >>= 1; }
            if (levels > bl) levels = bl;                                  /* :235 */
            /* slices: (start, stop) pairs, recursive halving :238-249 */
            int64_t cap = 1;
            for (int64_t l = 0; l < levels; ++l) cap *= 2;
            int64_t* st = malloc(sizeof(int64_t) * (size_t)cap * 2);
            int64_t* st2 = malloc(sizeof(int64_t) * (size_t)cap * 2);
            if (!st || !st2) { free(st); free(st2); status = OR_ERR_NOMEM; goto done; }
            int64_t ns = 1;
            st[0] = 0; st[1] = nz;
            for (int64_t l = 0; l < levels; ++l) {
                int64_t nn = 0;
                for (int64_t s = 0; s < ns; ++s) {
                    int64_t a = st[2 * s], b = st[2 * s + 1], m = b - a;
                    if (m <= 1) { st2[2 * nn] = a; st2[2 * nn + 1] = b; nn++; continue; }
                    int64_t mid = a + m / 2;
                    st2[2 * nn] = a; st2[2 * nn + 1] = mid; nn++;
                    st2[2 * nn] = mid; st2[2 * nn + 1] = b; nn++;
                }
                int64_t* tmp = st; st = st2; st2 = tmp;
                ns = nn;
            }
            free(st2);
            /* e_sorted(pos): exponent of sorted stream position pos (:252-253),
             * searched through the offsets instead of materialising the repeat */
#define ESORT(pos, out) do { int64_t lo_ = 0, hi_ = span - 1;                \
                while (lo_ < hi_) { int64_t md_ = (lo_ + hi_ + 1) / 2;       \
                    if (offsets[md_] <= (pos)) lo_ = md_; else hi_ = md_ - 1; } \
                (out) = lo_; } while (0)
            /* cuts :258-264 */
            int64_t* cuts = malloc(sizeof(int64_t) * (size_t)(ns > 0 ? ns : 1));
            if (!cuts) { free(st); status = OR_ERR_NOMEM; goto done; }
            int64_t nc = 0;
            for (int64_t s = 0; s + 1 < ns; ++s) {
                int64_t c = st[2 * s + 1];
                int64_t va, vb;
                ESORT(c - 1, va);
                ESORT(c, vb);
                if (va == vb) c = offsets[vb + 1];       /* searchsorted(side="right") */
                if (c < nz && (nc == 0 || c > cuts[nc - 1])) cuts[nc++] = c;
            }
            free(st);
            /* bins :266-273 */
            int64_t prev_u = e_min - 1;
            for (int64_t b = 0; b <= nc; ++b) {
                int64_t start = b == 0 ? 0 : cuts[b - 1];
                int64_t stop = b == nc ? nz : cuts[b];
                int64_t v;
                ESORT(stop - 1, v);
                int64_t u = e_min + v;
                if (nb >= max_bins) { free(cuts); status = OR_ERR_ARG; goto done; }
                qsort(order + start, (size_t)(stop - start), sizeof(int64_t), cmp_i64);
                bins[nb].lower = prev_u;
                bins[nb].upper = u;
                bins[nb].cardinality = stop - start;
                bins[nb].member_start = start;
                nb++;
                prev_u = u;
            }
#undef ESORT
            free(cuts);
        }
    }

    /* ---- assign_precisions  scoring.py:181-216 ---- */
    {
        res->n_bins = nb;
        double eps_eff = (split_per_bin && nb) ? eps / (double)nb : eps;      /* :193 */
        res->eps_eff = eps_eff;
        int ok = 1;
        int64_t fl = or_floor_log2(eps_eff, &ok);
        if (!ok) { status = OR_ERR_EPS; goto done; }
        double rb = 0.0;
        for (int64_t b = 0; b < nb; ++b) {
            int64_t sc = or_ceil_log2(bins[b].cardinality) + bins[b].upper - e_max - fl + 1; /* :96-105 */
            bins[b].score = sc;
            bins[b].precision = or_precision_of(sc, input_mu);
            double peps = ldexp(1.0, -MU_OF[bins[b].precision]);
            int64_t sh = bins[b].upper - e_max + 1;
            if (sh > 4000) sh = 4000;
            if (sh < -4000) sh = -4000;
            rb += (double)bins[b].cardinality * ldexp(peps, (int)sh);           /* :171-173 */
        }
        res->rel_bound_plain = rb;
    }

    /* ---- compute phase  kernel.py:201-202 ---- */
    {
        int any_ovf = 0;
#pragma omp parallel for num_threads(g_threads) schedule(dynamic, 1) reduction(|:any_ovf)
        for (int64_t b = 0; b < nb; ++b) {
            int ovf = 0;
            bins[b].value = or_bin_dot(x, y, order + bins[b].member_start, bins[b].cardinality,
                                       bins[b].precision, bins[b].upper, &ovf);
            any_ovf |= ovf;
        }
        if (any_ovf) { status = OR_ERR_OVERFLOW; goto done; }
        or_neu acc = {0.0, 0.0};                                          /* emulate.py:157-163 */
        for (int64_t b = 0; b < nb; ++b) or_neu_add(&acc, bins[b].value);
        res->value = or_neu_total(&acc);
        for (int64_t b = 0; b < nb; ++b) res->counts[bins[b].precision] += bins[b].cardinality;
        res->counts[OR_PERFORATE] += n - nnz;                             /* kernel.py:175 */
    }
    if (members) memcpy(members, order, sizeof(int64_t) * (size_t)nnz);

done:
    free(cnz);
    free(idx);
    free(e);
    free(order);
    free(counts);
    free(offsets);
    return status;
}

/* ------------------------------------------------------------------ */
/* Exact dot product (the reference_dot contract, kernel.py:98-133: the
 * correctly rounded true sum, OverflowError if it overflows).  Restated
 * as an exact fixed-point superaccumulator over exact 106-bit products,
 * which yields the same correctly rounded value as Dekker+fsum and the
 * Fraction fallback.  `plain` is the left-to-right double dot (:122,128). */
#define SA_DIGITS 140   /* 32-bit digits covering bit positions [-2148, 2332) */
#define SA_BASE 2148

typedef struct { int64_t d[SA_DIGITS]; int64_t adds; } or_sacc;

static void sa_normalize(or_sacc* a) {
    int64_t carry = 0;
    for (int i = 0; i < SA_DIGITS; ++i) {
        int64_t v = a->d[i] + carry;
        int64_t lo = v & 0xFFFFFFFFLL;
        carry = (v - lo) / 4294967296LL;   /* exact: v - lo is a multiple of 2^32 */
        a->d[i] = lo;
    }
    a->d[SA_DIGITS - 1] += carry * 4294967296LL;  /* sign lives in the top digit */
    a->adds = 0;
}

static inline void sa_add_product(or_sacc* a, double xv, double yv) {
    uint64_t bx, by;
    memcpy(&bx, &xv, 8);
    memcpy(&by, &yv, 8);
    int neg = (int)((bx ^ by) >> 63);
    int ex = (int)((bx >> 52) & 0x7FF), ey = (int)((by >> 52) & 0x7FF);
    uint64_t mx = bx & ((1ULL << 52) - 1), my = by & ((1ULL << 52) - 1);
    if (ex) mx |= 1ULL << 52; else ex = 1;
    if (ey) my |= 1ULL << 52; else ey = 1;
    if (!mx || !my) return;
    unsigned __int128 p = (unsigned __int128)mx * my;
    int pos = (ex - 1075) + (ey - 1075) + SA_BASE;   /* >= 0 */
    int di = pos >> 5, off = pos & 31;
    /* p << off spans <= 138 bits: up to 5 digits */
    unsigned __int128 lo = p << off;                  /* low 128 bits */
    uint64_t top = off ? (uint64_t)(p >> (128 - off)) : 0;
    uint32_t dig[5];
    dig[0] = (uint32_t)lo; dig[1] = (uint32_t)(lo >> 32);
    dig[2] = (uint32_t)(lo >> 64); dig[3] = (uint32_t)(lo >> 96);
    dig[4] = (uint32_t)top;
    for (int k = 0; k < 5; ++k) {
        if (neg) a->d[di + k] -= dig[k]; else a->d[di + k] += dig[k];
    }
    if (++a->adds >= (1LL << 29)) sa_normalize(a);
}

/* correctly round the (normalised) accumulator to a double; *inf_out on overflow */
static double sa_round(or_sacc* a, int* overflow) {
    sa_normalize(a);
    int neg = a->d[SA_DIGITS - 1] < 0;
    uint32_t mag[SA_DIGITS];
    if (neg) {   /* magnitude = two's complement negation */
        int64_t borrow = 0;
        for (int i = 0; i < SA_DIGITS; ++i) {
            int64_t v = -a->d[i] - borrow;
            if (v < 0) { v += 4294967296LL; borrow = 1; } else borrow = 0;
            mag[i] = (uint32_t)v;
        }
    } else {
        for (int i = 0; i < SA_DIGITS; ++i) mag[i] = (uint32_t)a->d[i];
    }
    int top = -1;
    for (int i = SA_DIGITS - 1; i >= 0 && top < 0; --i)
        if (mag[i]) top = i * 32 + (31 - __builtin_clz(mag[i]));
    if (top < 0) return 0.0;
    int vexp = top - SA_BASE;                        /* value exponent of the top bit */
    int qexp = vexp - 52 > -1074 ? vexp - 52 : -1074; /* double quantum exponent */
    int qpos = qexp + SA_BASE;                       /* bit position of the quantum */
#define BIT(p) ((p) < 0 ? 0u : ((mag[(p) >> 5] >> ((p) & 31)) & 1u))
    uint64_t m = 0;
    for (int p = top; p >= qpos; --p) m = (m << 1) | BIT(p);
    int rb = qpos - 1 >= 0 ? (int)BIT(qpos - 1) : 0;
    int sticky = 0;
    for (int p = qpos - 2; p >= 0 && !sticky; --p) sticky = (int)BIT(p);
#undef BIT
    if (rb && (sticky || (m & 1))) m += 1;
    double r = ldexp((double)m, qexp);
    if (isinf(r)) *overflow = 1;
    return neg ? -r : r;
}

/* returns OR_OK / OR_ERR_NONFINITE / OR_ERR_OVERFLOW; value, flexp_e (valid if has_e), plain */
int or_exact_dot(const double* x, const double* y, int64_t n, double* value,
                 int64_t* flexp_e, int* has_e, double* plain) {
    *value = 0.0; *plain = 0.0; *has_e = 0; *flexp_e = 0;
    if (n == 0) return OR_OK;                                         /* kernel.py:112-113 */
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(x[i]) || !isfinite(y[i])) return OR_ERR_NONFINITE;
    int nt = g_threads;
    or_sacc* acc = calloc((size_t)nt, sizeof(or_sacc));
    if (!acc) return OR_ERR_NOMEM;
#pragma omp parallel num_threads(nt)
    {
#ifdef _OPENMP
        int tid = omp_get_thread_num();
#else
        int tid = 0;
#endif
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) sa_add_product(&acc[tid], x[i], y[i]);
    }
    for (int t = 0; t < nt; ++t) sa_normalize(&acc[t]);
    for (int t = 1; t < nt; ++t)
        for (int i = 0; i < SA_DIGITS; ++i) acc[0].d[i] += acc[t].d[i];
    int ovf = 0;
    double v = sa_round(&acc[0], &ovf);
    free(acc);
    if (ovf) return OR_ERR_OVERFLOW;                                  /* :130-131 */
    double p = 0.0;
    for (int64_t i = 0; i < n; ++i) p = p + x[i] * y[i];
    *value = v;
    *plain = p;
    if (v != 0.0) { *has_e = 1; *flexp_e = or_flexp(v); }
    return OR_OK;
}
