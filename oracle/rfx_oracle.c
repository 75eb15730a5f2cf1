/*
 * rfx_oracle.c — CPU restatement of the RFX proximity hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it, and only as the checker or
 * as the timed CPU baseline.  It restates the reference algorithm
 * (pure-Python + Numba package under /root/reference/pkg/src/rfx) in plain
 * C so that it can run on the GPU box, where the reference does not exist.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, tests/test_oracle.py).
 *
 * Functions and the reference code they restate:
 *   orc_pcg32_*            rng.py:41-70 (pcg32_next, make_stream, pcg32_bounded)
 *   orc_fill_normals       rng.py:102-115 (Box-Muller, r*cos then r*sin)
 *   orc_descend_all        _kernels.py:333-348, :369-374 (descend / descend_all)
 *   orc_leaf_membership    proximity.py:100-116 (+ forest.py:95-99 leaf_codes)
 *   orc_pair_counts_tree   _kernels.py:483-510 (accumulate_pair_counts)
 *   orc_pair_counts_block  _kernels.py:452-480 (accumulate_pair_counts_block)
 *   orc_pair_counts        proximity.py:159-185 (_pair_counts orchestration)
 *   orc_sketch_pass        proximity.py:389-398 (M @ (Mt @ X) with M the
 *                          1/sqrt(B)-scaled one-hot, evaluated per tree)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ PCG32 */
/* rng.py:41-48 — returns the next 32-bit output. */
static uint32_t orc_next(uint64_t *s)
{
    uint64_t old = s[0];
    s[0] = old * 6364136223846793005ULL + s[1];
    uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

/* rng.py:51-59 — make_stream(seed, seq); seed wraps mod 2^64. */
void orc_pcg32_make(int64_t seed, int64_t seq, uint64_t *s)
{
    s[0] = 0;
    s[1] = ((uint64_t)seq << 1) | 1ULL;
    orc_next(s);
    s[0] += (uint64_t)seed;
    orc_next(s);
}

uint32_t orc_pcg32_next(uint64_t *s) { return orc_next(s); }

/* rng.py:62-70 — rejection-sampled draw in [0, bound). */
uint32_t orc_pcg32_bounded(uint64_t *s, uint32_t bound)
{
    uint64_t b = bound;
    uint64_t threshold = (0x100000000ULL - b) % b;
    for (;;) {
        uint64_t r = orc_next(s);
        if (r >= threshold) return (uint32_t)(r % b);
    }
}

/* rng.py:102-115 — standard normals, emitted in pairs r*cos, r*sin. */
void orc_fill_normals(uint64_t *s, double *out, int64_t n)
{
    const double two_pi = 2.0 * 3.141592653589793;
    int64_t i = 0;
    while (i < n) {
        double u1 = ((double)orc_next(s) + 1.0) / 4294967296.0;
        double u2 = (double)orc_next(s) / 4294967296.0;
        double r = sqrt(-2.0 * log(u1));
        out[i++] = r * cos(two_pi * u2);
        if (i < n) out[i++] = r * sin(two_pi * u2);
    }
}

/* ------------------------------------------------------------- traversal */
/*
 * _kernels.py:333-348 — walk sample i from node 0 to a terminal.
 * values is column-major (n, p) float64 (dataset.py:59-71, F-order).
 * Numeric: left iff x <= threshold.  Categorical: left iff bit (int64)x of
 * cat_mask is set.
 */
static int32_t orc_descend(const int8_t *status, const int32_t *split_var,
                           const double *threshold, const int64_t *cat_mask,
                           const int32_t *left, const int32_t *right,
                           const uint8_t *col_cat, const double *values,
                           int64_t n, int64_t i)
{
    int32_t node = 0;
    while (status[node] == 0) {
        int32_t j = split_var[node];
        double v = values[(int64_t)j * n + i];
        int go;
        if (col_cat[j] == 1)
            go = (int)((cat_mask[node] >> (int64_t)v) & 1);
        else
            go = v <= threshold[node];
        node = go ? left[node] : right[node];
    }
    return node;
}

/* _kernels.py:369-374 — terminal node id per row for one tree. */
void orc_descend_all(const int8_t *status, const int32_t *split_var,
                     const double *threshold, const int64_t *cat_mask,
                     const int32_t *left, const int32_t *right,
                     const uint8_t *col_cat, const double *values, int64_t n,
                     int32_t *out)
{
    for (int64_t i = 0; i < n; i++)
        out[i] = orc_descend(status, split_var, threshold, cat_mask, left,
                             right, col_cat, values, n, i);
}

/*
 * proximity.py:100-116 + forest.py:95-99 — codes (n, B) int32 C-order.
 * Trees are concatenated; tree b owns nodes [node_off[b], node_off[b+1]).
 * Child ids are tree-local.  Parallel over trees like map_in_order
 * (_parallel.py:23-30); results do not depend on the thread count.
 */
void orc_leaf_membership(const int64_t *node_off, int32_t B,
                         const int8_t *status, const int32_t *split_var,
                         const double *threshold, const int64_t *cat_mask,
                         const int32_t *left, const int32_t *right,
                         const uint8_t *col_cat, const double *values,
                         int64_t n, int32_t *codes, int32_t *leaf_counts,
                         int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int32_t b = 0; b < B; b++) {
        int64_t o = node_off[b], nc = node_off[b + 1] - node_off[b];
        int32_t *leaf_code = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
        int32_t run = -1;
        for (int64_t t = 0; t < nc; t++) {
            if (status[o + t] == 1) leaf_code[t] = ++run;
            else leaf_code[t] = -1;
        }
        leaf_counts[b] = run + 1;
        for (int64_t i = 0; i < n; i++) {
            int32_t node = orc_descend(status + o, split_var + o,
                                       threshold + o, cat_mask + o, left + o,
                                       right + o, col_cat, values, n, i);
            codes[i * B + b] = leaf_code[node];
        }
        free(leaf_code);
    }
}

/* ------------------------------------------------------------ pair counts */
/* Stable counting sort of one tree's codes (_kernels.py:491-501). */
static void orc_bucket(const int32_t *codes, int64_t stride, int64_t n,
                       int32_t leaf_count, int64_t *occ, int64_t *bucket)
{
    memset(occ, 0, sizeof(int64_t) * (size_t)(leaf_count + 1));
    for (int64_t i = 0; i < n; i++) occ[codes[i * stride] + 1]++;
    for (int32_t l = 0; l < leaf_count; l++) occ[l + 1] += occ[l];
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(leaf_count + 1));
    memcpy(pos, occ, sizeof(int64_t) * (size_t)leaf_count);
    for (int64_t i = 0; i < n; i++) bucket[pos[codes[i * stride]]++] = i;
    free(pos);
}

/*
 * _kernels.py:483-510 — add one tree's co-membership to the packed i<j
 * counter (row-major upper triangle, proximity.py:59-61 index).
 * codes may be strided (column b of the (n, B) membership: stride B).
 */
void orc_pair_counts_tree(const int32_t *codes, int64_t stride, int64_t n,
                          int32_t leaf_count, int64_t *packed)
{
    int64_t *occ = (int64_t *)malloc(sizeof(int64_t) * (size_t)(leaf_count + 1));
    int64_t *bucket = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    orc_bucket(codes, stride, n, leaf_count, occ, bucket);
    for (int32_t l = 0; l < leaf_count; l++) {
        int64_t lo = occ[l], hi = occ[l + 1];
        for (int64_t a = lo; a < hi; a++) {
            int64_t i = bucket[a];
            int64_t base = i * (2 * n - i - 1) / 2 - i - 1;
            for (int64_t c = a + 1; c < hi; c++) packed[base + bucket[c]]++;
        }
    }
    free(occ);
    free(bucket);
}

/*
 * _kernels.py:452-480 — rows [row_lo, row_hi) into an int32 (rows x n)
 * block, columns j > i only; stops a bucket walk once i >= row_hi.
 */
void orc_pair_counts_block(const int32_t *codes, int64_t stride, int64_t n,
                           int32_t leaf_count, int64_t row_lo, int64_t row_hi,
                           int32_t *block)
{
    int64_t *occ = (int64_t *)malloc(sizeof(int64_t) * (size_t)(leaf_count + 1));
    int64_t *bucket = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    orc_bucket(codes, stride, n, leaf_count, occ, bucket);
    for (int32_t l = 0; l < leaf_count; l++) {
        int64_t lo = occ[l], hi = occ[l + 1];
        for (int64_t a = lo; a < hi; a++) {
            int64_t i = bucket[a];
            if (i >= row_hi) break;
            if (i < row_lo) continue;
            int32_t *row = block + (i - row_lo) * n;
            for (int64_t c = a + 1; c < hi; c++) row[bucket[c]]++;
        }
    }
    free(occ);
    free(bucket);
}

/*
 * proximity.py:159-185 — integer counts over all trees, packed i<j.
 * Per-thread buffers only when pairs*8*threads <= 256 MiB and B >= 2*threads,
 * otherwise a serial loop (proximity.py:165) — the reference's own policy,
 * kept so the CPU baseline has the reference's parallelism.
 */
void orc_pair_counts(const int32_t *codes, int64_t n, int32_t B,
                     const int32_t *leaf_counts, int64_t *packed, int nthreads)
{
    int64_t pairs = n * (n - 1) / 2;
    memset(packed, 0, sizeof(int64_t) * (size_t)pairs);
    int w = nthreads > 0 ? nthreads : 1;
    if (w > 1 && pairs * 8 * (int64_t)w <= 256LL * 1024 * 1024 && B >= 2 * w) {
        int64_t **parts = (int64_t **)calloc((size_t)w, sizeof(int64_t *));
#ifdef _OPENMP
        omp_set_num_threads(w);
#pragma omp parallel for schedule(static, 1)
#endif
        for (int t = 0; t < w; t++) {
            int32_t b0 = (int32_t)((int64_t)B * t / w);
            int32_t b1 = (int32_t)((int64_t)B * (t + 1) / w);
            parts[t] = (int64_t *)calloc((size_t)pairs, sizeof(int64_t));
            for (int32_t b = b0; b < b1; b++)
                orc_pair_counts_tree(codes + b, B, n, leaf_counts[b], parts[t]);
        }
        for (int t = 0; t < w; t++) {
            for (int64_t q = 0; q < pairs; q++) packed[q] += parts[t][q];
            free(parts[t]);
        }
        free(parts);
        return;
    }
    for (int32_t b = 0; b < B; b++)
        orc_pair_counts_tree(codes + b, B, n, leaf_counts[b], packed);
}

/* ------------------------------------------------------------ sketch pass */
/*
 * proximity.py:389-398 — Y = M (M^T X) with M the one-hot membership scaled
 * by 1/sqrt(B) (proximity.py:88-97), i.e. Y = (1/B) sum_b E_b E_b^T X.
 * Evaluated per tree with per-leaf sums; X and Y are (n, k) row-major f64.
 * Tree blocks are summed in a fixed order, so the result does not depend on
 * the thread count.
 */
void orc_sketch_pass(const int32_t *codes, int64_t n, int32_t B,
                     const int32_t *leaf_counts, const double *X, int32_t k,
                     double *Y, int nthreads)
{
    int w = nthreads > 0 ? nthreads : 1;
    double **parts = (double **)calloc((size_t)w, sizeof(double *));
#ifdef _OPENMP
    omp_set_num_threads(w);
#pragma omp parallel for schedule(static, 1)
#endif
    for (int t = 0; t < w; t++) {
        int32_t b0 = (int32_t)((int64_t)B * t / w);
        int32_t b1 = (int32_t)((int64_t)B * (t + 1) / w);
        double *acc = (double *)calloc((size_t)(n * k), sizeof(double));
        for (int32_t b = b0; b < b1; b++) {
            int32_t L = leaf_counts[b];
            double *S = (double *)calloc((size_t)L * k, sizeof(double));
            for (int64_t i = 0; i < n; i++) {
                const double *x = X + i * k;
                double *s = S + (int64_t)codes[i * B + b] * k;
                for (int32_t c = 0; c < k; c++) s[c] += x[c];
            }
            for (int64_t i = 0; i < n; i++) {
                const double *s = S + (int64_t)codes[i * B + b] * k;
                double *y = acc + i * k;
                for (int32_t c = 0; c < k; c++) y[c] += s[c];
            }
            free(S);
        }
        parts[t] = acc;
    }
    double inv = 1.0 / (double)B;
    for (int64_t q = 0; q < n * k; q++) {
        double s = 0.0;
        for (int t = 0; t < w; t++) s += parts[t][q];
        Y[q] = s * inv;
    }
    for (int t = 0; t < w; t++) free(parts[t]);
    free(parts);
}
