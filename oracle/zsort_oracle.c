/*
 * zsort_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded CPU restatement of the reference zSort
 * algorithm (arxiv 2605.14419, reference package `zsort`), used as the
 * parity checker for the B200 implementation and as the timed CPU baseline
 * ("port") in bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * path (paper_2605_14419_b200) never links or calls it.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/pkg/src/zsort/.  Arithmetic follows the
 * reference bit for bit: fp64 expressions are evaluated in the same order
 * with no contraction (build with -ffp-contract=off), int64 -> fp64
 * conversions round to nearest, and the top-level mean is the correctly
 * rounded quotient of the exact integer sum (Python int / int true division,
 * core.py:226).  The oracle is pinned against the reference itself (imported
 * in the build container) by tests/golden/make_golden.py and
 * tests/test_oracle_pin.py, including SortStats counters.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
typedef uint64_t u64;
typedef __int128 i128;
typedef unsigned __int128 u128;

/* Counter slots, _kernels.py:16-21 */
enum { ST_MAX_DEPTH = 0, ST_FALLBACKS = 1, ST_COUNTING = 2, ST_INSERTION = 3, ST_SCATTERS = 4, ST_SLOTS = 5 };

/* Error codes returned to the ctypes wrapper. */
enum { ZO_OK = 0, ZO_ERR_SIZE = 1, ZO_ERR_NOMEM = 2, ZO_ERR_ARG = 3 };

/* ---------------------------------------------------------------- passes */

/* _kernels.py:28-48  first_pass: exact sum as (hi, lo) 32-bit limbs, min, max */
void zo_first_pass(const i64 *keys, i64 lo, i64 hi, i64 *sum_hi, i64 *sum_lo, i64 *mn_out, i64 *mx_out) {
    i64 shi = 0, slo = 0, mn = keys[lo], mx = keys[lo];
    for (i64 i = lo; i < hi; i++) {
        i64 k = keys[i];
        shi += k >> 32;
        slo += k & (i64)0xFFFFFFFF;
        if (k < mn) mn = k;
        else if (k > mx) mx = k;
    }
    *sum_hi = shi; *sum_lo = slo; *mn_out = mn; *mx_out = mx;
}

/* _kernels.py:51-61 */
static void minmax_pass(const i64 *keys, i64 lo, i64 hi, i64 *mn_out, i64 *mx_out) {
    i64 mn = keys[lo], mx = keys[lo];
    for (i64 i = lo + 1; i < hi; i++) {
        i64 k = keys[i];
        if (k < mn) mn = k;
        else if (k > mx) mx = k;
    }
    *mn_out = mn; *mx_out = mx;
}

/* _kernels.py:64-71 */
double zo_variance_pass(const i64 *keys, i64 lo, i64 hi, double mean) {
    double acc = 0.0;
    for (i64 i = lo; i < hi; i++) {
        double d = (double)keys[i] - mean;
        acc += d * d;
    }
    return acc / (double)(hi - lo);
}

/* _kernels.py:74-88 */
static void fused_stats_pass(const i64 *keys, i64 lo, i64 hi, double center, i64 *mn_out, i64 *mx_out, double *var_out) {
    i64 mn = keys[lo], mx = keys[lo];
    double acc = 0.0;
    for (i64 i = lo; i < hi; i++) {
        i64 k = keys[i];
        if (k < mn) mn = k;
        else if (k > mx) mx = k;
        double d = (double)k - center;
        acc += d * d;
    }
    *mn_out = mn; *mx_out = mx; *var_out = acc / (double)(hi - lo);
}

/* _kernels.py:91-100  Eq. 1 bucket id clamped to [0, k-1] */
i64 zo_bucket_of(i64 key, double mean, double std, double zmin, double scale, i64 k) {
    double h = (((double)key - mean) / std + zmin) * scale;
    double f = floor(h);
    if (!(f > 0.0)) return 0;
    if (f >= (double)k) return k - 1;
    return (i64)f;
}

/* _kernels.py:103-106 */
double zo_estimated_center(i64 bucket, double scale, double zmin, double std, double mean) {
    return (((double)bucket + 0.5) / scale - zmin) * std + mean;
}

/* _kernels.py:109-112 */
void zo_histogram_pass(const i64 *keys, i64 lo, i64 hi, double mean, double std, double zmin, double scale, i64 k,
                       i64 *counts) {
    for (i64 i = lo; i < hi; i++) counts[zo_bucket_of(keys[i], mean, std, zmin, scale, k)] += 1;
}

/* _kernels.py:115-121 */
i64 zo_exclusive_offsets(const i64 *counts, i64 *offsets, i64 k) {
    i64 total = 0;
    for (i64 i = 0; i < k; i++) { offsets[i] = total; total += counts[i]; }
    return total;
}

/* _kernels.py:124-133  stable front-to-back scatter */
void zo_scatter_pass(const i64 *keys, const i64 *carry, i64 lo, i64 hi, double mean, double std, double zmin,
                     double scale, i64 k, i64 *cursors, i64 *dst_keys, i64 *dst_carry, i64 dst_lo) {
    for (i64 i = lo; i < hi; i++) {
        i64 b = zo_bucket_of(keys[i], mean, std, zmin, scale, k);
        i64 pos = dst_lo + cursors[b];
        cursors[b] += 1;
        dst_keys[pos] = keys[i];
        dst_carry[pos] = carry[i];
    }
}

/* _kernels.py:136-140 */
static void copy_segment(const i64 *sk, const i64 *sc, i64 slo, i64 *dk, i64 *dc, i64 dlo, i64 n) {
    memmove(dk + dlo, sk + slo, (size_t)n * sizeof(i64));
    memmove(dc + dlo, sc + slo, (size_t)n * sizeof(i64));
}

/* _kernels.py:143-156  stable insertion sort (only strictly greater keys shift) */
void zo_insertion_sort_range(i64 *keys, i64 *carry, i64 lo, i64 hi) {
    for (i64 i = lo + 1; i < hi; i++) {
        i64 kv = keys[i], cv = carry[i];
        i64 j = i - 1;
        while (j >= lo && keys[j] > kv) {
            keys[j + 1] = keys[j];
            carry[j + 1] = carry[j];
            j--;
        }
        keys[j + 1] = kv;
        carry[j + 1] = cv;
    }
}

/* _kernels.py:159-180  stable counting sort; slot arithmetic in uint64 */
int zo_counting_sort_range(const i64 *sk, const i64 *sc, i64 slo, i64 n, i64 mn, i64 bins, i64 *dk, i64 *dc, i64 dlo) {
    i64 *counts = (i64 *)calloc((size_t)bins, sizeof(i64));
    if (!counts) return ZO_ERR_NOMEM;
    for (i64 i = slo; i < slo + n; i++) counts[(i64)((u64)sk[i] - (u64)mn)] += 1;
    i64 total = 0;
    for (i64 b = 0; b < bins; b++) { i64 c = counts[b]; counts[b] = total; total += c; }
    for (i64 i = slo; i < slo + n; i++) {
        i64 slot = (i64)((u64)sk[i] - (u64)mn);
        i64 pos = dlo + counts[slot];
        counts[slot] += 1;
        dk[pos] = sk[i];
        dc[pos] = sc[i];
    }
    free(counts);
    return ZO_OK;
}

/* _kernels.py:183-231  bottom-up stable merge sort of keys[lo:lo+n] */
void zo_merge_sort_range(i64 *keys, i64 *carry, i64 lo, i64 n, i64 *aux_k, i64 *aux_c) {
    if (n <= 1) return;
    i64 *src_k = keys, *src_c = carry, *dst_k = aux_k, *dst_c = aux_c;
    int in_place = 1;
    for (i64 width = 1; width < n; width *= 2) {
        for (i64 start = 0; start < n;) {
            i64 mid = start + width < n ? start + width : n;
            i64 stop = start + 2 * width < n ? start + 2 * width : n;
            i64 p = start, q = mid, o = start;
            while (p < mid && q < stop) {
                if (src_k[lo + q] < src_k[lo + p]) { dst_k[lo + o] = src_k[lo + q]; dst_c[lo + o] = src_c[lo + q]; q++; }
                else { dst_k[lo + o] = src_k[lo + p]; dst_c[lo + o] = src_c[lo + p]; p++; }
                o++;
            }
            while (p < mid) { dst_k[lo + o] = src_k[lo + p]; dst_c[lo + o] = src_c[lo + p]; p++; o++; }
            while (q < stop) { dst_k[lo + o] = src_k[lo + q]; dst_c[lo + o] = src_c[lo + q]; q++; o++; }
            start = stop;
        }
        i64 *t = src_k; src_k = dst_k; dst_k = t;
        t = src_c; src_c = dst_c; dst_c = t;
        in_place = !in_place;
    }
    if (!in_place) {
        for (i64 i = 0; i < n; i++) { keys[lo + i] = src_k[lo + i]; carry[lo + i] = src_c[lo + i]; }
    }
}

/* ------------------------------------------------------------- recursion */

typedef struct {
    i64 *base, *cnt, *level;
    double *mean;
    uint8_t *scratch;
    i64 cap;
} stack_t_;

/* _kernels.py:272-279 */
static void fallback_to_out(i64 *out_k, i64 *out_c, i64 *scr_k, i64 *scr_c, i64 base, i64 n, int in_scratch, i64 *counters) {
    if (in_scratch) copy_segment(scr_k, scr_c, base, out_k, out_c, base, n);
    zo_merge_sort_range(out_k, out_c, base, n, scr_k, scr_c);
    counters[ST_FALLBACKS] += 1;
}

/* _kernels.py:282-318 */
static i64 dispatch_large_bucket(i64 *buf_k, i64 *buf_c, int in_scratch, i64 base, i64 n, i64 bucket, double mean,
                                 double std, double zmin, double scale, i64 k, i64 level, i64 counting_limit,
                                 i64 *out_k, i64 *out_c, i64 *scr_k, i64 *scr_c, i64 *counters, stack_t_ *st, i64 top,
                                 int *err) {
    (void)k;
    i64 bmn, bmx;
    minmax_pass(buf_k, base, base + n, &bmn, &bmx);
    u64 spread = (u64)bmx - (u64)bmn;
    if (spread < (u64)counting_limit) {
        i64 bins = (i64)spread + 1;
        if (in_scratch) {
            *err |= zo_counting_sort_range(buf_k, buf_c, base, n, bmn, bins, out_k, out_c, base);
        } else {
            copy_segment(buf_k, buf_c, base, scr_k, scr_c, base, n);
            *err |= zo_counting_sort_range(scr_k, scr_c, base, n, bmn, bins, out_k, out_c, base);
        }
        counters[ST_COUNTING] += 1;
        return top;
    }
    if (top < st->cap) {
        st->base[top] = base;
        st->cnt[top] = n;
        st->mean[top] = zo_estimated_center(bucket, scale, zmin, std, mean);
        st->level[top] = level + 1;
        st->scratch[top] = in_scratch ? 1 : 0;
        return top + 1;
    }
    fallback_to_out(out_k, out_c, scr_k, scr_c, base, n, in_scratch, counters);
    return top;
}

/* _kernels.py:321-390 */
static void run_worklist(i64 *out_k, i64 *out_c, i64 *scr_k, i64 *scr_c, i64 k, double scale, i64 insertion_limit,
                         i64 counting_limit, i64 depth_guard, i64 *counters, stack_t_ *st, i64 top, i64 *counts,
                         i64 *offsets, i64 *cursors, int *err) {
    while (top > 0) {
        top -= 1;
        i64 base = st->base[top], n = st->cnt[top], level = st->level[top];
        double center = st->mean[top];
        int in_scratch = st->scratch[top] == 1;
        i64 *cur_k = in_scratch ? scr_k : out_k;
        i64 *cur_c = in_scratch ? scr_c : out_c;
        if (level > depth_guard) {
            fallback_to_out(out_k, out_c, scr_k, scr_c, base, n, in_scratch, counters);
            continue;
        }
        i64 mn, mx;
        double var;
        fused_stats_pass(cur_k, base, base + n, center, &mn, &mx, &var);
        if (mn == mx) {
            if (in_scratch) copy_segment(cur_k, cur_c, base, out_k, out_c, base, n);
            continue;
        }
        double std = sqrt(var);
        if (!(std > 0.0) || !isfinite(std)) {
            fallback_to_out(out_k, out_c, scr_k, scr_c, base, n, in_scratch, counters);
            continue;
        }
        double zmin = fabs(((double)mn - center) / std);
        memset(counts, 0, (size_t)k * sizeof(i64));
        zo_histogram_pass(cur_k, base, base + n, center, std, zmin, scale, k, counts);
        i64 occupied = 0;
        for (i64 b = 0; b < k; b++) occupied += counts[b] > 0;
        if (occupied <= 1) {
            fallback_to_out(out_k, out_c, scr_k, scr_c, base, n, in_scratch, counters);
            continue;
        }
        zo_exclusive_offsets(counts, offsets, k);
        memcpy(cursors, offsets, (size_t)k * sizeof(i64));
        i64 *dst_k = in_scratch ? out_k : scr_k;
        i64 *dst_c = in_scratch ? out_c : scr_c;
        zo_scatter_pass(cur_k, cur_c, base, base + n, center, std, zmin, scale, k, cursors, dst_k, dst_c, base);
        counters[ST_SCATTERS] += 1;
        if (counters[ST_MAX_DEPTH] < level) counters[ST_MAX_DEPTH] = level;
        int dst_in_scratch = !in_scratch;
        for (i64 b = 0; b < k; b++) {
            i64 cnt = counts[b];
            if (cnt == 0) continue;
            i64 gbase = base + offsets[b];
            if (cnt <= insertion_limit) {
                if (dst_in_scratch) copy_segment(dst_k, dst_c, gbase, out_k, out_c, gbase, cnt);
                zo_insertion_sort_range(out_k, out_c, gbase, gbase + cnt);
                counters[ST_INSERTION] += 1;
            } else {
                top = dispatch_large_bucket(dst_k, dst_c, dst_in_scratch, gbase, cnt, b, center, std, zmin, scale, k,
                                            level, counting_limit, out_k, out_c, scr_k, scr_c, counters, st, top, err);
            }
        }
    }
}

static int stack_alloc(stack_t_ *st, i64 cap) {
    st->cap = cap;
    st->base = (i64 *)malloc((size_t)cap * sizeof(i64));
    st->cnt = (i64 *)malloc((size_t)cap * sizeof(i64));
    st->level = (i64 *)malloc((size_t)cap * sizeof(i64));
    st->mean = (double *)malloc((size_t)cap * sizeof(double));
    st->scratch = (uint8_t *)malloc((size_t)cap);
    return (st->base && st->cnt && st->level && st->mean && st->scratch) ? ZO_OK : ZO_ERR_NOMEM;
}

static void stack_free(stack_t_ *st) {
    free(st->base); free(st->cnt); free(st->level); free(st->mean); free(st->scratch);
}

/* _kernels.py:393-450 */
int zo_zsort_driver(const i64 *src_k, const i64 *src_c, i64 n, i64 *out_k, i64 *out_c, i64 *scr_k, i64 *scr_c, i64 k,
                    double scale, double mean, double std, double zmin, i64 insertion_limit, i64 counting_limit,
                    i64 depth_guard, i64 *counters) {
    int err = 0;
    i64 *counts = (i64 *)calloc((size_t)k * 3, sizeof(i64));
    if (!counts) return ZO_ERR_NOMEM;
    i64 *offsets = counts + k, *cursors = counts + 2 * k;
    zo_histogram_pass(src_k, 0, n, mean, std, zmin, scale, k, counts);
    i64 occupied = 0;
    for (i64 b = 0; b < k; b++) occupied += counts[b] > 0;
    if (occupied <= 1) {
        copy_segment(src_k, src_c, 0, out_k, out_c, 0, n);
        zo_merge_sort_range(out_k, out_c, 0, n, scr_k, scr_c);
        counters[ST_FALLBACKS] += 1;
        free(counts);
        return ZO_OK;
    }
    zo_exclusive_offsets(counts, offsets, k);
    memcpy(cursors, offsets, (size_t)k * sizeof(i64));
    zo_scatter_pass(src_k, src_c, 0, n, mean, std, zmin, scale, k, cursors, scr_k, scr_c, 0);
    counters[ST_SCATTERS] += 1;
    if (counters[ST_MAX_DEPTH] < 1) counters[ST_MAX_DEPTH] = 1;

    stack_t_ st;
    if (stack_alloc(&st, depth_guard * k + 64) != ZO_OK) { stack_free(&st); free(counts); return ZO_ERR_NOMEM; }
    i64 top = 0;
    for (i64 b = 0; b < k; b++) {
        i64 cnt = counts[b];
        if (cnt == 0) continue;
        i64 gbase = offsets[b];
        if (cnt <= insertion_limit) {
            copy_segment(scr_k, scr_c, gbase, out_k, out_c, gbase, cnt);
            zo_insertion_sort_range(out_k, out_c, gbase, gbase + cnt);
            counters[ST_INSERTION] += 1;
        } else {
            top = dispatch_large_bucket(scr_k, scr_c, 1, gbase, cnt, b, mean, std, zmin, scale, k, 1, counting_limit,
                                        out_k, out_c, scr_k, scr_c, counters, &st, top, &err);
        }
    }
    run_worklist(out_k, out_c, scr_k, scr_c, k, scale, insertion_limit, counting_limit, depth_guard, counters, &st, top,
                 counts, offsets, cursors, &err);
    stack_free(&st);
    free(counts);
    return err;
}

/* _kernels.py:453-473 */
int zo_zsort_rec_driver(const i64 *src_k, const i64 *src_c, i64 n, i64 *out_k, i64 *out_c, i64 *scr_k, i64 *scr_c,
                        i64 k, double scale, double center, i64 level, i64 insertion_limit, i64 counting_limit,
                        i64 depth_guard, i64 *counters) {
    int err = 0;
    copy_segment(src_k, src_c, 0, scr_k, scr_c, 0, n);
    stack_t_ st;
    i64 *counts = (i64 *)calloc((size_t)k * 3, sizeof(i64));
    if (!counts || stack_alloc(&st, depth_guard * k + 64) != ZO_OK) { free(counts); return ZO_ERR_NOMEM; }
    st.base[0] = 0; st.cnt[0] = n; st.mean[0] = center; st.level[0] = level; st.scratch[0] = 1;
    run_worklist(out_k, out_c, scr_k, scr_c, k, scale, insertion_limit, counting_limit, depth_guard, counters, &st, 1,
                 counts, counts + k, counts + 2 * k, &err);
    stack_free(&st);
    free(counts);
    return err;
}

/* ------------------------------------------------------------ top level */

/* Correctly rounded fp64 of the exact rational a / n (n >= 1), i.e. Python's
 * int / int true division used for the mean at core.py:226. */
double zo_exact_div(i128 a, i64 n) {
    if (a == 0) return 0.0;
    int neg = a < 0;
    u128 A = neg ? (u128)(-(a + 1)) + 1u : (u128)a;
    u128 N = (u128)(u64)n;
    int s = 0;
    /* scale so the integer quotient carries >= 55 significant bits */
    u128 q = A / N;
    while (q < ((u128)1 << 54)) {
        s += 1;
        q = (A << s) / N;
    }
    u128 r = (A << s) % N;
    int bits = 0;
    for (u128 t = q; t; t >>= 1) bits++;
    int drop = bits - 53;
    u128 mant = q >> drop;
    u128 rem = q & (((u128)1 << drop) - 1);
    u128 half = (u128)1 << (drop - 1);
    int sticky = r != 0;
    if (rem > half || (rem == half && (sticky || (mant & 1)))) mant += 1;
    double v = ldexp((double)(u64)mant, drop - s);
    return neg ? -v : v;
}

/* core.py:196 + :226  mean = ((hi << 32) + lo) / n, correctly rounded */
double zo_mean_from_limbs(i64 sum_hi, i64 sum_lo, i64 n) {
    return zo_exact_div(((i128)sum_hi << 32) + (i128)sum_lo, n);
}

/* core.py:146-148  k = max(2, round(alpha * sqrt(n))) with banker's rounding */
i64 zo_cluster_count(i64 n, double alpha) {
    double v = nearbyint(alpha * sqrt((double)n));
    i64 k = (i64)v;
    return k < 2 ? 2 : k;
}

/* core.py:212-234  build_mapping_params from exact first-pass stats.
 * Returns 0 on success, 1 for DegenerateSpreadError. out = mean,std,zmin,scale */
int zo_mapping_params(const i64 *keys, i64 n, i64 k, double *out) {
    i64 shi, slo, mn, mx;
    zo_first_pass(keys, 0, n, &shi, &slo, &mn, &mx);
    i128 sum = ((i128)shi << 32) + (i128)slo;
    double mean = zo_exact_div(sum, n);
    double var = zo_variance_pass(keys, 0, n, mean);
    double std = sqrt(var);
    out[0] = mean; out[1] = std;
    if (!(std > 0.0) || !isfinite(std)) return 1;
    out[2] = fabs(((double)mn - mean) / std);
    out[3] = (double)k / 4.0;
    return 0;
}

/* core.py:348-400  zsort routing over an int64 carry column.
 * cfg = {alpha}, icfg = {insertion_threshold, counting_range_threshold, depth_guard} */
int zo_zsort(const i64 *keys, const i64 *carry, i64 n, i64 *out_k, i64 *out_c, double alpha, const i64 *icfg,
             i64 *counters) {
    i64 insertion = icfg[0], counting = icfg[1], guard = icfg[2];
    for (int i = 0; i < ST_SLOTS; i++) counters[i] = 0;
    if (n == 0) return ZO_OK;
    if (n <= insertion) {
        memcpy(out_k, keys, (size_t)n * sizeof(i64));
        memcpy(out_c, carry, (size_t)n * sizeof(i64));
        zo_insertion_sort_range(out_k, out_c, 0, n);
        counters[ST_INSERTION] = 1;
        return ZO_OK;
    }
    if (n > (i64)0x7FFFFFFF) return ZO_ERR_SIZE; /* core.py:193-194 */
    i64 shi, slo, mn, mx;
    zo_first_pass(keys, 0, n, &shi, &slo, &mn, &mx);
    i128 sum = ((i128)shi << 32) + (i128)slo;
    if (sum == (i128)mn * (i128)n) { /* all_equal, core.py:200-209 */
        memcpy(out_k, keys, (size_t)n * sizeof(i64));
        memcpy(out_c, carry, (size_t)n * sizeof(i64));
        return ZO_OK;
    }
    i64 k = zo_cluster_count(n, alpha);
    double mean = zo_exact_div(sum, n);
    double var = zo_variance_pass(keys, 0, n, mean);
    double std = sqrt(var);
    i64 *scr_k = (i64 *)malloc((size_t)n * sizeof(i64));
    i64 *scr_c = (i64 *)malloc((size_t)n * sizeof(i64));
    if (!scr_k || !scr_c) { free(scr_k); free(scr_c); return ZO_ERR_NOMEM; }
    int err;
    if (!(std > 0.0) || !isfinite(std)) { /* DegenerateSpreadError path, core.py:382-391 */
        memcpy(out_k, keys, (size_t)n * sizeof(i64));
        memcpy(out_c, carry, (size_t)n * sizeof(i64));
        zo_merge_sort_range(out_k, out_c, 0, n, scr_k, scr_c);
        counters[ST_FALLBACKS] = 1;
        err = ZO_OK;
    } else {
        double zmin = fabs(((double)mn - mean) / std);
        double scale = (double)k / 4.0;
        err = zo_zsort_driver(keys, carry, n, out_k, out_c, scr_k, scr_c, k, scale, mean, std, zmin, insertion,
                              counting, guard, counters);
    }
    free(scr_k); free(scr_c);
    return err;
}

/* core.py:403-437  zsort_rec over an int64 carry column (validated by caller) */
int zo_zsort_rec(const i64 *keys, const i64 *carry, i64 n, i64 *out_k, i64 *out_c, i64 k, double scale,
                 double mean_est, i64 depth, const i64 *icfg, i64 *counters) {
    for (int i = 0; i < ST_SLOTS; i++) counters[i] = 0;
    i64 *scr_k = (i64 *)malloc((size_t)n * sizeof(i64));
    i64 *scr_c = (i64 *)malloc((size_t)n * sizeof(i64));
    if (!scr_k || !scr_c) { free(scr_k); free(scr_c); return ZO_ERR_NOMEM; }
    int err = zo_zsort_rec_driver(keys, carry, n, out_k, out_c, scr_k, scr_c, k, scale, mean_est, depth + 1, icfg[0],
                                  icfg[1], icfg[2], counters);
    free(scr_k); free(scr_c);
    return err;
}

/* --------------------------------------------------------------- checks */

/* verify.py:55-108 structural stable-permutation check on ordered u64 keys.
 * in_ord/out_ord are order-preserving u64 images of the keys; out_p holds
 * the original index of each output record.  Returns the first failing index
 * as (kind << 56 | index): kind 1 = not sorted, 2 = out_p out of range or
 * repeated, 3 = key mismatch, 4 = stability violation; 0 when stable. */
u64 zo_check_stable_perm(const u64 *in_ord, const u64 *out_ord, const i64 *out_p, i64 n, uint8_t *bitmap) {
    memset(bitmap, 0, (size_t)((n + 7) / 8));
    for (i64 j = 0; j < n; j++) {
        i64 p = out_p[j];
        if (p < 0 || p >= n || (bitmap[p >> 3] >> (p & 7)) & 1) return ((u64)2 << 56) | (u64)j;
        bitmap[p >> 3] |= (uint8_t)(1u << (p & 7));
        if (in_ord[p] != out_ord[j]) return ((u64)3 << 56) | (u64)j;
        if (j > 0) {
            if (out_ord[j] < out_ord[j - 1]) return ((u64)1 << 56) | (u64)j;
            if (out_ord[j] == out_ord[j - 1] && out_p[j] <= out_p[j - 1]) return ((u64)4 << 56) | (u64)j;
        }
    }
    return 0;
}

/* ---------------------------------------------------------------- datagen */

/* _mt19937.py:24-48  MT19937-64 raw words (reference workload families). */
void zo_mt19937_64(u64 seed, u64 *out, i64 count) {
    enum { NN = 312, MM = 156 };
    const u64 MATRIX_A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    u64 mt[NN];
    mt[0] = seed;
    for (int i = 1; i < NN; i++) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (u64)i;
    int mti = NN;
    for (i64 j = 0; j < count; j++) {
        if (mti >= NN) {
            int i;
            u64 x;
            for (i = 0; i < NN - MM; i++) {
                x = (mt[i] & UM) | (mt[i + 1] & LM);
                mt[i] = mt[i + MM] ^ (x >> 1) ^ ((x & 1ULL) * MATRIX_A);
            }
            for (; i < NN - 1; i++) {
                x = (mt[i] & UM) | (mt[i + 1] & LM);
                mt[i] = mt[i + MM - NN] ^ (x >> 1) ^ ((x & 1ULL) * MATRIX_A);
            }
            x = (mt[NN - 1] & UM) | (mt[0] & LM);
            mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ ((x & 1ULL) * MATRIX_A);
            mti = 0;
        }
        u64 x = mt[mti++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= x >> 43;
        out[j] = x;
    }
}

/* _kernels.py:541-549 */
void zo_apply_index_swaps(i64 *keys, const i64 *pairs, i64 npairs) {
    for (i64 r = 0; r < npairs; r++) {
        i64 i = pairs[2 * r], j = pairs[2 * r + 1];
        i64 t = keys[i]; keys[i] = keys[j]; keys[j] = t;
    }
}
