// kernels.cuh -- sm_100a kernels of the stable z-score partitioning sort.
//
//  K1  k_moments        grid-wide fp64 moments + exact int sum -> level-1 params
//  K1s k_seg_moments    per-segment min/max/squared deviation (recursion levels)
//      k_seg_params     per-segment mapping parameters (one thread per segment)
//  K2  k_hist           per-tile bucket histogram -> bucket-major count matrix
//  K3  k_scan           single-pass decoupled-lookback exclusive scan
//  K4  k_scatter        stable scatter: warp match ranking + token ring
//      k_classify       bucket totals -> finish runs / next-level segments
//      k_plan           tiling and matrix layout of the next level
//  K5  k_finish         shared-memory stable finish of runs <= capacity
//
// Reference citations are /root/reference/pkg/src/zsort/<file>:<line>.
#pragma once

#include "common.cuh"

namespace zsb {

constexpr int NT = 256;        // threads per CTA for the streaming kernels
constexpr int NWARPS = NT / 32;
constexpr int SCAN_ITEMS = 16;  // entries per thread in k_scan
constexpr int SCAN_TILE = NT * SCAN_ITEMS;

struct Buffers {
    const uint64_t *in_k;
    const void *in_p;
    uint64_t *tmp_k;
    void *tmp_p;
    uint64_t *out_k;
    void *out_p;
};

__device__ __forceinline__ const uint64_t *src_keys(const Buffers &B, int src) {
    return src == 0 ? B.in_k : (src == 1 ? (const uint64_t *)B.tmp_k : (const uint64_t *)B.out_k);
}
template <int PB>
__device__ __forceinline__ const typename PayloadT<PB>::T *src_pay(const Buffers &B, int src) {
    using P = typename PayloadT<PB>::T;
    return src == 0 ? (const P *)B.in_p : (src == 1 ? (const P *)B.tmp_p : (const P *)B.out_p);
}

// Locate the segment owning tile `t` (segments sorted by tile_first).
__device__ __forceinline__ int find_seg(const SegParams *segs, int nseg, int64_t t) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (segs[mid].tile_first <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------------ exact mean
// Correctly rounded fp64 of (hi*2^32 + lo)/n: Python int/int true division
// of the exact first-pass sum (core.py:196,226).  Runs on one thread.
struct U128 {
    uint64_t hi, lo;
};
__device__ inline U128 u128_shl(U128 a, int s) {
    if (s == 0) return a;
    if (s >= 64) return {a.lo << (s - 64), 0};
    return {(a.hi << s) | (a.lo >> (64 - s)), a.lo << s};
}
// divide by d < 2^32 using 32-bit digits; returns quotient, sets remainder
__device__ inline U128 u128_div32(U128 a, uint32_t d, uint64_t *rem) {
    uint32_t dig[4] = {(uint32_t)(a.hi >> 32), (uint32_t)a.hi, (uint32_t)(a.lo >> 32), (uint32_t)a.lo};
    uint64_t r = 0;
    uint32_t q[4];
    for (int i = 0; i < 4; i++) {
        uint64_t cur = (r << 32) | dig[i];
        q[i] = (uint32_t)(cur / d);
        r = cur % d;
    }
    *rem = r;
    return {((uint64_t)q[0] << 32) | q[1], ((uint64_t)q[2] << 32) | q[3]};
}
__device__ inline bool u128_lt(U128 a, U128 b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }

__device__ inline double exact_mean(long long sum_hi, unsigned long long sum_lo, uint32_t n) {
    // S = sum_hi * 2^32 + sum_lo as signed 128-bit
    uint64_t hi = (uint64_t)(sum_hi >> 32);  // sign-extended high word of sum_hi*2^32
    uint64_t lo = (uint64_t)sum_hi << 32;
    uint64_t nlo = lo + sum_lo;
    hi += (nlo < lo) ? 1 : 0;
    lo = nlo;
    bool neg = (int64_t)hi < 0;
    if (neg) {  // two's complement negate
        lo = ~lo + 1;
        hi = ~hi + (lo == 0 ? 1 : 0);
    }
    if (hi == 0 && lo == 0) return 0.0;
    U128 A = {hi, lo};
    const U128 LIM = {0, 1ull << 54};
    uint64_t r;
    int s = 0;
    U128 q = u128_div32(A, n, &r);
    while (u128_lt(q, LIM)) {
        s++;
        q = u128_div32(u128_shl(A, s), n, &r);
    }
    int bits = q.hi ? 128 - __clzll((long long)q.hi) : 64 - __clzll((long long)q.lo);
    int drop = bits - 53;
    // q has <= 56 significant bits here unless the integer part was huge
    U128 mant = drop >= 64 ? U128{0, q.hi >> (drop - 64)}
                           : U128{q.hi >> drop, (q.lo >> drop) | (drop ? (q.hi << (64 - drop)) : 0)};
    uint64_t remb = drop >= 64 ? 0 : (q.lo & ((1ull << drop) - 1));  // drop < 64 in practice
    uint64_t half = 1ull << (drop - 1);
    bool sticky = r != 0;
    uint64_t m = mant.lo;
    if (remb > half || (remb == half && (sticky || (m & 1)))) m += 1;
    double v = ldexp((double)m, drop - s);
    return neg ? -v : v;
}

// --------------------------------------------------------- params finalize

struct MapCfg {
    int32_t mapping;      // 0 fitted, 1 paper
    int32_t depth_guard;  // levels before the exact integer split
};

// Decide the mapping of one segment from its center, variance and exact
// extremes (core.py:212-234 for level 1; _kernels.py:338-361 for recursion).
template <int KK>
__device__ void finalize_params(SegParams &p, double var, uint64_t omin, uint64_t omax, const MapCfg &mc,
                                unsigned long long *ctrl) {
    if (omin == omax) {  // all equal: copy through
        p.mode = MODE_COPY;
        return;
    }
    double sd = sqrt(var);
    double vmin = key_value<KK>(key_from_ord<KK>(omin));
    double vmax = key_value<KK>(key_from_ord<KK>(omax));
    bool ok = (sd > 0.0) && isfinite(sd) && p.mode == MODE_ZSCORE && p.level <= mc.depth_guard;
    p.std = sd;
    if (ok) {
        if (mc.mapping == 1) {  // paper Eq. 1: zmin = |min - mean| / std, scale = k / 4
            p.zmin = fabs(__ddiv_rn(__dsub_rn(vmin, p.center), sd));
            p.scale = (double)p.k / 4.0;
        } else {  // fitted: min -> 0, max -> just below k
            double span = __ddiv_rn(__dsub_rn(vmax, vmin), sd);
            ok = (span > 0.0) && isfinite(span);
            if (ok) {
                p.zmin = __ddiv_rn(__dsub_rn(p.center, vmin), sd);
                p.scale = ((double)p.k * (1.0 - 0x1p-20)) / span;
                ok = p.scale > 0.0 && isfinite(p.scale) && isfinite(p.zmin);
            }
        }
    }
    if (!ok) {  // degenerate spread / depth guard / non-splitting: exact MSD digit split
        if (p.mode != MODE_INTEGER && ctrl) atomicAdd(&ctrl[C_ST_FALLBACKS], 1ull);
        p.mode = MODE_INTEGER;
        p.umin = omin;
        int kb = 31 - __clz(p.k);  // floor(log2 k)
        int bl = bitlen64(omax - omin);
        p.shift = bl > kb ? bl - kb : 0;
    } else {
        p.mode = MODE_ZSCORE;
    }
}

// ------------------------------------------------------------------- K1

struct MomPartial {
    unsigned long long omin, omax;
    long long shi;
    unsigned long long slo;
    double s1, s2;
    unsigned long long nan;
    unsigned long long pad;
};

template <int KK>
__global__ void __launch_bounds__(NT) k_moments(const uint64_t *__restrict__ keys, int64_t n,
                                                MomPartial *__restrict__ parts, unsigned long long *ctrl,
                                                SegParams *seg, MapCfg mc, double *h_dbg) {
    const double c0 = key_value<KK>(keys[0]);
    unsigned long long omin = ~0ull, omax = 0, slo = 0, nan = 0;
    long long shi = 0;
    double s1 = 0.0, s2 = 0.0;
    const int64_t stride = (int64_t)gridDim.x * NT;
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint64_t b[4];
#pragma unroll
        for (int u = 0; u < 4; u++) b[u] = __ldcs(keys + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            uint64_t o = ord_key<KK>(b[u]);
            omin = o < omin ? o : omin;
            omax = o > omax ? o : omax;
            if constexpr (KK == KEY_I64) {
                shi += (long long)b[u] >> 32;
                slo += b[u] & 0xFFFFFFFFull;
            }
            double x = key_value<KK>(b[u]);
            if (KK == KEY_F64 && x != x) {
                nan++;
            } else {
                double d = x - c0;
                s1 += d;
                s2 += d * d;
            }
        }
    }
    for (; i < n; i += stride) {
        uint64_t b = __ldcs(keys + i);
        uint64_t o = ord_key<KK>(b);
        omin = o < omin ? o : omin;
        omax = o > omax ? o : omax;
        if constexpr (KK == KEY_I64) {
            shi += (long long)b >> 32;
            slo += b & 0xFFFFFFFFull;
        }
        double x = key_value<KK>(b);
        if (KK == KEY_F64 && x != x) {
            nan++;
        } else {
            double d = x - c0;
            s1 += d;
            s2 += d * d;
        }
    }
    // warp shuffles, then one partial per CTA
    omin = warp_min_u64(omin);
    omax = warp_max_u64(omax);
    shi = warp_sum(shi);
    slo = warp_sum(slo);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    nan = warp_sum(nan);
    __shared__ MomPartial wp[NWARPS];
    __shared__ bool last;
    int w = threadIdx.x >> 5;
    if (lane_id() == 0) wp[w] = {omin, omax, shi, slo, s1, s2, nan, 0};
    __syncthreads();
    if (threadIdx.x == 0) {
        MomPartial acc = wp[0];
        for (int j = 1; j < NWARPS; j++) {
            acc.omin = wp[j].omin < acc.omin ? wp[j].omin : acc.omin;
            acc.omax = wp[j].omax > acc.omax ? wp[j].omax : acc.omax;
            acc.shi += wp[j].shi;
            acc.slo += wp[j].slo;
            acc.s1 += wp[j].s1;
            acc.s2 += wp[j].s2;
            acc.nan += wp[j].nan;
        }
        parts[blockIdx.x] = acc;
        __threadfence();
        unsigned long long t = atomicAdd(&ctrl[C_MOM_TICKET], 1ull);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // last CTA: reduce the partials (warp 0), then finalize on thread 0
    if (w != 0) return;
    MomPartial acc{~0ull, 0, 0, 0, 0.0, 0.0, 0, 0};
    for (int j = lane_id(); j < (int)gridDim.x; j += 32) {
        MomPartial q;
        q.omin = __ldcg(&parts[j].omin);
        q.omax = __ldcg(&parts[j].omax);
        q.shi = __ldcg(&parts[j].shi);
        q.slo = __ldcg(&parts[j].slo);
        q.s1 = __ldcg(&parts[j].s1);
        q.s2 = __ldcg(&parts[j].s2);
        q.nan = __ldcg(&parts[j].nan);
        acc.omin = q.omin < acc.omin ? q.omin : acc.omin;
        acc.omax = q.omax > acc.omax ? q.omax : acc.omax;
        acc.shi += q.shi;
        acc.slo += q.slo;
        acc.s1 += q.s1;
        acc.s2 += q.s2;
        acc.nan += q.nan;
    }
    acc.omin = warp_min_u64(acc.omin);
    acc.omax = warp_max_u64(acc.omax);
    acc.shi = warp_sum(acc.shi);
    acc.slo = warp_sum(acc.slo);
    acc.s1 = warp_sum(acc.s1);
    acc.s2 = warp_sum(acc.s2);
    acc.nan = warp_sum(acc.nan);
    if (lane_id() != 0) return;
    ctrl[C_MOM_TICKET] = 0;
    if (acc.nan) {
        ctrl[C_STATUS] = 3;  // ZSB_ERR_NAN
        seg->mode = MODE_COPY;
        return;
    }
    double dn = (double)n;
    double mean;
    if constexpr (KK == KEY_I64) {
        mean = exact_mean(acc.shi, acc.slo, (uint32_t)n);
    } else {
        mean = c0 + acc.s1 / dn;
    }
    // mean squared deviation around the mean from sums around c0
    double dm = mean - c0;
    double m2 = acc.s2 - 2.0 * dm * acc.s1 + dn * dm * dm;
    if (m2 < 0.0) m2 = 0.0;
    SegParams p = *seg;
    p.center = mean;
    p.mode = MODE_ZSCORE;
    finalize_params<KK>(p, m2 / dn, acc.omin, acc.omax, mc, ctrl);
    *seg = p;
    if (h_dbg) {
        h_dbg[0] = dn;
        h_dbg[1] = mean;
        h_dbg[2] = m2;
        h_dbg[3] = key_value<KK>(key_from_ord<KK>(acc.omin));
        h_dbg[4] = key_value<KK>(key_from_ord<KK>(acc.omax));
        h_dbg[5] = (double)acc.shi;
        h_dbg[6] = (double)acc.slo;
        h_dbg[7] = (double)acc.nan;
        ((long long *)h_dbg)[8] = acc.shi;
        ((unsigned long long *)h_dbg)[9] = acc.slo;
        ((unsigned long long *)h_dbg)[10] = key_from_ord<KK>(acc.omin);
        ((unsigned long long *)h_dbg)[11] = key_from_ord<KK>(acc.omax);
    }
}

// ------------------------------------------------------------------ K1s

template <int KK>
__global__ void __launch_bounds__(NT) k_seg_moments(Buffers B, const SegParams *__restrict__ segs, int nseg,
                                                    SegAcc *acc) {
    int s = find_seg(segs, nseg, blockIdx.x);
    const SegParams &p = segs[s];
    if (p.mode == MODE_COPY) return;
    int64_t ti = blockIdx.x - p.tile_first;
    int64_t t0 = p.start + ti * p.tile_len;
    int64_t t1 = min(t0 + p.tile_len, p.start + p.len);
    const uint64_t *src = src_keys(B, p.src);
    const double c = p.center;
    unsigned long long omin = ~0ull, omax = 0;
    double s2 = 0.0;
    for (int64_t i = t0 + threadIdx.x; i < t1; i += NT) {
        uint64_t b = src[i];
        uint64_t o = ord_key<KK>(b);
        omin = o < omin ? o : omin;
        omax = o > omax ? o : omax;
        double d = key_value<KK>(b) - c;
        s2 += d * d;
    }
    omin = warp_min_u64(omin);
    omax = warp_max_u64(omax);
    s2 = warp_sum(s2);
    __shared__ unsigned long long smin[NWARPS], smax[NWARPS];
    __shared__ double ss[NWARPS];
    int w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        smin[w] = omin;
        smax[w] = omax;
        ss[w] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 1; j < NWARPS; j++) {
            omin = smin[j] < omin ? smin[j] : omin;
            omax = smax[j] > omax ? smax[j] : omax;
            s2 += ss[j];
        }
        atomicMin(&acc[s].omin, omin);
        atomicMax(&acc[s].omax, omax);
        atomicAdd(&acc[s].s2, s2);
    }
}

template <int KK>
__global__ void k_seg_params(SegParams *segs, int nseg, const SegAcc *acc, MapCfg mc, unsigned long long *ctrl) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    SegParams p = segs[s];
    if (p.mode == MODE_COPY) return;
    finalize_params<KK>(p, acc[s].s2 / (double)p.len, acc[s].omin, acc[s].omax, mc, ctrl);
    segs[s] = p;
}

// ------------------------------------------------------------------- K2

template <int KK>
__global__ void __launch_bounds__(NT) k_hist(Buffers B, const SegParams *__restrict__ segs, int nseg,
                                             uint32_t *__restrict__ mat) {
    extern __shared__ uint32_t hist[];
    int s = find_seg(segs, nseg, blockIdx.x);
    const SegParams p = segs[s];
    int64_t ti = blockIdx.x - p.tile_first;
    int64_t t0 = p.start + ti * p.tile_len;
    int64_t t1 = min(t0 + p.tile_len, p.start + p.len);
    uint32_t *col = mat + p.mat_base + ti;
    if (p.mode == MODE_COPY) {  // one bucket holds the whole tile
        for (int b = threadIdx.x; b < p.k; b += NT) col[(int64_t)b * p.ntiles] = b == 0 ? (uint32_t)(t1 - t0) : 0u;
        return;
    }
    for (int b = threadIdx.x; b < p.k; b += NT) hist[b] = 0;
    __syncthreads();
    const uint64_t *src = src_keys(B, p.src);
    const int lane = lane_id();
    // warp-uniform trip counts: every lane reaches each __match_any_sync
    int64_t i0 = t0 + (threadIdx.x & ~31);
    for (; i0 + 3 * NT + 31 < t1; i0 += 4 * NT) {
        uint64_t b[4];
#pragma unroll
        for (int u = 0; u < 4; u++) b[u] = __ldcs(src + i0 + u * NT + lane);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            int32_t bk = seg_bucket<KK>(b[u], p);
            unsigned peers = __match_any_sync(0xffffffffu, bk);
            if ((peers & lanemask_lt()) == 0) atomicAdd(&hist[bk], (uint32_t)__popc(peers));
        }
    }
    for (; i0 < t1; i0 += NT) {
        int64_t i = i0 + lane;
        int32_t bk = i < t1 ? seg_bucket<KK>(__ldcs(src + i), p) : -1;
        unsigned peers = __match_any_sync(0xffffffffu, bk);
        if (bk >= 0 && (peers & lanemask_lt()) == 0) atomicAdd(&hist[bk], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < p.k; b += NT) col[(int64_t)b * p.ntiles] = hist[b];
}

// ------------------------------------------------------------------- K3
// Exclusive scan of `total` uint32 entries in place; single pass with
// decoupled look-back (status word = flag<<62 | inclusive-or-aggregate).

constexpr unsigned long long FLAG_AGG = 1ull << 62;
constexpr unsigned long long FLAG_PRE = 2ull << 62;
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

__global__ void __launch_bounds__(NT) k_scan(uint32_t *data, int64_t total, unsigned long long *status,
                                             unsigned long long *ctrl) {
    __shared__ uint32_t s_bid;
    __shared__ unsigned long long s_warp[NWARPS];
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_bid = (uint32_t)atomicAdd(&ctrl[C_SCAN_TICKET], 1ull);
    __syncthreads();
    const int64_t bid = s_bid;
    const int64_t base = bid * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    unsigned long long tsum = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        v[j] = (base + j < total) ? data[base + j] : 0u;
        tsum += v[j];
    }
    // block exclusive scan of thread sums
    unsigned long long x = tsum;
    int lane = lane_id(), w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    unsigned long long wpre = 0, agg = 0;
    for (int j = 0; j < NWARPS; j++) {
        if (j < w) wpre += s_warp[j];
        agg += s_warp[j];
    }
    unsigned long long texcl = wpre + x - tsum;
    // publish aggregate and look back (warp 0)
    if (w == 0) {
        volatile unsigned long long *vs = status;
        if (bid == 0) {
            if (lane == 0) {
                vs[0] = FLAG_PRE | agg;
                s_prefix = 0;
            }
        } else {
            if (lane == 0) vs[bid] = FLAG_AGG | agg;
            unsigned long long excl = 0;
            int64_t j = bid - 1;
            while (true) {
                int64_t idx = j - lane;
                unsigned long long st = 0;
                if (idx >= 0) {
                    do {
                        st = vs[idx];
                    } while ((st >> 62) == 0);
                } else {
                    st = FLAG_PRE;  // virtual prefix 0 before the first tile
                }
                unsigned pre = __ballot_sync(0xffffffffu, (st >> 62) == 2);
                int stop = pre ? __ffs(pre) - 1 : 32;  // nearest inclusive prefix
                unsigned long long val = (lane <= stop) ? (st & VAL_MASK) : 0ull;
                excl += warp_sum(val);
                if (pre) break;
                j -= 32;
            }
            if (lane == 0) {
                __threadfence();
                vs[bid] = FLAG_PRE | (excl + agg);
                s_prefix = excl;
            }
        }
    }
    __syncthreads();
    unsigned long long run = s_prefix + texcl;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        if (base + j < total) data[base + j] = (uint32_t)run;
        run += v[j];
    }
}

// ------------------------------------------------------------------- K4
// Stable scatter.  Each CTA owns one tile (a contiguous input range) and
// starts from its column of the scanned count matrix, so tiles land in
// input order inside every bucket.  Inside the CTA the 8 warps take turns
// (a token ring over named barriers) to advance the per-bucket cursors in
// shared memory, and inside a warp equal-bucket keys are ranked by
// __match_any_sync + popc(peers & lanemask_lt): every record keeps its input
// order within its bucket (_kernels.py:124-133 front-to-back semantics).

template <int KK, int PB, int ITEMS>
__global__ void __launch_bounds__(NT) k_scatter(Buffers B, const SegParams *__restrict__ segs, int nseg,
                                                const uint32_t *__restrict__ mat, int dst_sel) {
    using P = typename PayloadT<PB>::T;
    extern __shared__ uint32_t cur[];
    int s = find_seg(segs, nseg, blockIdx.x);
    const SegParams p = segs[s];
    int64_t ti = blockIdx.x - p.tile_first;
    int64_t t0 = p.start + ti * p.tile_len;
    int64_t t1 = min(t0 + p.tile_len, p.start + p.len);
    const uint64_t *sk = src_keys(B, p.src);
    const P *sp = src_pay<PB>(B, p.src);
    if (p.mode == MODE_COPY) {  // all-equal segment: land it in the output directly
        if (p.src == 2) return;
        P *op = (P *)B.out_p;
        for (int64_t i = t0 + threadIdx.x; i < t1; i += NT) {
            B.out_k[i] = sk[i];
            if constexpr (PB != 0) op[i] = sp[i];
        }
        return;
    }
    uint64_t *dk = dst_sel == 1 ? B.tmp_k : B.out_k;
    P *dp = (P *)(dst_sel == 1 ? B.tmp_p : B.out_p);
    const uint32_t *col = mat + p.mat_base + ti;
    const uint32_t adj = (uint32_t)(p.start - p.scan_base);
    for (int b = threadIdx.x; b < p.k; b += NT) cur[b] = col[(int64_t)b * p.ntiles] + adj;
    __syncthreads();

    const int w = threadIdx.x >> 5, lane = lane_id();
    const unsigned lt = lanemask_lt();
    constexpr int R = NT * ITEMS;
    const int64_t nr = (t1 - t0 + R - 1) / R;
    for (int64_t r = 0; r < nr; r++) {
        const int64_t base = t0 + r * R + (int64_t)w * (32 * ITEMS) + lane;
        uint64_t key[ITEMS];
        P pay[ITEMS];
        int32_t bk[ITEMS];
        unsigned peers[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; j++) {
            int64_t idx = base + j * 32;
            bool v = idx < t1;
            key[j] = v ? __ldcs(sk + idx) : 0ull;
            if constexpr (PB != 0) pay[j] = v ? __ldcs(sp + idx) : (P)0;
            bk[j] = v ? seg_bucket<KK>(key[j], p) : -1;
        }
#pragma unroll
        for (int j = 0; j < ITEMS; j++) peers[j] = __match_any_sync(0xffffffffu, bk[j]);
        // ---- critical section: cursor advance in (warp, item, lane) order
        if (!(r == 0 && w == 0)) named_bar_sync(1 + w, 64);
        uint32_t pos0[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; j++) {
            pos0[j] = 0;
            if (bk[j] >= 0 && (peers[j] & lt) == 0) {
                uint32_t c = cur[bk[j]];
                pos0[j] = c;
                cur[bk[j]] = c + __popc(peers[j]);
            }
            __syncwarp();
        }
        if (!(w == NWARPS - 1 && r == nr - 1)) {
            __threadfence_block();
            named_bar_arrive(1 + ((w + 1) & (NWARPS - 1)), 64);
        }
        // ---- scatter
#pragma unroll
        for (int j = 0; j < ITEMS; j++) {
            int leader = __ffs(peers[j]) - 1;
            uint32_t b0 = __shfl_sync(0xffffffffu, pos0[j], leader);
            if (bk[j] >= 0) {
                uint32_t pos = b0 + __popc(peers[j] & lt);
                dk[pos] = key[j];
                if constexpr (PB != 0) dp[pos] = pay[j];
            }
        }
    }
}

// ------------------------------------------------------------ classify

struct ClassCfg {
    int32_t cap;        // finish capacity (records)
    int32_t half;       // grouping window
    int32_t depth_guard;
    int32_t mapping;
};

__device__ __forceinline__ int64_t bucket_start(const SegParams &p, const uint32_t *mat, int b) {
    if (b >= p.k) return p.start + p.len;
    return p.start + (int64_t)mat[p.mat_base + (int64_t)b * p.ntiles] - p.scan_base;
}

// One thread per (segment, bucket): bucket runs <= capacity become finish
// entries (whole buckets only, grouped within a window so each entry stays
// <= cap); larger buckets become next-level segments with the bucket's
// estimated center (_kernels.py:282-318, 103-106).
__global__ void k_classify(const SegParams *__restrict__ segs, int nseg, const int64_t *__restrict__ kfirst,
                           const uint32_t *__restrict__ mat, Entry *entries, SegParams *children, SegAcc *acc,
                           unsigned long long *ctrl, ClassCfg cc, int64_t total_buckets) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= total_buckets) return;
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (kfirst[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    const SegParams &p = segs[lo];
    int b = (int)(g - kfirst[lo]);
    if (p.mode == MODE_COPY) return;
    if (b == 0) {
        atomicAdd(&ctrl[C_ST_SCATTERS], 1ull);
        atomicMax(&ctrl[C_ST_MAXDEPTH], (unsigned long long)p.level);
    }
    const int dst = (p.src == 1) ? 2 : 1;
    int64_t st = bucket_start(p, mat, b);
    int64_t c = bucket_start(p, mat, b + 1) - st;
    if (c > cc.cap) {
        SegParams ch{};
        ch.start = st;
        ch.len = c;
        ch.level = p.level + 1;
        ch.src = dst;
        ch.k = p.k;
        bool integer = p.mode == MODE_INTEGER || c == p.len || ch.level > cc.depth_guard;
        if (integer) {
            ch.mode = MODE_INTEGER;
            atomicAdd(&ctrl[C_ST_FALLBACKS], 1ull);
        } else {
            ch.mode = MODE_ZSCORE;
            // estimated center of bucket b (_kernels.py:103-106)
            ch.center = __dadd_rn(__dmul_rn(__dsub_rn(__ddiv_rn((double)b + 0.5, p.scale), p.zmin), p.std), p.center);
        }
        unsigned long long slot = atomicAdd(&ctrl[C_NCHILD], 1ull);
        children[slot] = ch;
        acc[slot] = SegAcc{~0ull, 0ull, 0.0, 0.0};
        return;
    }
    if (c > cc.half) {
        unsigned long long e = atomicAdd(&ctrl[C_NENTRY], 1ull);
        entries[e] = Entry{st, (int32_t)c, dst};
        return;
    }
    // groupable bucket: does it start a run?
    int64_t win = (st - p.start) / cc.half;
    bool starts = true;
    if (b > 0) {
        int64_t pst = bucket_start(p, mat, b - 1);
        int64_t pc = st - pst;
        starts = pc > cc.half || (pst - p.start) / cc.half != win;
    }
    if (!starts) return;
    int64_t end = st + c;
    for (int b2 = b + 1; b2 < p.k; b2++) {
        int64_t s2 = end;
        int64_t e2 = bucket_start(p, mat, b2 + 1);
        if (e2 - s2 > cc.half || (s2 - p.start) / cc.half != win) break;
        end = e2;
    }
    if (end > st) {
        unsigned long long e = atomicAdd(&ctrl[C_NENTRY], 1ull);
        entries[e] = Entry{st, (int32_t)(end - st), dst};
    }
}

// ----------------------------------------------------------------- plan
// Tiling and matrix layout of the next level (single CTA, prefix sums over
// the children).  Children keep the parent's k in paper mode (the reference
// keeps k fixed across levels, core.py:355); fitted mode sizes k to the
// child so its buckets average ~cap/4 records.
__global__ void __launch_bounds__(1024) k_plan(SegParams *segs, const unsigned long long *nseg_ptr, int64_t *kfirst,
                                               unsigned long long *ctrl, int32_t mapping, int32_t cap,
                                               int32_t kmax_child, int32_t min_tile) {
    (void)mapping;
    const int nseg = (int)*nseg_ptr;
    __shared__ long long sh_t[32], sh_m[32], sh_l[32], sh_k[32];
    __shared__ long long carry_t, carry_m, carry_l, carry_k;
    __shared__ int kmax;
    if (threadIdx.x == 0) {
        carry_t = carry_m = carry_l = carry_k = 0;
        kmax = 1;
    }
    __syncthreads();
    for (int base = 0; base < nseg; base += 1024) {
        int s = base + threadIdx.x;
        long long nt = 0, nm = 0, ln = 0, kk = 0;
        SegParams p;
        if (s < nseg) {
            p = segs[s];
            // k sized to the child so buckets average ~cap/4 records (both
            // mappings; the reference's fixed k is a CPU choice, core.py:355)
            int64_t want = (p.len * 4 + cap - 1) / cap;
            int k = 16;
            while (k < want && k < kmax_child) k <<= 1;
            p.k = k;
            int64_t tl = max((int64_t)min_tile, (int64_t)4 * k);
            tl = (tl + 255) & ~(int64_t)255;
            p.tile_len = tl;
            p.ntiles = (int32_t)((p.len + tl - 1) / tl);
            nt = p.ntiles;
            nm = (long long)p.ntiles * k;
            ln = p.len;
            kk = k;
            atomicMax(&kmax, k);
        }
        // block inclusive scans of (nt, nm, ln, kk)
        long long a = nt, m = nm, l = ln, q = kk;
        int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            long long ya = __shfl_up_sync(0xffffffffu, a, o), ym = __shfl_up_sync(0xffffffffu, m, o);
            long long yl = __shfl_up_sync(0xffffffffu, l, o), yq = __shfl_up_sync(0xffffffffu, q, o);
            if (lane >= o) {
                a += ya;
                m += ym;
                l += yl;
                q += yq;
            }
        }
        if (lane == 31) {
            sh_t[w] = a;
            sh_m[w] = m;
            sh_l[w] = l;
            sh_k[w] = q;
        }
        __syncthreads();
        long long pa = carry_t, pm = carry_m, pl = carry_l, pq = carry_k;
        for (int j = 0; j < w; j++) {
            pa += sh_t[j];
            pm += sh_m[j];
            pl += sh_l[j];
            pq += sh_k[j];
        }
        if (s < nseg) {
            p.tile_first = pa + a - nt;
            p.mat_base = pm + m - nm;
            p.scan_base = pl + l - ln;
            kfirst[s] = pq + q - kk;
            segs[s] = p;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            carry_t = pa + a;
            carry_m = pm + m;
            carry_l = pl + l;
            carry_k = pq + q;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctrl[C_TILES_NEXT] = carry_t;
        ctrl[C_MAT_NEXT] = carry_m;
        ctrl[C_KMAX_NEXT] = kmax;
        ctrl[C_NEXT_BIG] = carry_k;
        kfirst[nseg] = carry_k;
    }
}

// ------------------------------------------------------------------- K5
// Shared-memory stable finish of one entry (a run of whole buckets,
// len <= cap): load keys + payload, split by the top bits of
// (ord(key) - ord(min)) into sub-buckets with a stable warp-ranked counting
// pass (per-warp u16 counters, block scan), insertion-sort the tiny
// sub-buckets (only strictly greater keys shift, _kernels.py:143-156), and a
// warp bitonic network on (key, original position) for the rare large ones.
// Everything is staged in shared memory, so src may alias the output.

constexpr int FIN_INS = 24;  // sub-buckets up to this size use insertion sort

struct FinLayout {
    int cap, sb_max;
    size_t off_a, off_b, off_pl, off_i, off_cnt, off_st, off_q, total;
};

__host__ __device__ inline FinLayout fin_layout(int cap, int pb, int sb_max) {
    FinLayout L;
    L.cap = cap;
    L.sb_max = sb_max;
    size_t o = 0;
    L.off_a = o;
    o += (size_t)cap * 8;
    L.off_b = o;
    o += (size_t)cap * 8;
    L.off_pl = o;
    o += (size_t)cap * pb;
    o = (o + 15) & ~(size_t)15;
    L.off_i = o;
    o += (size_t)cap * 2;
    o = (o + 15) & ~(size_t)15;
    L.off_cnt = o;
    o += (size_t)sb_max * NWARPS * 2;
    L.off_st = o;
    o += (size_t)(sb_max + 1) * 2;
    o = (o + 15) & ~(size_t)15;
    L.off_q = o;
    o += (size_t)1024 * 4;
    L.total = o;
    return L;
}

template <int KK>
__device__ __forceinline__ bool kless(uint64_t a, uint16_t ia, uint64_t b, uint16_t ib) {
    uint64_t oa = ord_key<KK>(a), ob = ord_key<KK>(b);
    return oa < ob || (oa == ob && ia < ib);
}

template <int KK, int PB>
__global__ void __launch_bounds__(NT) k_finish(Buffers B, const Entry *__restrict__ entries, int cap, int sb_max) {
    using P = typename PayloadT<PB>::T;
    extern __shared__ __align__(16) unsigned char smem[];
    const FinLayout L = fin_layout(cap, PB, sb_max);
    uint64_t *A = (uint64_t *)(smem + L.off_a);
    uint64_t *Bk = (uint64_t *)(smem + L.off_b);
    P *PL = (P *)(smem + L.off_pl);
    uint16_t *I = (uint16_t *)(smem + L.off_i);
    uint16_t *cnt = (uint16_t *)(smem + L.off_cnt);
    uint16_t *sst = (uint16_t *)(smem + L.off_st);
    int *q = (int *)(smem + L.off_q);
    __shared__ unsigned long long r_min[NWARPS], r_max[NWARPS];
    __shared__ int nq;

    const Entry e = entries[blockIdx.x];
    const int m = e.len;
    const uint64_t *sk = src_keys(B, e.src) + e.start;
    const P *sp = src_pay<PB>(B, e.src) + e.start;
    uint64_t *ok = B.out_k + e.start;
    P *op = (P *)B.out_p + e.start;
    const int tid = threadIdx.x, w = tid >> 5, lane = lane_id();

    unsigned long long omin = ~0ull, omax = 0;
    for (int i = tid; i < m; i += NT) {
        uint64_t k = sk[i];
        A[i] = k;
        if constexpr (PB != 0) PL[i] = sp[i];
        uint64_t o = ord_key<KK>(k);
        omin = o < omin ? o : omin;
        omax = o > omax ? o : omax;
    }
    omin = warp_min_u64(omin);
    omax = warp_max_u64(omax);
    if (lane == 0) {
        r_min[w] = omin;
        r_max[w] = omax;
    }
    if (tid == 0) nq = 0;
    __syncthreads();
    omin = r_min[0];
    omax = r_max[0];
    for (int j = 1; j < NWARPS; j++) {
        omin = r_min[j] < omin ? r_min[j] : omin;
        omax = r_max[j] > omax ? r_max[j] : omax;
    }
    if (omin == omax) {  // all equal: already in stable order
        if (e.src != 2) {
            for (int i = tid; i < m; i += NT) {
                ok[i] = A[i];
                if constexpr (PB != 0) op[i] = PL[i];
            }
        }
        return;
    }
    // sub-bucket count: ~m/4, power of two, <= sb_max
    int sbits = 5;
    while ((1 << sbits) < (m >> 2) && (1 << sbits) < sb_max) sbits++;
    const int S = 1 << sbits;
    const uint64_t range = omax - omin;
    const int bl = bitlen64(range);
    const int sh = bl > sbits ? bl - sbits : 0;
    const bool exact = (sh == 0);  // each sub-bucket holds one key value
    const int nc = S * NWARPS;
    for (int i = tid; i < nc; i += NT) cnt[i] = 0;
    __syncthreads();
    // warp w owns the contiguous slice [w0, w1) of the entry (input order)
    const int per = (m + NWARPS - 1) / NWARPS;
    const int w0 = min(m, w * per), w1 = min(m, w0 + per);
    const unsigned lt = lanemask_lt();
    for (int i0 = w0; i0 < w1; i0 += 32) {
        int i = i0 + lane;
        int sbk = i < w1 ? (int)((ord_key<KK>(A[i]) - omin) >> sh) : -1;
        unsigned peers = __match_any_sync(0xffffffffu, sbk);
        if (sbk >= 0 && (peers & lt) == 0) cnt[sbk * NWARPS + w] += (uint16_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // block exclusive scan over cnt in (sub-bucket, warp) order
    {
        const int per_t = nc / NT;  // nc is a multiple of NT (S >= 32, NWARPS = 8)
        const int c0 = tid * per_t;
        uint32_t tsum = 0;
        for (int j = 0; j < per_t; j++) tsum += cnt[c0 + j];
        uint32_t x = tsum;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __shared__ uint32_t wsum[NWARPS];
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        uint32_t pre = 0;
        for (int j = 0; j < w; j++) pre += wsum[j];
        uint32_t run = pre + x - tsum;
        for (int j = 0; j < per_t; j++) {
            uint16_t c = cnt[c0 + j];
            cnt[c0 + j] = (uint16_t)run;
            run += c;
        }
    }
    __syncthreads();
    for (int sbk = tid; sbk < S; sbk += NT) sst[sbk] = cnt[sbk * NWARPS];
    if (tid == 0) sst[S] = (uint16_t)m;
    __syncthreads();
    // stable placement
    for (int i0 = w0; i0 < w1; i0 += 32) {
        int i = i0 + lane;
        uint64_t k = i < w1 ? A[i] : 0ull;
        int sbk = i < w1 ? (int)((ord_key<KK>(k) - omin) >> sh) : -1;
        unsigned peers = __match_any_sync(0xffffffffu, sbk);
        int leader = __ffs(peers) - 1;
        uint32_t b0 = 0;
        if (sbk >= 0 && lane == leader) {
            b0 = cnt[sbk * NWARPS + w];
            cnt[sbk * NWARPS + w] = (uint16_t)(b0 + __popc(peers));
        }
        b0 = __shfl_sync(0xffffffffu, b0, leader);
        if (sbk >= 0) {
            uint32_t pos = b0 + __popc(peers & lt);
            Bk[pos] = k;
            I[pos] = (uint16_t)i;
        }
        __syncwarp();
    }
    __syncthreads();
    if (!exact) {
        for (int sbk = tid; sbk < S; sbk += NT) {
            int a = sst[sbk], z = sst[sbk + 1];
            int c = z - a;
            if (c <= 1) continue;
            if (c <= FIN_INS) {
                for (int x = a + 1; x < z; x++) {
                    uint64_t kv = Bk[x];
                    uint16_t iv = I[x];
                    uint64_t ov = ord_key<KK>(kv);
                    int y = x - 1;
                    while (y >= a && ord_key<KK>(Bk[y]) > ov) {
                        Bk[y + 1] = Bk[y];
                        I[y + 1] = I[y];
                        y--;
                    }
                    Bk[y + 1] = kv;
                    I[y + 1] = iv;
                }
            } else {
                int slot = atomicAdd(&nq, 1);
                if (slot < 1024) q[slot] = sbk;
            }
        }
        __syncthreads();
        const int nbig = min(nq, 1024);
        for (int t = w; t < nbig; t += NWARPS) {
            int a = sst[q[t]], z = sst[q[t] + 1];
            int c = z - a;
            // already ordered (incl. all-equal)?  placement kept input order
            bool sorted = true;
            for (int x = a + lane; x + 1 < z; x += 32)
                if (ord_key<KK>(Bk[x]) > ord_key<KK>(Bk[x + 1])) sorted = false;
            if (__all_sync(0xffffffffu, sorted)) continue;
            // bitonic network with all comparators ascending; virtual +inf padding
            int P2 = 1;
            while (P2 < c) P2 <<= 1;
            for (int size = 2; size <= P2; size <<= 1) {
                for (int x = lane; x < P2 / 2; x += 32) {  // flip stage
                    int blk = x / (size / 2), off = x % (size / 2);
                    int i1 = blk * size + off, i2 = blk * size + size - 1 - off;
                    if (i2 < c) {
                        uint64_t k1 = Bk[a + i1], k2 = Bk[a + i2];
                        uint16_t j1 = I[a + i1], j2 = I[a + i2];
                        if (kless<KK>(k2, j2, k1, j1)) {
                            Bk[a + i1] = k2;
                            Bk[a + i2] = k1;
                            I[a + i1] = j2;
                            I[a + i2] = j1;
                        }
                    }
                }
                __syncwarp();
                for (int str = size / 4; str >= 1; str >>= 1) {  // half cleaners
                    for (int x = lane; x < P2 / 2; x += 32) {
                        int blk = x / str, off = x % str;
                        int i1 = blk * 2 * str + off, i2 = i1 + str;
                        if (i2 < c) {
                            uint64_t k1 = Bk[a + i1], k2 = Bk[a + i2];
                            uint16_t j1 = I[a + i1], j2 = I[a + i2];
                            if (kless<KK>(k2, j2, k1, j1)) {
                                Bk[a + i1] = k2;
                                Bk[a + i2] = k1;
                                I[a + i1] = j2;
                                I[a + i2] = j1;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < m; i += NT) {
        ok[i] = Bk[i];
        if constexpr (PB != 0) op[i] = PL[I[i]];
    }
}

// Entry builder for the small-n path (one finish over the whole input).
__global__ void k_single_entry(Entry *entries, int64_t n) { entries[0] = Entry{0, (int32_t)n, 0}; }

}  // namespace zsb
