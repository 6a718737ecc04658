// sort_kernels.cuh -- sm_100a kernels of the stable z-score partitioning sort.
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

#include <cooperative_groups.h>
#include <type_traits>
namespace cg = cooperative_groups;

#include "common.cuh"

namespace zsb {

constexpr int NT = 256;        // threads per CTA for the streaming kernels
#ifndef ZSB_BM_ZSCORE
#define ZSB_BM_ZSCORE 1  // z-score segments (recursion levels) run a body specialised to Eq. 1
#endif
#ifndef ZSB_ZLIN
#define ZSB_ZLIN 1  // fitted recursion levels map with Eq. 1's line in fp32 (MODE_ZLIN, own body)
#endif
#ifndef ZSB_EXP_NOSTORE
#define ZSB_EXP_NOSTORE 0  // what-if experiments (wrong results): scatter without its global stores
#endif
#ifndef ZSB_HIST_UNROLL
#define ZSB_HIST_UNROLL 8  // keys per thread in flight in the recursion-level histogram (per-thread loads)
#endif
#ifndef ZSB_SCAT_SMALLK
#define ZSB_SCAT_SMALLK 1  // fan-outs <= 32 rank by a register multi-split (ballots), not shared atomics
#endif
constexpr int NWARPS = NT / 32;
#ifndef ZSB_SCAN_ITEMS
#define ZSB_SCAN_ITEMS 16
#endif
constexpr int SCAN_ITEMS = ZSB_SCAN_ITEMS;  // entries per thread in k_scan
constexpr int SCAN_TILE = NT * SCAN_ITEMS;

struct Buffers {
    const uint64_t *in_k;
    const void *in_p;
    uint64_t *tmp_k;
    void *tmp_p;
    uint64_t *out_k;
    void *out_p;
    const DestCuts *cuts;  // MODE_DEST only
    const float2 *cdf;     // MODE_ZCDF only: kf knot pairs (cdf[s], cdf[s+1]) in bucket units (staged in smem)
    unsigned long long *status;  // ZSB_ERR_NAN is raised here by a finish run holding a NaN (nullable)
    int64_t n;                   // records (bounds of every buffer above; ZSB_CHECKS)
    const PeerDest *peers;       // MODE_DEST only: write each destination's records to its (peer) buffer
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
    int32_t scale_level;  // paper mode: segments at this level take `scale` (zsort_rec's given scale); 0: none
    int32_t pad;
    double scale;
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
            p.scale = (mc.scale_level && p.level == mc.scale_level) ? mc.scale : (double)p.k / 4.0;
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
    if (ctrl[C_SAMPLE_OK]) return;  // level 1 already mapped from the sample
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
    if (p.mode == MODE_COPY || p.mode == MODE_ZLIN) return;  // ZLIN: ranged by the level-1 CDF (classify)
    finalize_params<KK>(p, acc[s].s2 / (double)p.len, acc[s].omin, acc[s].omax, mc, ctrl);
    if (ZSB_ZLIN && mc.mapping == 0 && p.mode == MODE_ZSCORE) {
        // fitted recursion: h = (x - center) * scale / std + zmin * scale as fp32 after one rounded
        // fp64 subtraction -- monotone in x (every step is a rounded monotone map), so the final
        // order is unchanged; paper mode keeps the exact Eq. 1 (one fp64 division per key)
        const float za = (float)(p.scale / p.std), zb = (float)(p.zmin * p.scale);
        if (za > 0.0f && za < 3.0e38f && fabsf(zb) < 3.0e38f) {
            p.za = za;
            p.zb = zb;
            p.mode = MODE_ZLIN;
        }
    }
    segs[s] = p;
}

// ------------------------------------------------------------------- K2

constexpr int HT = 1024;  // threads of the histogram kernel (one tile per CTA)
constexpr int CDF_KNOTS = 1024;  // coarse z-bins of the level-1 equalisation table

// Keys reach the histogram through a HIST_STAGES-deep ring of TMA bulk
// copies (HIST_CHUNK keys each, one mbarrier per stage) when the tile is
// 16-byte aligned and the launch provided the ring (stage_ok): the copy
// engine keeps ~128 KB per SM in flight, which per-thread loads do not.
constexpr int HIST_CHUNK = 4096;
#ifndef ZSB_HIST_STAGES
#define ZSB_HIST_STAGES 4
#endif
constexpr int HIST_STAGES = ZSB_HIST_STAGES;

__host__ __device__ inline size_t hist_smem(int kmax, bool ring) {
    size_t o = (size_t)((kmax + 1) & ~1) * 4 + (size_t)CDF_KNOTS * 8;
    if (ring) o = ((o + 127) & ~(size_t)127) + (size_t)HIST_STAGES * HIST_CHUNK * 8;
    return o;
}

template <int KK, int BM>
__device__ __forceinline__ void hist_body(const Buffers &B, const SegParams *__restrict__ segs, int nseg,
                                          uint32_t *__restrict__ mat, unsigned long long *status, int stage_ok,
                                          unsigned long long *scan_status, int scan_words,
                                          unsigned long long *ctrl) {
    extern __shared__ __align__(128) uint32_t hist[];
    __shared__ uint64_t full[HIST_STAGES];
    if (blockIdx.x == 0 && ctrl) {  // state of the kernels that follow (saves separate memsets)
        for (int q = threadIdx.x; q < scan_words; q += HT) scan_status[q] = 0ull;
        if (threadIdx.x == 0) {
            ctrl[C_SCAN_TICKET] = 0ull;
            ctrl[C_NCHILD] = 0ull;
            ctrl[C_REC_NEXT] = 0ull;
            ctrl[C_NENTRY] = 0ull;
            ctrl[C_NTEAM] = 0ull;
            ctrl[C_TTICK] = 0ull;
            ctrl[C_NEED_STATS] = 0ull;
        }
    }
    int s = find_seg(segs, nseg, blockIdx.x);
    const SegParams p = segs[s];
    int64_t ti = blockIdx.x - p.tile_first;
    int64_t t0 = p.start + ti * p.tile_len;
    int64_t t1 = min(t0 + p.tile_len, p.start + p.len);
    uint32_t *col = mat + p.mat_base + ti;
    if (p.mode == MODE_COPY) {  // one bucket holds the whole tile
        for (int b = threadIdx.x; b < p.k; b += HT) col[(int64_t)b * p.ntiles] = b == 0 ? (uint32_t)(t1 - t0) : 0u;
        return;
    }
    for (int b = threadIdx.x; b < p.k; b += HT) hist[b] = 0;
    float2 *cdf = (float2 *)(hist + ((p.k + 1) & ~1));
    if (p.mode == MODE_ZCDF)
        for (int q = threadIdx.x; q < p.kf; q += HT) cdf[q] = B.cdf[q];
    const uint64_t *src = src_keys(B, p.src);
    // a sampled level 1 (MODE_ZCDF) has not screened the input for NaN: K2 does
    const bool screen = KK == KEY_F64 && p.mode == MODE_ZCDF && p.level == 1;
    bool nan = false;
    auto count = [&](uint64_t b, int64_t i) {
        if (screen) nan |= __longlong_as_double((long long)b) != __longlong_as_double((long long)b);
        const int bk = seg_bucket<KK, BM>(b, p, i, B.cuts, cdf);
        ZSB_CHECK(bk >= 0 && bk < p.k);
        atomicAdd(&hist[bk], 1u);
    };

    const uint64_t *tsrc = src + t0;
    int64_t len = t1 - t0;
    if (stage_ok && ((uintptr_t)tsrc & 15) != 0 && len > 0) {  // 8-byte head before the 16-byte-aligned copies
        if (threadIdx.x == 0) count(__ldcs(tsrc), t0);
        tsrc++;
        t0++;
        len--;
    }
    if (stage_ok) {
        uint64_t *ring = (uint64_t *)((unsigned char *)hist + (((size_t)((p.k + 1) & ~1) * 4 + (size_t)CDF_KNOTS * 8 + 127) &
                                                                ~(size_t)127));
        const int nch = (int)((len + HIST_CHUNK - 1) / HIST_CHUNK);
        auto issue = [&](int c) {  // thread 0: chunk c into stage c % HIST_STAGES (whole 16-byte units)
            const int st = c % HIST_STAGES;
            const uint32_t bytes = (uint32_t)(min((int64_t)HIST_CHUNK, len - (int64_t)c * HIST_CHUNK) * 8) & ~15u;
            fence_proxy_async_smem();
            mbar_expect_tx(&full[st], bytes);
            if (bytes) bulk_g2s(ring + (size_t)st * HIST_CHUNK, tsrc + (int64_t)c * HIST_CHUNK, bytes, &full[st]);
        };
        if (threadIdx.x == 0) {
            for (int q = 0; q < HIST_STAGES; q++) mbar_init(&full[q], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int c = 0; c < min(nch, HIST_STAGES); c++) issue(c);
        for (int c = 0; c < nch; c++) {
            const int st = c % HIST_STAGES;
            mbar_wait(&full[st], (uint32_t)((c / HIST_STAGES) & 1));
            const int64_t c0 = (int64_t)c * HIST_CHUNK;
            const int clen = (int)min((int64_t)HIST_CHUNK, len - c0);
            const uint64_t *kb = ring + (size_t)st * HIST_CHUNK;
            const int cfull = clen & ~1;  // an odd last key is outside the 16-byte copy
            if (clen == HIST_CHUNK) {  // full chunk: fixed trip count, loads first, then buckets, then atomics
                constexpr int PER = HIST_CHUNK / HT;
                uint64_t kv[PER];
#pragma unroll
                for (int u = 0; u < PER; u++) kv[u] = kb[threadIdx.x + u * HT];
                #pragma unroll
                for (int u = 0; u < PER; u++) count(kv[u], t0 + c0 + threadIdx.x + u * HT);
            } else {
#pragma unroll 4
                for (int i = threadIdx.x; i < cfull; i += HT) count(kb[i], t0 + c0 + i);
            }
            if (clen & 1 && threadIdx.x == 0) count(__ldcs(tsrc + c0 + clen - 1), t0 + c0 + clen - 1);
            __syncthreads();  // stage consumed
            if (threadIdx.x == 0 && c + HIST_STAGES < nch) issue(c + HIST_STAGES);
        }
    } else {
        __syncthreads();
        int64_t i = t0 + threadIdx.x;
        constexpr int HU = ZSB_HIST_UNROLL;  // keys per thread in flight
        for (int64_t ib = t0; ib + HU * HT <= t1; ib += HU * HT, i += HU * HT) {  // CTA-uniform trip count
            uint64_t b[HU];
#pragma unroll
            for (int u = 0; u < HU; u++) b[u] = __ldcs(src + i + u * HT);
            #pragma unroll
            for (int u = 0; u < HU; u++) count(b[u], i + u * HT);
        }
        for (; i < t1; i += HT) count(__ldcs(src + i), i);
    }
    if (__syncthreads_or(nan) && threadIdx.x == 0) *status = 3;  // ZSB_ERR_NAN
    for (int b = threadIdx.x; b < p.k; b += HT) col[(int64_t)b * p.ntiles] = hist[b];
}

// L1: level-1 launch (bodies: CDF mapping, generic); else recursion levels
// (bodies: Eq. 1, its fp32 line, generic).  One kernel per group keeps each
// hot loop's code and registers to the mappings it can meet (measured on
// B200: every extra body in one kernel cost the 10^7-key scatter ~3 %).
template <int KK, int L1>
__global__ void __launch_bounds__(HT) k_hist(Buffers B, const SegParams *__restrict__ segs, int nseg,
                                             uint32_t *__restrict__ mat, unsigned long long *status, int stage_ok,
                                             unsigned long long *scan_status, int scan_words,
                                             unsigned long long *ctrl) {
    const int mode = segs[find_seg(segs, nseg, blockIdx.x)].mode;
    if (L1 && mode == MODE_ZCDF)
        hist_body<KK, 1>(B, segs, nseg, mat, status, stage_ok, scan_status, scan_words, ctrl);
    else if (!L1 && ZSB_BM_ZSCORE && mode == MODE_ZSCORE)
        hist_body<KK, 3>(B, segs, nseg, mat, status, stage_ok, scan_status, scan_words, ctrl);
    else if (!L1 && ZSB_ZLIN && mode == MODE_ZLIN)
        hist_body<KK, 4>(B, segs, nseg, mat, status, stage_ok, scan_status, scan_words, ctrl);
    else
        hist_body<KK, 0>(B, segs, nseg, mat, status, stage_ok, scan_status, scan_words, ctrl);
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
// input order inside every bucket.  The tile is processed in rounds of
// NT*ITEMS records; each round is stably sorted by bucket in shared memory:
//   count  warp w owns the slice [w*32*ITEMS, (w+1)*32*ITEMS) of the round
//          (item j of lane l = record w*32*ITEMS + j*32 + l); every item takes
//          a rank from its per-(warp, bucket) u16 counter with one shared
//          atomic (ranks follow j; lane ties inside one instruction are
//          detected by re-reading the counter and re-ranked in lane order,
//          one tie group per iteration of a ballot loop); segments of at
//          most 32 buckets rank by a register multi-split instead (ballots
//          and two shuffles, no shared atomic);
//   scan   exclusive scan of the counters in (bucket, warp) order;
//   place  records go to shared memory at (warp, bucket) base + rank;
//   write  thread i stores staged record i to cursor[b] + (i - run_start[b]):
//          consecutive threads write consecutive addresses of each bucket run
//          (coalesced), then the bucket cursors advance by the run lengths.
// Every record keeps its input order within its bucket, the front-to-back
// semantics of scatter_pass (_kernels.py:124-133), with no cross-warp
// serialization.

#ifndef ZSB_SCAT_ITEMS
#define ZSB_SCAT_ITEMS 16
#endif
constexpr int SCAT_ITEMS = ZSB_SCAT_ITEMS;
constexpr int KSCAT_MAX = 2048;  // fan-out limit of one pass
#ifndef ZSB_SCAT_AHEAD
#define ZSB_SCAT_AHEAD 0  // 1: each item's bucket computed one item ahead of its ranking (measured neutral)
#endif
// SW warps per CTA: 8 (4096-record rounds, two CTAs per SM) for k <= 1024,
// 16 (8192-record rounds, one CTA per SM) above, so that a bucket's run in a
// round stays >= 4 records = one 32-byte sector of keys (shorter runs leave
// partially written sectors that cost a DRAM read-modify-write).
inline int scat_warps(int k, int threshold = 1024) { return k <= threshold ? 8 : 16; }


struct ScatLayout {
    size_t off_cur, off_cnt, off_lst, off_k, off_p, off_b, off_cdf, total;
};

__host__ __device__ inline ScatLayout scat_layout(int k, int pb, int sw, int nset = 2) {
    const int round = sw * 32 * SCAT_ITEMS;
    ScatLayout L;
    size_t o = 0;
    L.off_cur = o;
    o += (size_t)k * 4;
    o = (o + 15) & ~(size_t)15;
    L.off_cnt = o;  // nset counter sets (with two, consecutive rounds alternate)
    o += (size_t)nset * k * sw * 2;
    o = (o + 15) & ~(size_t)15;
    L.off_lst = o;  // two run-start tables
    o += (size_t)2 * (k + 2) * 2;
    o = (o + 15) & ~(size_t)15;
    L.off_k = o;
    o += (size_t)round * 8;
    L.off_p = o;
    o += (size_t)round * pb;
    o = (o + 15) & ~(size_t)15;
    L.off_b = o;
    o += (size_t)round * 2;
    o = (o + 15) & ~(size_t)15;
    L.off_cdf = o;  // the CDF table (level-1 equalisation only) follows the layout
    L.total = o;
    return L;
}

// Exclusive scan in (digit, warp) order of per-(warp, digit) u16 counters laid
// out [warp][ndig] (a warp's leaders then touch distinct banks).  Thread t
// owns digits [t*per, (t+1)*per): per digit it walks the SW warps in order,
// then one block scan of the thread totals and a write-back pass.  Writes the
// digit starts to dstart[0..ndig].  Ends with a barrier.  (Folding the
// cursor update in here and storing each staged record's destination instead
// of its bucket measured 5 % slower on B200: placement is the critical phase.)
template <int SW>
__device__ __forceinline__ void scan_wd(uint16_t *cnt, int ndig, uint16_t *dstart, uint32_t *wsum) {
    constexpr int T = SW * 32;
    const int tid = threadIdx.x, w = tid >> 5, lane = lane_id();
    const int per = (ndig + T - 1) / T;
    const int d0 = min(ndig, tid * per), d1 = min(ndig, d0 + per);
    if ((per == 2 || per == 4) && ndig == per * T) {
        // packed path (k = 2T or 4T, the level-1 fan-outs): a thread's digit
        // pairs are u32 words of every warp's row; both digits of a pair
        // advance together in one packed add (counts and positions stay below
        // 2^16), and the rows are re-read in the write-back rather than held
        // in registers (the round's keys and ranks are live here)
        const int np = per >> 1;
        uint32_t *c32 = (uint32_t *)cnt;
        uint32_t ps0 = 0, ps1 = 0;
#pragma unroll
        for (int ww = 0; ww < SW; ww++) ps0 += c32[(ww * ndig + d0) >> 1];
        if (np == 2)
#pragma unroll
            for (int ww = 0; ww < SW; ww++) ps1 += c32[((ww * ndig + d0) >> 1) + 1];
        const uint32_t tsum = (ps0 & 0xFFFFu) + (ps0 >> 16) + (ps1 & 0xFFFFu) + (ps1 >> 16);
        uint32_t x = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        uint32_t run = x - tsum + warps_before(wsum, w, lane);
        for (int q = 0; q < np; q++) {
            const uint32_t ps = q ? ps1 : ps0;
            const uint32_t lo = run, hi = run + (ps & 0xFFFFu);
            uint32_t r = lo | (hi << 16);
            *(uint32_t *)(dstart + d0 + 2 * q) = r;
#pragma unroll
            for (int ww = 0; ww < SW; ww++) {
                uint32_t *a = c32 + ((ww * ndig + d0) >> 1) + q;
                const uint32_t c = *a;
                *a = r;
                r += c;
            }
            run = hi + (ps >> 16);
        }
        if (tid == T - 1) dstart[ndig] = (uint16_t)run;
        __syncthreads();
        return;
    }
    uint32_t tsum = 0;
    for (int d = d0; d < d1; d++)
#pragma unroll
        for (int ww = 0; ww < SW; ww++) tsum += cnt[ww * ndig + d];
    uint32_t x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    uint32_t run = x - tsum + warps_before(wsum, w, lane);
    for (int d = d0; d < d1; d++) {
        dstart[d] = (uint16_t)run;
#pragma unroll
        for (int ww = 0; ww < SW; ww++) {
            const uint32_t c = cnt[ww * ndig + d];
            cnt[ww * ndig + d] = (uint16_t)run;
            run += c;
        }
    }
    if (tid == T - 1) dstart[ndig] = (uint16_t)run;
    __syncthreads();
}

template <int KK, int PB, int SW, int BM, int NSET>
__device__ __forceinline__ void scatter_body(const Buffers &B, const SegParams *__restrict__ segs, int nseg,
                                             const uint32_t *__restrict__ mat, int dst_sel, long long *prof) {
#ifdef ZSB_PHASE_PROFILE  // per-phase clock64 accounting (build with ZSB_PHASE_PROFILE=1)
    long long t_mark = prof ? clock64() : 0;
    long long acc_ph[6] = {0, 0, 0, 0, 0, 0};
#define SCAT_MARK(slot)                                  \
    do {                                                 \
        if (prof) {                                      \
            long long t_ = clock64();                    \
            acc_ph[slot] += t_ - t_mark;                 \
            t_mark = t_;                                 \
        }                                                \
    } while (0)
#else
#define SCAT_MARK(slot) \
    do {                \
    } while (0)
#endif
    using P = typename PayloadT<PB>::T;
    constexpr int ITEMS = SCAT_ITEMS;
    constexpr int ST = SW * 32;             // threads
    constexpr int ROUND = ST * ITEMS;       // records per round
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t wtot[SW];
    int s = find_seg(segs, nseg, blockIdx.x);
    const SegParams p = segs[s];
    const int64_t ti = blockIdx.x - p.tile_first;
    const int64_t t0 = p.start + ti * p.tile_len;
    const int64_t t1 = min(t0 + p.tile_len, p.start + p.len);
    const uint64_t *sk = src_keys(B, p.src);
    const P *sp = src_pay<PB>(B, p.src);
    if (p.mode == MODE_COPY) {  // all-equal segment: land it in the output directly
        if (p.src == 2) return;
        P *op = (P *)B.out_p;
        for (int64_t i = t0 + threadIdx.x; i < t1; i += ST) {
            B.out_k[i] = sk[i];
            if constexpr (PB != 0) op[i] = sp[i];
        }
        return;
    }
    const int k = p.k;
    const ScatLayout L = scat_layout(k, PB, SW, NSET);
    const int NC = k * SW;
    uint32_t *cur = (uint32_t *)(smem + L.off_cur);
    uint16_t *cnt2 = (uint16_t *)(smem + L.off_cnt);  // [NSET][SW][k]
    uint16_t *lst2 = (uint16_t *)(smem + L.off_lst);  // [2][k + 2]
    uint64_t *stk = (uint64_t *)(smem + L.off_k);
    P *stp = (P *)(smem + L.off_p);
    uint16_t *stb = (uint16_t *)(smem + L.off_b);
    float2 *cdf = (float2 *)(smem + L.off_cdf);
    if (p.mode == MODE_ZCDF)
        for (int q = threadIdx.x; q < p.kf; q += ST) cdf[q] = B.cdf[q];
    uint64_t *dk = dst_sel == 1 ? B.tmp_k : B.out_k;
    P *dp = (P *)(dst_sel == 1 ? B.tmp_p : B.out_p);
    const uint32_t *col = mat + p.mat_base + ti;
    const uint32_t adj = (uint32_t)(p.start - p.scan_base);
    for (int b = threadIdx.x; b < k; b += ST) cur[b] = col[(int64_t)b * p.ntiles] + adj;
    for (int q = threadIdx.x; q < NSET * NC; q += ST) cnt2[q] = 0;
    __syncthreads();

    const int w = threadIdx.x >> 5, lane = lane_id();
    const unsigned lt = lanemask_lt();
    const uint64_t l2pol = l2_evict_last_policy();
    // Pipeline across rounds.  Round r's staged records are written to HBM
    // while round r+1 computes its buckets and counts (phase A), so the store
    // traffic overlaps the arithmetic; counters and run-start tables
    // alternate between two sets so no barrier separates the two.  Keys of
    // round r+1 are loaded during round r's placement; payloads at the start
    // of their round, consumed at placement.
    const int base = w * 32 * ITEMS + lane;
    uint64_t key[ITEMS];
    {
        const int nv0 = (int)min((int64_t)ROUND, t1 - t0);
#pragma unroll
        for (int j = 0; j < ITEMS; j++) key[j] = base + j * 32 < nv0 ? __ldcs(sk + t0 + base + j * 32) : 0ull;
    }
    int rb = 0, prev_nvalid = 0;  // counter/run-start set of this round; records staged by the previous round
    // FULL: this round and the previous one hold ROUND records (all rounds
    // but the first and the last): no per-item bounds checks
    auto round_t = [&](auto full_t, int64_t r0, int nvalid) {
        constexpr bool FULL = decltype(full_t)::value;
        uint16_t *cnt = cnt2 + (NSET == 2 ? rb * NC : 0);
        if constexpr (NSET == 1) {  // one counter set: cleared behind the previous round's placement
            if (r0 != t0) {
                for (int q = threadIdx.x; q < NC / 2; q += ST) ((uint32_t *)cnt)[q] = 0u;
                __syncthreads();
            }
        }
        uint16_t *lst = lst2 + rb * (k + 2);
        const uint16_t *lstp = lst2 + (rb ^ 1) * (k + 2);
        P pay[PB != 0 ? ITEMS : 1];
        if constexpr (PB != 0) {
#pragma unroll
            for (int j = 0; j < ITEMS; j++)
                pay[j] = (FULL || base + j * 32 < nvalid) ? __ldcs(sp + r0 + base + j * 32) : (P)0;
        }
        // phase A: bucket + rank of item j (one shared atomic on its
        // per-(warp, bucket) u16 counter: the returned count is its rank among
        // its warp's items of that bucket; items run in program order behind
        // a __syncwarp, so ranks follow j).  The lanes of one instruction that
        // share a bucket -- a tie group -- may get their counts in any order:
        // the converged warp re-reads its counters after the atomic, a group
        // of g lanes finds the group start + g there, and every such group is
        // re-ranked in lane order, one group per iteration of a ballot loop --
        // the checked path, always on, paid only by instructions holding a tie
        // group.  Interleaved with the coalesced write of staged slot
        // tid + j*ST of the previous round.
        // (Measured on B200 and not used at 1024 buckets: a ballot-per-bucket-
        // bit multi-split with no re-read, 27 % slower -- it is the path of
        // fan-outs <= 32, five ballots; one MATCH.ANY per tie row instead of
        // the loop, C4 +2 %; a second __syncwarp between the atomic and the
        // re-read, 8 % slower; one atomic per run of equal adjacent buckets
        // for ordered inputs, no gain.)
        uint32_t pk[ITEMS];  // bucket | rank << 16
        // (Measured and not used: computing every item's bucket and the
        // previous round's writes in a barrier-free loop before the ranking
        // loop -- C4 scatter +11 %: the stores interleaved with the ranking
        // chain are what hides their issue.)
        auto bucket_of_item = [&](int j) -> int {
            return (FULL || base + j * 32 < nvalid) ? seg_bucket<KK, BM>(key[j], p, r0 + base + j * 32, B.cuts, cdf)
                                                    : -1;
        };
        // the coalesced write of staged slot tid + j*ST of the previous round
        auto write_prev = [&](int j) {
            const int i = threadIdx.x + j * ST;
            if (FULL || i < prev_nvalid) {
                const int b = stb[i];
                const uint32_t dst = cur[b] + (uint32_t)(i - lstp[b]);
                ZSB_CHECK(b < k && (int64_t)dst >= p.start && (int64_t)dst < p.start + p.len);
                if constexpr (BM == 5) {  // straight into destination b's (peer) receive buffer
                    const int64_t at = (int64_t)dst + B.peers->delta[b];
                    ((uint64_t *)B.peers->k[b])[at] = stk[i];
                    if constexpr (PB != 0) ((P *)B.peers->p[b])[at] = stp[i];
                } else if (!ZSB_EXP_NOSTORE || dst == 0xffffffffu) {
                    // evict_last: the runs (and the finish's input) stay in L2
                    st_keep(dk + dst, stk[i], l2pol);
                    if constexpr (PB != 0) st_keep(dp + dst, stp[i], l2pol);
                }
            }
        };
        if (BM != 1 && SW == 8 && ZSB_SCAT_SMALLK && k <= 32) {  // (8-warp kernels: kmax <= 512)
            // Small fan-out (recursion children, destination ranks): every
            // instruction holds many lanes per bucket, so the ranking is a warp
            // multi-split in registers -- one ballot per bucket bit gives lane b
            // the lanes of bucket b (`mine`); a lane takes its group's mask and
            // running count from lane `bucket` by two shuffles.  No shared
            // atomics, no re-read, no match; items are independent but for one
            // register add.  Ordered by construction (lane order inside an
            // instruction, program order across instructions).
            uint32_t wc = 0;  // lane b: the warp's records of bucket b so far in this round
#pragma unroll
            for (int j = 0; j < ITEMS; j++) {
                const int bkj = bucket_of_item(j);
                const bool v = FULL || bkj >= 0;
                unsigned mine = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, v);
#pragma unroll
                for (int q = 0; q < 5; q++) {
                    const unsigned bal = __ballot_sync(0xffffffffu, (bkj >> q) & 1);
                    mine &= ((lane >> q) & 1) ? bal : ~bal;
                }
                const int srcl = v ? bkj : lane;
                const unsigned gm = __shfl_sync(0xffffffffu, mine, srcl);
                const uint32_t basec = __shfl_sync(0xffffffffu, wc, srcl);
                const uint32_t old = basec + (uint32_t)__popc(gm & lt);
                wc += (uint32_t)__popc(mine);
                pk[j] = v ? (uint32_t)bkj | (old << 16) : 0xffffffffu;
                write_prev(j);
            }
            if (lane < k) cnt[w * k + lane] = (uint16_t)wc;
        } else {
            // the next item's bucket (its mapping-table load) is computed ahead,
            // before this item's warp barrier, so it overlaps the ranking chain
            int bk_next = ZSB_SCAT_AHEAD ? bucket_of_item(0) : 0;
#pragma unroll
            for (int j = 0; j < ITEMS; j++) {
                int bkj;
                if constexpr (ZSB_SCAT_AHEAD) {
                    bkj = bk_next;
                    if (j + 1 < ITEMS) bk_next = bucket_of_item(j + 1);
                } else {
                    bkj = bucket_of_item(j);
                }
                const bool v = FULL || bkj >= 0;
                uint32_t old = 0, after = 0;
                const int q = w * k + (v ? bkj : 0);
                const uint32_t sh = 16 * (q & 1);
                uint32_t *word = (uint32_t *)cnt + (q >> 1);
                __syncwarp();  // item j - 1's re-reads before item j's atomics
                if (v) {
                    old = (atomicAdd(word, 1u << sh) >> sh) & 0xFFFFu;
                    after = (*(volatile uint32_t *)word >> sh) & 0xFFFFu;
                }
                {
                    // tie groups one at a time (a MATCH.ANY occupies the SM for
                    // ~64 cycles; a group costs two ballots and a shuffle): all
                    // lanes of a group but its last-served one see the tie; the
                    // lowest of them names the bucket, the group re-ranks itself
                    // in lane order from the group's end count
                    unsigned tm = __ballot_sync(0xffffffffu, v && after != old + 1u);
                    while (tm) {
                        const int bl = __shfl_sync(0xffffffffu, bkj, __ffs(tm) - 1);
                        const unsigned grp = __ballot_sync(0xffffffffu, bkj == bl);
                        if (bkj == bl) old = after - (uint32_t)__popc(grp) + (uint32_t)__popc(grp & lt);
                        tm &= ~grp;
                    }
                }
                pk[j] = v ? (uint32_t)bkj | (old << 16) : 0xffffffffu;
                write_prev(j);
            }
        }
        __syncthreads();
        SCAT_MARK(1);  // buckets + counting + previous round's writes
        // phase B: cursors advance past the previous round's runs; scan
        if (FULL || prev_nvalid)
            for (int b = threadIdx.x; b < k; b += ST) cur[b] += (uint32_t)(lstp[b + 1] - lstp[b]);
        scan_wd<SW>(cnt, k, lst, wtot);
        SCAT_MARK(2);  // scan
        // phase C: place (slot = (warp, bucket) base + rank); clear the other
        // counter set for the next round; load the next round's keys
#pragma unroll
        for (int j = 0; j < ITEMS; j++) {
            if (FULL || pk[j] != 0xffffffffu) {
                const int b = (int)(pk[j] & 0xFFFFu);
                const uint32_t pos = (uint32_t)cnt[w * k + b] + (pk[j] >> 16);
                ZSB_CHECK(b < k && pos < (uint32_t)ROUND);
                stk[pos] = key[j];
                if constexpr (PB != 0) stp[pos] = pay[j];
                stb[pos] = (uint16_t)b;
            }
        }
        {
            if constexpr (NSET == 2) {
                uint16_t *cn = cnt2 + (rb ^ 1) * NC;
                for (int q = threadIdx.x; q < NC / 2; q += ST) ((uint32_t *)cn)[q] = 0u;
            }
            const int64_t rn = r0 + ROUND;
            const int nvn = rn < t1 ? (int)min((int64_t)ROUND, t1 - rn) : 0;
#pragma unroll
            for (int j = 0; j < ITEMS; j++) key[j] = base + j * 32 < nvn ? __ldcs(sk + rn + base + j * 32) : 0ull;
        }
        __syncthreads();
        SCAT_MARK(3);  // placement
    };
    for (int64_t r0 = t0; r0 < t1; r0 += ROUND) {
        SCAT_MARK(5);
        const int nvalid = (int)min((int64_t)ROUND, t1 - r0);
        if (nvalid == ROUND && prev_nvalid == ROUND) round_t(std::true_type{}, r0, nvalid);
        else round_t(std::false_type{}, r0, nvalid);
        prev_nvalid = nvalid;
        rb ^= 1;
    }
    {  // epilogue: write the last round
        const uint16_t *lstp = lst2 + (rb ^ 1) * (k + 2);
        for (int i = threadIdx.x; i < prev_nvalid; i += ST) {
            const int b = stb[i];
            const uint32_t dst = cur[b] + (uint32_t)(i - lstp[b]);
            ZSB_CHECK(b < k && (int64_t)dst >= p.start && (int64_t)dst < p.start + p.len);
            if constexpr (BM == 5) {
                const int64_t at = (int64_t)dst + B.peers->delta[b];
                ((uint64_t *)B.peers->k[b])[at] = stk[i];
                if constexpr (PB != 0) ((P *)B.peers->p[b])[at] = stp[i];
            } else {
                st_keep(dk + dst, stk[i], l2pol);
                if constexpr (PB != 0) st_keep(dp + dst, stp[i], l2pol);
            }
        }
    }
    SCAT_MARK(4);
#ifdef ZSB_PHASE_PROFILE
    if (prof && threadIdx.x == 0)
        for (int q = 0; q < 6; q++) prof[(int64_t)blockIdx.x * 8 + q] = acc_ph[q];
#endif
#undef SCAT_MARK
}

template <int KK, int PB, int SW, int NSET, int L1>
__global__ void __launch_bounds__(SW * 32, 16 / SW) k_scatter(Buffers B, const SegParams *__restrict__ segs,
                                                              int nseg, const uint32_t *__restrict__ mat,
                                                              int dst_sel, long long *prof) {
    const int mode = segs[find_seg(segs, nseg, blockIdx.x)].mode;
    if (L1 && mode == MODE_ZCDF)
        scatter_body<KK, PB, SW, 1, NSET>(B, segs, nseg, mat, dst_sel, prof);
    else if (!L1 && ZSB_BM_ZSCORE && mode == MODE_ZSCORE)
        scatter_body<KK, PB, SW, 3, NSET>(B, segs, nseg, mat, dst_sel, prof);
    else if (!L1 && ZSB_ZLIN && mode == MODE_ZLIN)
        scatter_body<KK, PB, SW, 4, NSET>(B, segs, nseg, mat, dst_sel, prof);
    else if (!L1 && mode == MODE_DEST && B.peers)
        scatter_body<KK, PB, SW, 5, NSET>(B, segs, nseg, mat, dst_sel, prof);
    else
        scatter_body<KK, PB, SW, 0, NSET>(B, segs, nseg, mat, dst_sel, prof);
}

// ------------------------------------------------------- equalisation
// Level 1, fitted mapping: a histogram of CDF_KNOTS coarse z-score bins (Eq. 1
// with that many bins) and the piecewise-linear empirical CDF through it, in
// bucket units; bucket_cdf maps a key through it, so buckets hold ~n/k
// records whatever the shape of the distribution at the knot resolution.
// The kernels act only if K1 left the segment in z-score mode.

constexpr int KF_MAX = CDF_KNOTS;

template <int KK>
__global__ void __launch_bounds__(512) k_fine_hist(const uint64_t *__restrict__ keys, int64_t n,
                                                   const SegParams *__restrict__ seg, int kf,
                                                   unsigned int *__restrict__ counts) {
    extern __shared__ uint32_t fh[];
    const SegParams p = *seg;
    float za, zb;
    if (p.mode != MODE_ZSCORE || !zc_coeffs(p, kf, za, zb)) return;
    const double c = p.center;
    for (int b = threadIdx.x; b < kf; b += 512) fh[b] = 0;
    __syncthreads();
    int64_t i = (int64_t)blockIdx.x * 512 + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * 512;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint64_t b[4];
#pragma unroll
        for (int u = 0; u < 4; u++) b[u] = __ldcs(keys + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; u++) atomicAdd(&fh[zc_bin(zc_coord(key_value<KK>(b[u]), c, za, zb), kf)], 1u);
    }
    for (; i < n; i += stride) atomicAdd(&fh[zc_bin(zc_coord(key_value<KK>(__ldcs(keys + i)), c, za, zb), kf)], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < kf; b += 512)
        if (fh[b]) atomicAdd(&counts[b], fh[b]);
}

// Knot pairs (cdf[s], cdf[s+1]) of the piecewise-linear CDF in bucket units
// (fp32: rounding is monotone, so the knots stay non-decreasing) from the
// coarse-bin counts (summing to `total`), and the switch of the level-1
// segment to MODE_ZCDF.  One CTA of NTHR threads; NTHR divides kf.
template <int NTHR>
__device__ void build_cdf_block(const unsigned int *counts, int kf, int64_t total, SegParams *seg, SegParams p,
                                float za, float zb, float2 *cdf) {
    constexpr int PER_MAX = KF_MAX / NTHR;
    __shared__ unsigned long long wsum[NTHR / 32];
    __shared__ float knot[KF_MAX + 1];
    const int per = kf / NTHR;
    const int f0 = threadIdx.x * per;
    unsigned int cv[PER_MAX];
    unsigned long long tsum = 0;
#pragma unroll
    for (int q = 0; q < PER_MAX; q++) cv[q] = q < per ? __ldcg(&counts[f0 + q]) : 0u;
#pragma unroll
    for (int q = 0; q < PER_MAX; q++) tsum += cv[q];
    unsigned long long x = tsum;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    unsigned long long run = x - tsum;
    for (int q = 0; q < w; q++) run += wsum[q];
    const double inv = (double)p.k / (double)total;  // knots in bucket units
#pragma unroll
    for (int q = 0; q < PER_MAX; q++) {
        if (q < per) {
            knot[f0 + q] = (float)((double)run * inv);
            run += cv[q];
        }
    }
    if (threadIdx.x == NTHR - 1) knot[kf] = (float)p.k;
    __syncthreads();
    for (int s = threadIdx.x; s < kf; s += NTHR) cdf[s] = make_float2(knot[s], knot[s + 1]);
    if (threadIdx.x == 0) {
        p.scale = p.scale * ((double)kf / (double)p.k);
        p.kf = kf;
        p.za = za;
        p.zb = zb;
        p.mode = MODE_ZCDF;
        *seg = p;
    }
}

__global__ void __launch_bounds__(1024) k_build_cdf(const unsigned int *__restrict__ counts, int kf, int64_t n,
                                                    SegParams *seg, float2 *cdf) {
    SegParams p = *seg;
    float za, zb;
    if (p.mode != MODE_ZSCORE || !zc_coeffs(p, kf, za, zb)) return;
    build_cdf_block<1024>(counts, kf, n, seg, p, za, zb, cdf);
}

// ---------------------------------------------------- sampled level 1
// Fitted mapping: the coarse z-coordinate and its CDF only need to be
// monotone, not exact, so level 1 takes them from a stratified sample --
// SAMP_CHUNKS_MAX evenly spaced runs of SAMP_CHUNK consecutive keys (every key
// when n <= ~256K) -- instead of two full passes over the input.  The first
// full pass is then K2's histogram, which also raises the NaN status.  A
// degenerate sample (NaN, all equal, no finite spread) leaves the segment in
// z-score mode with C_SAMPLE_OK = 0 and the exact K1 path runs instead.

constexpr int SAMP_CHUNK = 32;
constexpr int SAMP_CHUNKS_MAX = 8192;
constexpr int SAMP_UNROLL = 8;  // sample keys per thread, loads issued together (grid = sample / (NT * 8))

struct SampPartial {
    unsigned long long omin, omax, nan, pad;
    double s1, s2, cnt, pad2;
};

// position of sample item g (chunk g / SAMP_CHUNK, offset g % SAMP_CHUNK), -1 past a short chunk
__device__ __forceinline__ int64_t sample_pos(int64_t g, int64_t nitems, int64_t stride, int64_t clen) {
    const int64_t off = g & (SAMP_CHUNK - 1);
    return (g < nitems && off < clen) ? (g / SAMP_CHUNK) * stride + off : -1;
}

// ------------------------------------------------ fused level-1 mapping
// One cooperative launch (one CTA per SM, grid barriers between phases)
// replaces the level-1 chain init -> sample moments -> sample CDF -> exact
// K1 -> exact fine histogram -> CDF, which cost a launch gap each:
//   S1  stratified sample moments; every CTA reduces the
//       partials itself, in the same order, so all derive identical params;
//   S2  sample coarse-bin histogram -> CDF knots (CTA 0), mode MODE_ZCDF;
// and, only when the sample is degenerate (NaN, all equal, no spread):
//   E1  exact K1 over all keys (two-limb integer sum for int64 keys, shifted
//       fp64 sums, exact ordered min/max, NaN count) -> finalize_params;
//   E2  exact coarse-bin histogram -> CDF knots if E1 chose z-score mode.
constexpr int LT = 512;  // threads of the fused level-1 kernel

template <int KK>
__global__ void __launch_bounds__(LT) k_level1_map(const uint64_t *__restrict__ keys, int64_t n, SegParams *seg,
                                                   int64_t *kfirst, int64_t *wfirst, int64_t nwin, int64_t k,
                                                   int64_t tile_len, int64_t ntiles, int64_t nchunks, int64_t stride,
                                                   SampPartial *sparts, MomPartial *mparts, unsigned int *fine,
                                                   float2 *cdf, unsigned long long *ctrl, MapCfg mc, int kf) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t fh[KF_MAX];
    __shared__ SampPartial wps[LT / 32];
    __shared__ MomPartial wpm[LT / 32];
    const int tid = threadIdx.x, w = tid >> 5, lane = lane_id();
    SegParams p{};
    p.len = n;
    p.tile_len = tile_len;
    p.k = (int32_t)k;
    p.ntiles = (int32_t)ntiles;
    p.mode = MODE_ZSCORE;
    p.level = 1;
    p.center = 0.0;
    p.std = 1.0;
    p.scale = 1.0;
    if (blockIdx.x == 0 && tid == 0) {
        kfirst[0] = 0;
        kfirst[1] = k + 1;
        wfirst[0] = 0;
        wfirst[1] = nwin;
    }
    if (blockIdx.x == 0) {
        for (int b = tid; b < kf; b += LT) fine[b] = 0u;
        if (tid < C_SLOTS) ctrl[tid] = 0ull;  // fresh control block (nothing reads it before the first barrier)
    }
    const double c0 = key_value<KK>(keys[0]);
    const int64_t G = (int64_t)gridDim.x * LT, g0 = (int64_t)blockIdx.x * LT + tid;

    // ---- S1: sample moments
    {
        const int64_t clen = stride < SAMP_CHUNK ? stride : SAMP_CHUNK;
        const int64_t nitems = nchunks * SAMP_CHUNK;
        SampPartial a{~0ull, 0, 0, 0, 0.0, 0.0, 0.0, 0.0};
        uint64_t kb0[SAMP_UNROLL];  // the first batch stays in registers for S2
        bool kv0[SAMP_UNROLL];
        for (int64_t gb = g0; gb < nitems; gb += SAMP_UNROLL * G) {
            uint64_t b[SAMP_UNROLL];
            bool v[SAMP_UNROLL];
#pragma unroll
            for (int u = 0; u < SAMP_UNROLL; u++) {
                const int64_t i = sample_pos(gb + u * G, nitems, stride, clen);
                v[u] = i >= 0;
                b[u] = v[u] ? __ldcs(keys + i) : 0ull;
                if (gb == g0) {
                    kb0[u] = b[u];
                    kv0[u] = v[u];
                }
            }
#pragma unroll
            for (int u = 0; u < SAMP_UNROLL; u++) {
                if (!v[u]) continue;
                const double x = key_value<KK>(b[u]);
                if (KK == KEY_F64 && x != x) {
                    a.nan++;
                    continue;
                }
                const uint64_t o = ord_key<KK>(b[u]);
                a.omin = o < a.omin ? o : a.omin;
                a.omax = o > a.omax ? o : a.omax;
                const double d = x - c0;
                a.s1 += d;
                a.s2 += d * d;
                a.cnt += 1.0;
            }
        }
        auto reduce = [&](SampPartial q) -> SampPartial {  // block total (valid in every thread)
            q.omin = warp_min_u64(q.omin);
            q.omax = warp_max_u64(q.omax);
            q.nan = warp_sum(q.nan);
            q.s1 = warp_sum(q.s1);
            q.s2 = warp_sum(q.s2);
            q.cnt = warp_sum(q.cnt);
            __syncthreads();
            if (lane == 0) wps[w] = q;
            __syncthreads();
            SampPartial t = wps[0];
            for (int j = 1; j < LT / 32; j++) {
                t.omin = wps[j].omin < t.omin ? wps[j].omin : t.omin;
                t.omax = wps[j].omax > t.omax ? wps[j].omax : t.omax;
                t.nan += wps[j].nan;
                t.s1 += wps[j].s1;
                t.s2 += wps[j].s2;
                t.cnt += wps[j].cnt;
            }
            return t;
        };
        a = reduce(a);
        if (tid == 0) sparts[blockIdx.x] = a;
        grid.sync();
        SampPartial q{~0ull, 0, 0, 0, 0.0, 0.0, 0.0, 0.0};
        if (tid < (int)gridDim.x) q = sparts[tid];  // gridDim <= LT
        a = reduce(q);
        bool ok = !(a.nan || a.cnt < 2.0 || a.omin == a.omax);
        if (ok) {
            const double mean = c0 + a.s1 / a.cnt;
            const double dm = mean - c0;
            double m2 = a.s2 - 2.0 * dm * a.s1 + a.cnt * dm * dm;
            if (m2 < 0.0) m2 = 0.0;
            const double sd = sqrt(m2 / a.cnt);
            const double vmin = key_value<KK>(key_from_ord<KK>(a.omin)), vmax = key_value<KK>(key_from_ord<KK>(a.omax));
            const double span = (vmax - vmin) / sd;
            ok = sd > 0.0 && isfinite(sd) && span > 0.0 && isfinite(span);
            if (ok) {
                p.center = mean;
                p.std = sd;
                p.zmin = (mean - vmin) / sd;
                p.scale = ((double)p.k * (1.0 - 0x1p-20)) / span;
                ok = isfinite(p.zmin) && p.scale > 0.0 && isfinite(p.scale) && zc_coeffs(p, kf, p.za, p.zb);
            }
        }
        if (ok) {
            // ---- S2: sample coarse-bin histogram -> CDF.  (A second, ordered-
            // image coordinate -- log-like, chosen for one-signed heavy-tailed
            // samples -- balanced C4's level-1 buckets but cost the 10^7-key
            // scatter 7-14 % in code size and registers: not used.)
            for (int b = tid; b < kf; b += LT) fh[b] = 0;
            __syncthreads();
            for (int64_t gb = g0; gb < nitems; gb += SAMP_UNROLL * G) {
                uint64_t b[SAMP_UNROLL];
                bool v[SAMP_UNROLL];
#pragma unroll
                for (int u = 0; u < SAMP_UNROLL; u++) {
                    if (gb == g0) {  // still in registers from S1
                        b[u] = kb0[u];
                        v[u] = kv0[u];
                    } else {
                        const int64_t i = sample_pos(gb + u * G, nitems, stride, clen);
                        v[u] = i >= 0;
                        b[u] = v[u] ? __ldcs(keys + i) : 0ull;
                    }
                }
#pragma unroll
                for (int u = 0; u < SAMP_UNROLL; u++)
                    if (v[u]) atomicAdd(&fh[zc_bin(zc_coord(key_value<KK>(b[u]), p.center, p.za, p.zb), kf)], 1u);
            }
            __syncthreads();
            for (int b = tid; b < kf; b += LT)
                if (fh[b]) atomicAdd(&fine[b], fh[b]);
            grid.sync();
            if (blockIdx.x == 0) {
                if (tid == 0) ctrl[C_SAMPLE_OK] = 1;
                build_cdf_block<LT>(fine, kf, nchunks * clen, seg, p, p.za, p.zb, cdf);
            }
            return;
        }
    }

    // ---- E1: exact K1 (the sample was degenerate)
    MomPartial a{~0ull, 0, 0, 0, 0.0, 0.0, 0, 0};
    for (int64_t i = g0; i < n; i += G) {
        const uint64_t b = __ldcs(keys + i);
        const uint64_t o = ord_key<KK>(b);
        a.omin = o < a.omin ? o : a.omin;
        a.omax = o > a.omax ? o : a.omax;
        if constexpr (KK == KEY_I64) {
            a.shi += (long long)b >> 32;
            a.slo += b & 0xFFFFFFFFull;
        }
        const double x = key_value<KK>(b);
        if (KK == KEY_F64 && x != x) {
            a.nan++;
        } else {
            const double d = x - c0;
            a.s1 += d;
            a.s2 += d * d;
        }
    }
    auto mreduce = [&](MomPartial q) -> MomPartial {
        q.omin = warp_min_u64(q.omin);
        q.omax = warp_max_u64(q.omax);
        q.shi = warp_sum(q.shi);
        q.slo = warp_sum(q.slo);
        q.s1 = warp_sum(q.s1);
        q.s2 = warp_sum(q.s2);
        q.nan = warp_sum(q.nan);
        __syncthreads();
        if (lane == 0) wpm[w] = q;
        __syncthreads();
        MomPartial t = wpm[0];
        for (int j = 1; j < LT / 32; j++) {
            t.omin = wpm[j].omin < t.omin ? wpm[j].omin : t.omin;
            t.omax = wpm[j].omax > t.omax ? wpm[j].omax : t.omax;
            t.shi += wpm[j].shi;
            t.slo += wpm[j].slo;
            t.s1 += wpm[j].s1;
            t.s2 += wpm[j].s2;
            t.nan += wpm[j].nan;
        }
        return t;
    };
    a = mreduce(a);
    if (tid == 0) mparts[blockIdx.x] = a;
    grid.sync();
    MomPartial q{~0ull, 0, 0, 0, 0.0, 0.0, 0, 0};
    if (tid < (int)gridDim.x) q = mparts[tid];
    a = mreduce(q);
    if (a.nan) {
        if (blockIdx.x == 0 && tid == 0) {
            ctrl[C_STATUS] = 3;  // ZSB_ERR_NAN
            p.mode = MODE_COPY;
            *seg = p;
        }
        return;
    }
    const double dn = (double)n;
    const double mean = KK == KEY_I64 ? exact_mean(a.shi, a.slo, (uint32_t)n) : c0 + a.s1 / dn;
    const double dm = mean - c0;
    double m2 = a.s2 - 2.0 * dm * a.s1 + dn * dm * dm;
    if (m2 < 0.0) m2 = 0.0;
    p.center = mean;
    finalize_params<KK>(p, m2 / dn, a.omin, a.omax, mc, (blockIdx.x == 0 && tid == 0) ? ctrl : nullptr);
    float za = 0.f, zb = 0.f;
    if (p.mode != MODE_ZSCORE || mc.mapping != 0 || !zc_coeffs(p, kf, za, zb)) {
        if (blockIdx.x == 0 && tid == 0) *seg = p;
        return;
    }
    // ---- E2: exact coarse-bin histogram -> CDF
    for (int b = tid; b < kf; b += LT) fh[b] = 0;
    __syncthreads();
    for (int64_t i = g0; i < n; i += G)
        atomicAdd(&fh[zc_bin(zc_coord(key_value<KK>(__ldcs(keys + i)), p.center, za, zb), kf)], 1u);
    __syncthreads();
    for (int b = tid; b < kf; b += LT)
        if (fh[b]) atomicAdd(&fine[b], fh[b]);
    grid.sync();
    if (blockIdx.x == 0) build_cdf_block<LT>(fine, kf, n, seg, p, za, zb, cdf);
}

// ------------------------------------------------------------ classify
// Bucket totals of a partition level -> finish runs and next-level segments.
// k_bstart: one thread per (segment, bucket slot): absolute bucket starts into
//   bstart[kfirst[s] + b] (k_s + 1 slots per segment, last = segment end);
//   buckets above capacity become next-level segments centred on the
//   bucket's estimated mean (_kernels.py:103-106, 282-318).
// runs, level 1 (one segment): one thread per window of `half` records: the
//   buckets whose start lies in the window form one finish run (<= cap
//   records), found by binary search over bstart;
// runs, recursion levels: greedy_runs, one warp per segment.

struct ClassCfg {
    int32_t cap;   // finish capacity (records)
    int32_t half;  // level-1 window (recursion segments carry their own in SegParams::win)
    int32_t depth_guard;
    int32_t mapping;
    int32_t child_fill;  // recursion children: k = pow2 >= child_fill * len / kcap (buckets ~ kcap / child_fill)
    int32_t greedy;      // recursion levels pack finish runs greedily (else fixed windows)
    int32_t team_cap;    // buckets of cap < len <= team_cap are team runs (K5t); 0: none
    int32_t child_from_cdf;  // children of the equalised level 1 take their range from its CDF (no moments pass)
};

__device__ __forceinline__ int seg_of_slot(const int64_t *first, int nseg, int64_t g) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (first[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// A value whose equalised bucket is b (approximately its middle): the knot
// pair bracketing b + 0.5, linear inside the coarse bin, back through the
// coarse coordinate.
// The key value at equalised bucket coordinate t (t = b: the lower edge of
// bucket b): the knot pair bracketing t, linear inside the coarse bin, back
// through the coarse coordinate (the inverse of bucket_cdf up to rounding).
__device__ inline double zcdf_at(const SegParams &p, const float2 *cdf, float t) {
    int lo = 0, hi = p.kf - 1;  // first bin whose upper knot exceeds t
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cdf[mid].y <= t) lo = mid + 1;
        else hi = mid;
    }
    const float2 az = cdf[lo];
    float fr = az.y > az.x ? (t - az.x) / (az.y - az.x) : 0.0f;
    fr = fminf(fmaxf(fr, 0.0f), 1.0f);
    return p.center + ((double)lo + (double)fr - (double)p.zb) / (double)p.za;
}

__device__ inline double zcdf_inverse(const SegParams &p, const float2 *cdf, int b) {
    const float t = (float)b + 0.5f;
    int lo = 0, hi = p.kf - 1;  // first bin whose upper knot exceeds t
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cdf[mid].y <= t) lo = mid + 1;
        else hi = mid;
    }
    const float2 az = cdf[lo];
    float fr = az.y > az.x ? (t - az.x) / (az.y - az.x) : 0.5f;
    fr = fminf(fmaxf(fr, 0.0f), 1.0f);
    return p.center + ((double)lo + (double)fr - (double)p.zb) / (double)p.za;
}

__device__ __forceinline__ void bstart_slot(int64_t g, const SegParams *__restrict__ segs, int nseg,
                                            const int64_t *__restrict__ kfirst, const uint32_t *__restrict__ mat,
                                            int64_t *__restrict__ bstart, SegParams *children, SegAcc *acc,
                                            unsigned long long *ctrl, const ClassCfg &cc, const Buffers &B,
                                            int key_kind, Entry *teams) {
    const int s = seg_of_slot(kfirst, nseg, g);
    const SegParams &p = segs[s];
    const int b = (int)(g - kfirst[s]);
    const int64_t st = (b >= p.k) ? p.start + p.len
                                   : p.start + (int64_t)mat[p.mat_base + (int64_t)b * p.ntiles] - p.scan_base;
    bstart[g] = st;
    if (b >= p.k || p.mode == MODE_COPY) return;
    if (b == 0) {
        atomicAdd(&ctrl[C_ST_SCATTERS], 1ull);
        atomicMax(&ctrl[C_ST_MAXDEPTH], (unsigned long long)p.level);
    }
    const int64_t en = (b + 1 >= p.k) ? p.start + p.len
                                      : p.start + (int64_t)mat[p.mat_base + (int64_t)(b + 1) * p.ntiles] - p.scan_base;
    const int64_t c = en - st;
    if (c <= cc.cap) return;
    if (c <= cc.team_cap) {  // finished by a team (K5t) at this level
        teams[atomicAdd(&ctrl[C_NTEAM], 1ull)] = Entry{st, (int32_t)c, (p.src == 1) ? 2 : 1};
        return;
    }
    SegParams ch{};
    ch.start = st;
    ch.len = c;
    ch.level = p.level + 1;
    ch.src = (p.src == 1) ? 2 : 1;
    ch.k = p.k;
    // a parent ranged by the level-1 CDF (p.shift < 0: approximate extremes)
    // whose bucket took every record gets the exact moments pass, not the
    // integer fallback: all its keys may be equal (then MODE_COPY) or the
    // estimate may have missed their range
    const bool approx = p.mode == MODE_ZLIN && p.shift < 0;
    bool integer = p.mode == MODE_INTEGER || (c == p.len && !approx) || ch.level > cc.depth_guard;
    double lo = 0.0, hi = 0.0;
    if (!integer && p.mode == MODE_ZCDF && cc.child_from_cdf) {
        lo = zcdf_at(p, B.cdf, (float)b);
        hi = zcdf_at(p, B.cdf, (float)(b + 1));
    }
    if (integer) {
        ch.mode = MODE_INTEGER;
        atomicAdd(&ctrl[C_ST_FALLBACKS], 1ull);
        atomicOr(&ctrl[C_NEED_STATS], 1ull);
    } else if (p.mode == MODE_ZCDF && hi > lo && isfinite(lo) && isfinite(hi) && isfinite(hi - lo)) {
        // a child of the equalised level 1 (fitted): the fitted line over the
        // bucket's key range -- the level-1 CDF's inverse at the bucket's two
        // edges -- needs no moments pass over its records (the line depends on
        // min and max only; keys past the estimated edges clamp into the end
        // buckets); scale and the fp32 coefficients follow from k (plan_block)
        ch.mode = MODE_ZLIN;
        ch.center = lo;
        ch.std = hi - lo;
        ch.zmin = 0.0;
        ch.za = 0.0f;
        ch.shift = -1;  // approximate range (see `approx`)
    } else if (p.mode == MODE_ZCDF) {
        // an equal-population bucket is not a z-interval: centre the child on
        // the inverse of the equalised map at the bucket's middle (any value
        // in or near the bucket conditions the child's moments; it needs no
        // scattered data, so classify can run beside the scatter)
        ch.mode = MODE_ZSCORE;
        ch.center = zcdf_inverse(p, B.cdf, b);
        atomicOr(&ctrl[C_NEED_STATS], 1ull);
    } else {
        ch.mode = MODE_ZSCORE;
        ch.center = __dadd_rn(__dmul_rn(__dsub_rn(__ddiv_rn((double)b + 0.5, p.scale), p.zmin), p.std), p.center);
        atomicOr(&ctrl[C_NEED_STATS], 1ull);
    }
    unsigned long long slot = atomicAdd(&ctrl[C_NCHILD], 1ull);
    atomicAdd(&ctrl[C_REC_NEXT], (unsigned long long)ch.len);
    children[slot] = ch;
    acc[slot] = SegAcc{~0ull, 0ull, 0.0, 0.0};
}

__device__ __forceinline__ int lower_bound_i64(const int64_t *a, int n, int64_t v) {
    int lo = 0, hi = n;  // first index with a[i] >= v, in [0, n]
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Finish runs of window g (its buckets whose start lies in the window): up to
// two entries, returned in e[] (count in the result); the caller appends them.
__device__ __forceinline__ int window_item(int64_t g, const SegParams *__restrict__ segs, int nseg,
                                           const int64_t *__restrict__ kfirst, const int64_t *__restrict__ wfirst,
                                           const int64_t *__restrict__ bstart, const ClassCfg &cc,
                                           const int64_t *bs_one, Entry e[2]) {
    const int s = seg_of_slot(wfirst, nseg, g);
    const SegParams &p = segs[s];
    if (p.mode == MODE_COPY) return 0;
    const int64_t w = g - wfirst[s];
    const int64_t *bs = bs_one ? bs_one : bstart + kfirst[s];  // k + 1 slots (a shared copy for one segment)
    const int64_t W = p.win > 0 ? p.win : cc.half;
    const int64_t ws = p.start + w * W, we = ws + W;
    const int b0 = lower_bound_i64(bs, p.k, ws);
    const int b1 = lower_bound_i64(bs, p.k, we);
    if (b0 >= b1) return 0;  // no bucket starts inside this window
    const int dst = (p.src == 1) ? 2 : 1;
    const int64_t last = bs[b1] - bs[b1 - 1];
    int64_t e0 = bs[b0], e1 = bs[b1];
    int ne = 0;
    if (last > cc.cap - W) {
        e1 = bs[b1 - 1];
        if (last <= cc.cap) e[ne++] = Entry{bs[b1 - 1], (int32_t)last, dst};  // a mid-size bucket is a run of its own
    }
    if (e1 > e0) e[ne++] = Entry{e0, (int32_t)(e1 - e0), dst};
    return ne;
}

// ----------------------------------------------------------------- plan
// Tiling, matrix layout, bucket-slot and window prefixes of the next level
// (single CTA; the child count is read from the control block).  k is sized
// to the child so its buckets average ~cap/4 records (the reference's fixed
// k across levels is a CPU choice, core.py:355).
// Greedy finish runs of one segment (one warp): consecutive buckets join the
// current run while it stays within `cap` records; a bucket above `cap` is a
// child (recursed) and closes the run.  Runs fill to ~cap - a/2 for a mean
// bucket of a records (fixed windows reach only cap - a).  Each ballot finds
// the next bucket that breaks the run, so a chunk of 32 buckets costs one
// step per run it closes.
__device__ __forceinline__ void greedy_runs(const SegParams &p, const int64_t *__restrict__ bs, int cap,
                                            Entry *entries, unsigned long long *nentry, int lane) {
    const int dst = (p.src == 1) ? 2 : 1;
    const int k = p.k;
    int64_t R = bs[0];  // start of the open run (a bucket boundary)
    for (int c0 = 0; c0 < k; c0 += 32) {
        const int i = c0 + lane;
        const int64_t st = i < k ? bs[i] : 0, en = i < k ? bs[i + 1] : 0;
        int from = 0;
        while (true) {
            const bool valid = lane >= from && i < k;
            const bool brk = valid && (en - st > cap || en - R > cap);
            const unsigned m = __ballot_sync(0xffffffffu, brk);
            if (!m) break;  // the rest of the chunk joins the open run
            const int f = __ffs(m) - 1;
            const int64_t sf = __shfl_sync(0xffffffffu, st, f), ef = __shfl_sync(0xffffffffu, en, f);
            const bool child = ef - sf > cap;
            if (lane == 0 && sf > R) entries[atomicAdd(nentry, 1ull)] = Entry{R, (int32_t)(sf - R), dst};
            R = child ? ef : sf;  // a child is skipped; else bucket f opens the next run
            from = child ? f + 1 : f;
        }
    }
    if (lane == 0 && bs[k] > R) entries[atomicAdd(nentry, 1ull)] = Entry{R, (int32_t)(bs[k] - R), dst};
}

__device__ void plan_block(SegParams *segs, const unsigned long long *nseg_ptr, int64_t *kfirst, int64_t *wfirst,
                           unsigned long long *ctrl, int32_t cap, int32_t kmax_child, int32_t min_tile,
                           int32_t child_fill, int32_t kcap) {
    const int nseg = (int)*(volatile const unsigned long long *)nseg_ptr;
    constexpr int NV = 4;  // tiles, matrix entries, records, bucket slots, windows -> 5 with windows
    __shared__ long long sh[5][32];
    __shared__ long long carry[5];
    __shared__ int kmax;
    __shared__ unsigned long long tot_rec;
    if (threadIdx.x < 5) carry[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        kmax = 1;
        tot_rec = 0;
    }
    __syncthreads();
    (void)NV;
    // tile length of the level: min_tile, raised (up to 4x) while the level
    // still yields ~8 tiles per SM -- long recursion levels then run fewer,
    // longer tiles (more pipelined rounds per CTA), short ones keep parallelism
    {
        unsigned long long t = 0;
        for (int q = threadIdx.x; q < nseg; q += blockDim.x) t += (unsigned long long)segs[q].len;
        t = warp_sum(t);
        if ((threadIdx.x & 31) == 0) atomicAdd(&tot_rec, t);
        __syncthreads();
        int64_t mt = (int64_t)(tot_rec / (unsigned long long)(148 * 8));
        mt = mt < min_tile ? min_tile : (mt > 4 * (int64_t)min_tile ? 4 * (int64_t)min_tile : mt);
        min_tile = (int32_t)((mt + 255) & ~(int64_t)255);
    }
    for (int base = 0; base < nseg; base += 1024) {
        int s = base + threadIdx.x;
        long long v[5] = {0, 0, 0, 0, 0};
        SegParams p;
        if (s < nseg) {
            p = segs[s];
            int64_t want = (p.len * child_fill + kcap - 1) / kcap;  // buckets ~ kcap / child_fill
            int k = 16;
            while (k < want && k < kmax_child) k <<= 1;
            p.k = k;
            if (p.mode == MODE_ZLIN && p.za == 0.0f) {  // a child ranged by the level-1 CDF: its fitted line
                p.scale = (double)k * (1.0 - 0x1p-20);
                const float za = (float)(p.scale / p.std);
                if (za > 0.0f && za < 3.0e38f) {
                    p.za = za;
                    p.zb = 0.0f;
                } else {  // degenerate range estimate: moments pass and Eq. 1 instead
                    p.mode = MODE_ZSCORE;
                    p.center = p.center + 0.5 * p.std;
                    atomicOr(&ctrl[C_NEED_STATS], 1ull);
                }
            }
            int64_t tl = max((int64_t)min_tile, (int64_t)4 * k);
            tl = (tl + 255) & ~(int64_t)255;
            p.tile_len = tl;
            p.ntiles = (int32_t)((p.len + tl - 1) / tl);
            // finish windows sized to the children's mean bucket a: a run is
            // the buckets starting in a window of cap - 1.3a records plus the
            // last of them when it has <= 1.3a records, so runs fill to
            // ~cap - 0.3a whatever the bucket size
            {
                const int64_t a = p.len / k;
                int64_t W = (int64_t)cap - (a * 13) / 10;
                W = min((int64_t)cap - 256, max((int64_t)cap / 4, W));
                p.win = (int32_t)W;
            }
            v[0] = p.ntiles;
            v[1] = (long long)p.ntiles * k;
            v[2] = p.len;
            v[3] = k + 1;
            v[4] = (p.len + p.win - 1) / p.win;
            atomicMax(&kmax, k);
        }
        long long x[5];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int j = 0; j < 5; j++) {
            x[j] = v[j];
            for (int o = 1; o < 32; o <<= 1) {
                long long y = __shfl_up_sync(0xffffffffu, x[j], o);
                if (lane >= o) x[j] += y;
            }
            if (lane == 31) sh[j][w] = x[j];
        }
        __syncthreads();
        long long pre[5];
#pragma unroll
        for (int j = 0; j < 5; j++) {
            pre[j] = carry[j];
            for (int q = 0; q < w; q++) pre[j] += sh[j][q];
        }
        if (s < nseg) {
            p.tile_first = pre[0] + x[0] - v[0];
            p.mat_base = pre[1] + x[1] - v[1];
            p.scan_base = pre[2] + x[2] - v[2];
            kfirst[s] = pre[3] + x[3] - v[3];
            wfirst[s] = pre[4] + x[4] - v[4];
            segs[s] = p;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
#pragma unroll
            for (int j = 0; j < 5; j++) carry[j] = pre[j] + x[j];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctrl[C_TILES_NEXT] = carry[0];
        ctrl[C_MAT_NEXT] = carry[1];
        ctrl[C_NEXT_BIG] = carry[3];
        ctrl[C_WIN_NEXT] = carry[4];
        ctrl[C_KMAX_NEXT] = kmax;
        kfirst[nseg] = carry[3];
        wfirst[nseg] = carry[4];
    }
}

// Finish order of a level's runs, longest first (64 length classes, any
// order inside a class): the persistent finish takes runs by ticket, so the
// last wave is short runs instead of whichever came last in key order.
__device__ void order_runs(const Entry *entries, const unsigned long long *nentry_ptr, int32_t *order, int cap) {
    constexpr int NCLS = 64;
    __shared__ uint32_t ccount[NCLS];
    const int ne = (int)*(volatile const unsigned long long *)nentry_ptr;
    if (threadIdx.x < NCLS) ccount[threadIdx.x] = 0;
    __syncthreads();
    auto cls = [&](int i) { return NCLS - 1 - min(NCLS - 1, (int)((int64_t)entries[i].len * NCLS / (cap + 1))); };
    for (int i = threadIdx.x; i < ne; i += blockDim.x) atomicAdd(&ccount[cls(i)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int c = 0; c < NCLS; c++) {
            const uint32_t v = ccount[c];
            ccount[c] = run;
            run += v;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ne; i += blockDim.x) order[atomicAdd(&ccount[cls(i)], 1u)] = i;
}

// Classify, one cooperative launch (1024-thread CTAs, grid barriers): bucket
// starts and child segments, then finish windows, then (CTA 0) the plan of
// the next level -- which rewrites kfirst/wfirst, hence the second barrier.
__global__ void __launch_bounds__(1024) k_classify(const SegParams *__restrict__ segs, int nseg, int64_t *kfirst,
                                                   int64_t *wfirst, const uint32_t *__restrict__ mat, int64_t *bstart,
                                                   SegParams *children, SegAcc *acc, Entry *entries,
                                                   unsigned long long *ctrl, ClassCfg cc, int64_t total_slots,
                                                   int64_t total_windows, Buffers B, int key_kind, int32_t kmax_child,
                                                   int32_t min_tile, unsigned long long *ref_zero, Entry *teams,
                                                   int32_t *order) {
    cg::grid_group grid = cg::this_grid();
    if (blockIdx.x == 0 && threadIdx.x < 4 && ref_zero) ref_zero[threadIdx.x] = 0ull;  // the finish's refine counts/tickets
    const int64_t G = (int64_t)gridDim.x * blockDim.x, g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t g = g0; g < total_slots; g += G)
        bstart_slot(g, segs, nseg, kfirst, mat, bstart, children, acc, ctrl, cc, B, key_kind, teams);
    grid.sync();
    // one segment (level 1): every CTA binary-searches a shared copy of its bucket starts
    constexpr int BS_SHARED = 2049;
    __shared__ int64_t bs_sh[BS_SHARED];
    const int64_t *bs_one = nullptr;
    if (nseg == 1 && segs[0].k + 1 <= BS_SHARED) {
        for (int q = threadIdx.x; q <= segs[0].k; q += blockDim.x) bs_sh[q] = bstart[kfirst[0] + q];
        __syncthreads();
        bs_one = bs_sh;
    }
    const int lane = lane_id();
    if (nseg > 1 && cc.greedy) {
        // recursion levels: greedy runs per segment, one warp each
        for (int64_t sg = g0 >> 5; sg < nseg; sg += G >> 5) {
            const SegParams p = segs[sg];
            if (p.mode == MODE_COPY) continue;
            greedy_runs(p, bstart + kfirst[sg], cc.cap, entries, &ctrl[C_NENTRY], lane);
        }
        total_windows = 0;
    }
    // windows: whole warps iterate together so each warp appends its entries
    // with one atomic (the entry counter is otherwise a hot spot)
    for (int64_t gw = g0 - lane; gw < total_windows; gw += G) {
        Entry e[2];
        const int ne = gw + lane < total_windows
                           ? window_item(gw + lane, segs, nseg, kfirst, wfirst, bstart, cc, bs_one, e)
                           : 0;
        int pre = ne;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
        }
        const int tot = __shfl_sync(0xffffffffu, pre, 31);
        unsigned long long base = 0;
        if (lane == 31 && tot) base = atomicAdd(&ctrl[C_NENTRY], (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 31);
        for (int q = 0; q < ne; q++) entries[base + pre - ne + q] = e[q];
    }
    grid.sync();
    if (blockIdx.x == 0)
        plan_block(children, ctrl + C_NCHILD, kfirst, wfirst, ctrl, cc.cap, kmax_child, min_tile, cc.child_fill,
                   cc.team_cap > cc.cap ? cc.team_cap : cc.cap);
    if (order && blockIdx.x == (gridDim.x > 1 ? 1 : 0)) order_runs(entries, ctrl + C_NENTRY, order, cc.cap);
}

// ------------------------------------------------------------------- K5
// Shared-memory stable finish of one run of whole buckets (len <= NT*F).
//  load    every thread issues its F key (and payload) loads up front and
//          keeps them in registers; item j of lane l of warp w is record
//          w*32F + j*32 + l (input order = record index);
//  minmax  exact ordered min/max of the run (block reduce; all-equal runs
//          are already in stable order and are copied through);
//  digits  d = floor((ord(key) - ord(min)) * S / (range + 1)) with S ~ m/2,
//          monotone in the key, so sub-bucket order is key order;
//  count   shared-memory atomic histogram of the digits, exclusive scan;
//  place   records go to their sub-bucket with an atomic cursor (any order)
//          together with their record index;
//  rank    each record's rank inside its sub-bucket is the number of
//          members with a smaller (key, record index): equal keys keep input
//          order, so the result is the stable sort; it is stored straight to
//          its final position.
// Sub-buckets above `fin_ins` records take a stable path instead: records
// of those digits are re-placed in input order by per-(digit, warp)
// counters advanced by __match_any_sync leaders; if such a sub-bucket is not
// already ordered (it is whenever its keys are all equal) it is emitted as a
// refine run and finished again by a later launch (its key range shrinks by
// a factor ~S each time, so this terminates).  All loads complete before any
// output store, so src may alias the output (in-place refinement).

constexpr int FIN_INS = 32;         // sub-buckets up to this size are ranked by comparison
constexpr int FIN_SBITS_MAX = 13;   // <= 8192 sub-buckets (16-bit cursors)
#ifndef ZSB_FT
#define ZSB_FT 1024  // threads per finish CTA; 512: two CTAs per SM with half the run capacity (experiment, needs -DZSB_TEAM=0)
#endif
constexpr int FIN_BIG_MAX = ZSB_FT == 1024 ? 384 : 192;  // >= cap / (FIN_INS + 1): every oversized sub-bucket fits

constexpr int FT = ZSB_FT;      // threads per finish CTA
constexpr int FIN_CTAS = 1024 / FT;  // finish CTAs per SM
constexpr int FW = FT / 32;     // warps per finish CTA

template <int PB>
struct FinItems {
    static constexpr int F = PB == 8 ? 8 : 12;  // records per thread; cap = FT * F
};

struct FinLayout {
    int cap;
    size_t off_o, off_pb, off_i, off_cur, off_bcnt, total;
};

__host__ __device__ inline FinLayout fin_layout(int cap, int pb) {
    FinLayout L;
    L.cap = cap;
    size_t o = 0;
    L.off_o = o;  // placement buffer; first the keys staged in input order (+16 B alignment slack)
    o += (size_t)cap * 8 + 16;
    L.off_pb = o;  // payload staged in input order by a TMA bulk copy (+16 B alignment slack)
    o += (size_t)cap * pb + (pb ? 16 : 0);
    o = (o + 15) & ~(size_t)15;
    L.off_i = o;
    o += (size_t)cap * 2;
    o = (o + 15) & ~(size_t)15;
    L.off_cur = o;  // S 16-bit counters/cursors, packed two per word
    o += (size_t)(1 << FIN_SBITS_MAX) * 2;
    o = (o + 15) & ~(size_t)15;
    L.off_bcnt = o;
    o += (size_t)FIN_BIG_MAX * FW * 2 + (1 << FIN_SBITS_MAX) / 8 + 16;
    o = (o + 15) & ~(size_t)15;
    L.total = o;
    return L;
}

// TMA staging of a contiguous range src[0, m) into shared memory with the
// same address phase modulo 16, so element i lands at st + i: one bulk copy
// of the 16-byte-aligned interior plus plain loads of the ragged head
// [0, h) and tail [t0, m) (a few elements).
struct StageSpan {
    uintptr_t a16;    // first aligned byte of the interior
    uint32_t bytes;   // interior bytes (0: no bulk part)
    uint32_t phase;   // A & 15
    int h, t0;
};

__device__ __forceinline__ StageSpan stage_span(const void *src, int m, int esz) {
    const uintptr_t A = (uintptr_t)src, E = A + (uintptr_t)m * esz;
    const uintptr_t A16 = (A + 15) & ~(uintptr_t)15, E16 = E & ~(uintptr_t)15;
    const bool bulk = E16 > A16;
    return StageSpan{A16, bulk ? (uint32_t)(E16 - A16) : 0u, (uint32_t)(A & 15),
                     bulk ? (int)((A16 - A) / esz) : m, bulk ? (int)((E16 - A) / esz) : m};
}

// Stage the keys (and payload) of a finish run into shared memory: thread 0
// arms bar[0] with the key bytes and bar[1] with the payload bytes and issues
// the bulk copies; warps 1 and 2 load the ragged ends.  Callers wait on
// bar[0] and barrier before reading keys, and on bar[1] (one phase per run,
// armed even without payload bytes) before reading the payload, which is
// needed only at the final store: its copy lands while the keys are ranked.
template <typename P, int PB>
__device__ __forceinline__ void stage_run(unsigned char *karea, const uint64_t *sk, unsigned char *parea, const P *sp,
                                          int m, uint64_t *bar, const uint64_t *&kst, const P *&pst) {
    const StageSpan ks = stage_span(sk, m, 8);
    uint64_t *kd = (uint64_t *)(karea + ks.phase);
    kst = kd;
    StageSpan ps{};
    P *pd = nullptr;
    if constexpr (PB != 0) {
        ps = stage_span(sp, m, PB);
        pd = (P *)(parea + ps.phase);
        pst = pd;
    }
    const int tid = threadIdx.x;
    if (tid == 0) {
        fence_proxy_async_smem();
        mbar_expect_tx(&bar[0], ks.bytes);
        mbar_expect_tx(&bar[1], ps.bytes);
        if (ks.bytes) bulk_g2s((unsigned char *)kd + (ks.a16 - (uintptr_t)sk), (const void *)ks.a16, ks.bytes, &bar[0]);
        if (PB != 0 && ps.bytes)
            bulk_g2s((unsigned char *)pd + (ps.a16 - (uintptr_t)sp), (const void *)ps.a16, ps.bytes, &bar[1]);
    } else if (tid >= 32 && tid < 64) {  // key ends
        const int q = tid - 32;
        if (q < ks.h) kd[q] = sk[q];
        else if (q - ks.h < m - ks.t0) kd[ks.t0 + q - ks.h] = sk[ks.t0 + q - ks.h];
    } else if (PB != 0 && tid >= 64 && tid < 96) {  // payload ends
        const int q = tid - 64;
        if (q < ps.h) pd[q] = sp[q];
        else if (q - ps.h < m - ps.t0) pd[ps.t0 + q - ps.h] = sp[ps.t0 + q - ps.h];
    }
}

template <int KK, int PB>
__device__ __forceinline__ void finish_entry(const Buffers &B, const Entry e, int64_t eidx, int cap, Entry *refine,
                                             unsigned long long *refine_count, int fin_ins, long long *prof,
                                             uint64_t *bar, uint32_t &parity) {
#define FIN_MARK(slot)                                                                                   \
    do {                                                                                                 \
        if (prof && threadIdx.x == 0) prof[eidx * 8 + (slot)] = clock64();                              \
    } while (0)
    FIN_MARK(0);
    using P = typename PayloadT<PB>::T;
    constexpr int F = FinItems<PB>::F;
    extern __shared__ __align__(16) unsigned char smem[];
    const FinLayout L = fin_layout(cap, PB);
    uint64_t *Bo = (uint64_t *)(smem + L.off_o);  // ordered key images, placed
    uint16_t *Ix = (uint16_t *)(smem + L.off_i);  // record index of each placed element
    uint32_t *cw = (uint32_t *)(smem + L.off_cur);  // 16-bit counters, two per word
    uint16_t *bcnt = (uint16_t *)(smem + L.off_bcnt);
    uint32_t *bigmask = (uint32_t *)(smem + L.off_bcnt + FIN_BIG_MAX * FW * 2);
    __shared__ unsigned long long r_min[FW], r_max[FW];
    __shared__ uint32_t wsum[FW];
    __shared__ uint32_t negzero[FT];  // float64: bit per record index that was -0.0 (cap <= 16384)
    __shared__ int nbig;
    __shared__ uint16_t bslot[FIN_BIG_MAX];  // sorted oversized digits

    const int m = e.len;
    if (m <= 0) return;
    ZSB_CHECK(m <= cap && e.start >= 0 && e.start + m <= B.n);
    const uint64_t *sk = src_keys(B, e.src) + e.start;
    const P *sp = src_pay<PB>(B, e.src) + e.start;
    uint64_t *ok = B.out_k + e.start;
    P *op = (P *)B.out_p + e.start;
    const int tid = threadIdx.x, w = tid >> 5, lane = lane_id();
    const int base = w * 32 * F + lane;
    // keys and payload arrive in input order by TMA bulk copies (the copy
    // engine keeps far more bytes in flight than per-thread loads); keys are
    // staged in the placement buffer, which is free until placement, and
    // moved to registers; the payload stays staged and is gathered by
    // record index at the store
    const uint64_t *kin = nullptr;
    const P *pin = nullptr;
    stage_run<P, PB>(smem + L.off_o, sk, smem + L.off_pb, sp, m, bar, kin, pin);
    // sub-bucket count S depends on m only: clear the counters while the copies land
    // S = the smallest power of two >= 2m (>= 32), capped at 2^FIN_SBITS_MAX
    const int sbits = min(FIN_SBITS_MAX, max(5, 33 - __clz(m > 1 ? m - 1 : 1)));
    const int S = 1 << sbits;
    for (int q = tid; q < S / 2; q += FT) cw[q] = 0u;
    for (int q = tid; q < S / 32; q += FT) bigmask[q] = 0u;
    mbar_wait(&bar[0], parity);
    __syncthreads();
    FIN_MARK(7);  // staged

    // items past the run end load a copy of the last key (no effect on the
    // min/max); the histogram and the placement skip them.  A warp whose
    // items all lie inside the run (`wfull`, all but the last warps) runs
    // the unchecked loop bodies.
    const bool wfull = (w + 1) * 32 * F <= m;
    uint64_t o[F];
#pragma unroll
    for (int j = 0; j < F; j++) o[j] = kin[min(base + j * 32, m - 1)];
    if (tid == 0) nbig = 0;
    bool anyneg = false;
    if constexpr (KK == KEY_F64) {
        negzero[tid] = 0u;
#pragma unroll
        for (int j = 0; j < F; j++) anyneg |= (o[j] == SIGN);
    }
    unsigned long long omin = ~0ull, omax = 0;
#pragma unroll
    for (int j = 0; j < F; j++) {
        o[j] = ord_key<KK>(o[j]);
        omin = min(omin, (unsigned long long)o[j]);
        omax = max(omax, (unsigned long long)o[j]);
    }
    omin = warp_min_u64(omin);
    omax = warp_max_u64(omax);
    if (lane == 0) {
        r_min[w] = omin;
        r_max[w] = omax;
    }
    if constexpr (KK == KEY_F64) anyneg = __syncthreads_or(anyneg);
    else __syncthreads();
    FIN_MARK(1);  // loads landed
    if constexpr (KK == KEY_F64) {
        if (anyneg) {  // -0.0 and +0.0 share an ordered image; remember which records were -0.0
#pragma unroll
            for (int j = 0; j < F; j++)
                if (base + j * 32 < m && o[j] == ord_key<KK>(SIGN) && kin[base + j * 32] == SIGN)
                    atomicOr(&negzero[(base + j * 32) >> 5], 1u << lane);
            __syncthreads();
        }
    }
    omin = warp_min_u64(lane < FW ? r_min[lane] : ~0ull);  // every warp reduces the warp partials itself
    omax = warp_max_u64(lane < FW ? r_max[lane] : 0ull);
    if constexpr (KK == KEY_F64) {
        // NaNs order outside [-inf, +inf] in the ordered image: a run holding
        // one raises ZSB_ERR_NAN (the small-n path reaches no other screen)
        if (tid == 0 && B.status && (omax > ORD_PINF || omin < ORD_NINF)) *B.status = 3ull;
    }
    auto key_bits = [&](uint64_t ov, int idx) -> uint64_t {
        uint64_t kb = key_from_ord<KK>(ov);
        if (KK == KEY_F64 && anyneg && ((negzero[idx >> 5] >> (idx & 31)) & 1u)) kb = SIGN;
        return kb;
    };
    if (omin == omax) {  // all equal: already in stable order
        mbar_wait(&bar[1], parity);  // payload staged
        parity ^= 1u;
        if (e.src != 2) {
#pragma unroll
            for (int j = 0; j < F; j++) {
                const int i = base + j * 32;
                if (i < m) {
                    ok[i] = key_bits(o[j], i);
                    if constexpr (PB != 0) op[i] = pin[i];
                }
            }
        }
        return;
    }
    const uint64_t range = omax - omin;
    // When (ord - min) leaves 14 free bits, the placed image is packed as
    // (ord - min) << 14 | record index: one 64-bit compare then orders by
    // (key, index), and the index needs no separate shared array.
    constexpr int IB = 14;  // cap <= 16384
    const bool packed = bitlen64(range) + IB <= 64;
    const bool direct = range < (uint64_t)S;  // one key value per digit
    // d = ((ord - min) >> sh) * M >> 32 with the shifted range below 2^32:
    // monotone in the key and < S; 32-bit multiply only
    const int sh = max(0, bitlen64(range) - 32);
    const uint32_t r32 = (uint32_t)(range >> sh);
    // M <= S * 2^32 / (r32 + 1) (division rounded toward zero, then truncated),
    // so umulhi(x, M) < S for every x <= r32; a 64-bit integer division would
    // cost every thread ~70 instructions
    const uint32_t M = direct ? 0u
                              : (uint32_t)fmin(4294967295.0, __ddiv_rz((double)S * 4294967296.0, (double)r32 + 1.0));
    // float64 keys over a finite range take their digit in value space: the
    // ordered images are exponentially non-uniform near 0 (a run straddling
    // 0 would crowd into a few digits).  Rounded subtraction and product by a
    // positive constant keep the digit monotone in the key.
    bool vdig = false;
    double vlo = 0.0, vinv = 0.0;
    if constexpr (KK == KEY_F64) {
        const double lo = key_value<KK>(key_from_ord<KK>(omin)), hi = key_value<KK>(key_from_ord<KK>(omax));
        const double span = __dsub_rn(hi, lo);
        vinv = (double)S * __drcp_rn(span);  // any positive scale keeps the digit monotone (clamped to S - 1)
#ifndef ZSB_FIN_VDIG
#define ZSB_FIN_VDIG 1
#endif
        // inside one sign and at most two adjacent binades the ordered image is
        // linear in the value to within 2x: keep the cheaper integer digit there
        const uint64_t blo = key_from_ord<KK>(omin), bhi = key_from_ord<KK>(omax);
        const int elo = (int)((blo >> 52) & 0x7FF), ehi = (int)((bhi >> 52) & 0x7FF);
        const bool linear = ((blo ^ bhi) >> 63) == 0 && abs(ehi - elo) <= 1;
        vdig = ZSB_FIN_VDIG && !linear && isfinite(lo) && isfinite(hi) && span > 0.0 && isfinite(span) &&
               isfinite(vinv) && !direct;
        vlo = lo;
    }
    // digit of an ordered image; VD = value-space (float64 runs spanning
    // binades), else the integer map (`direct` folds into M = 2^32 with sh = 0)
    auto digit_t = [&](auto vd_t, uint64_t ov) -> int {
        if constexpr (decltype(vd_t)::value) {
            const int d = (int)__dmul_rn(__dsub_rn(key_value<KK>(key_from_ord<KK>(ov)), vlo), vinv);
            return d < S ? d : S - 1;
        } else {
            const uint64_t x = ov - omin;
            return direct ? (int)x : (int)__umulhi((uint32_t)(x >> sh), M);
        }
    };
    auto digit = [&](uint64_t ov) -> int {
        return (KK == KEY_F64 && vdig) ? digit_t(std::true_type{}, ov) : digit_t(std::false_type{}, ov);
    };
    FIN_MARK(2);
    // ---- histogram (16-bit counters: no carry, counts <= cap < 2^16)
    uint32_t dpk[(F + 1) / 2];  // digits, two per register
    auto hist_t = [&](auto vd_t, auto full_t) {
        constexpr bool FULL = decltype(full_t)::value;
#pragma unroll
        for (int j = 0; j < F; j++) {
            const int d = (FULL || base + j * 32 < m) ? digit_t(vd_t, o[j]) : 0xFFFF;
            if (j & 1) dpk[j >> 1] |= (uint32_t)d << 16;
            else dpk[j >> 1] = (uint32_t)d;
            if (FULL || d != 0xFFFF) atomicAdd(&cw[d >> 1], 1u << (16 * (d & 1)));
        }
    };
    if (KK == KEY_F64 && vdig) {
        if (wfull) hist_t(std::true_type{}, std::true_type{});
        else hist_t(std::true_type{}, std::false_type{});
    } else {
        if (wfull) hist_t(std::false_type{}, std::true_type{});
        else hist_t(std::false_type{}, std::false_type{});
    }
    __syncthreads();
    FIN_MARK(3);
    // ---- exclusive scan of the counters in place (they become the cursors;
    //      after placement cursor d = start of d + 1, so no separate start
    //      table); flag oversized digits.  Thread t owns digits
    //      [t*per, (t+1)*per), per = S/FT in {0 (S < FT), 1, 2, 4, 8, 16, 32},
    //      with 16-byte vector accesses from 8 on.
    {
        uint16_t *c16 = (uint16_t *)cw;
        const int per = S / FT;
        const int d0 = per ? tid * per : (tid < S ? tid : S), d1 = per ? d0 + per : (tid < S ? tid + 1 : S);
        auto sum8 = [](uint4 u) {
            return (u.x & 0xffffu) + (u.x >> 16) + (u.y & 0xffffu) + (u.y >> 16) + (u.z & 0xffffu) + (u.z >> 16) +
                   (u.w & 0xffffu) + (u.w >> 16);
        };
        uint32_t tsum = 0;
        if (per >= 8) {
            for (int q = 0; q < per; q += 8) tsum += sum8(*(const uint4 *)(c16 + d0 + q));
        } else {
            for (int d = d0; d < d1; d++) tsum += c16[d];
        }
        uint32_t x = tsum;
#pragma unroll
        for (int q = 1; q < 32; q <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, q);
            if (lane >= q) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        uint32_t run = x - tsum + warps_before(wsum, w, lane);
        auto excl = [&](uint32_t v, int d) -> uint32_t {  // start of digit d (count v); flags oversized
            const uint32_t st = run;
            if (v > (uint32_t)fin_ins) {
                const int bi = atomicAdd(&nbig, 1);
                if (bi < FIN_BIG_MAX) bslot[bi] = (uint16_t)d;
                atomicOr(&bigmask[d >> 5], 1u << (d & 31));
            }
            run += v;
            return st;
        };
        if (per >= 8) {
            for (int q = 0; q < per; q += 8) {
                const uint4 u = *(const uint4 *)(c16 + d0 + q);
                const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
                uint32_t ov[4];
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    const uint32_t lo = excl(wv[r] & 0xffffu, d0 + q + 2 * r);
                    const uint32_t hi = excl(wv[r] >> 16, d0 + q + 2 * r + 1);
                    ov[r] = lo | (hi << 16);
                }
                *(uint4 *)(c16 + d0 + q) = make_uint4(ov[0], ov[1], ov[2], ov[3]);
            }
        } else {
            for (int d = d0; d < d1; d++) c16[d] = (uint16_t)excl(c16[d], d);
        }
    }
    __syncthreads();
    const int nb = nbig;  // <= m / (fin_ins + 1) <= FIN_BIG_MAX
    FIN_MARK(4);
    // ---- place (atomic cursors; oversized digits go through the stable path)
    auto place_t = [&](auto pk_t, auto big_t, auto full_t) {
#pragma unroll
        for (int j = 0; j < F; j++) {
            const int d = (int)((dpk[j >> 1] >> (16 * (j & 1))) & 0xFFFF);
            bool go = decltype(full_t)::value || d != 0xFFFF;
            if constexpr (decltype(big_t)::value) go = go && !((bigmask[d >> 5] >> (d & 31)) & 1u);
            if (go) {
                const uint32_t old = atomicAdd(&cw[d >> 1], 1u << (16 * (d & 1)));
                const uint32_t pos = (old >> (16 * (d & 1))) & 0xFFFFu;
                const uint32_t ri = (uint32_t)(base + j * 32);
                ZSB_CHECK(d < S && pos < (uint32_t)m && ri < (uint32_t)m);
                if constexpr (decltype(pk_t)::value) {
                    Bo[pos] = ((o[j] - omin) << IB) | ri;
                } else {
                    Bo[pos] = o[j];
                    Ix[pos] = (uint16_t)ri;
                }
            }
        }
    };
    if (packed) {
        if (nb) place_t(std::true_type{}, std::true_type{}, std::false_type{});
        else if (wfull) place_t(std::true_type{}, std::false_type{}, std::true_type{});
        else place_t(std::true_type{}, std::false_type{}, std::false_type{});
    } else {
        if (nb) place_t(std::false_type{}, std::true_type{}, std::false_type{});
        else place_t(std::false_type{}, std::false_type{}, std::false_type{});
    }
    if (nb > 0) {
        // Stable placement of the oversized digits: sort their digit list,
        // then per-(slot, warp) counters advanced in input order.
        __syncthreads();
        if (tid < nb) {
            const int dv = bslot[tid];
            int rank = 0;
            for (int q = 0; q < nb; q++) rank += bslot[q] < dv;
            ((uint16_t *)bcnt)[FIN_BIG_MAX * FW - 1 - rank] = (uint16_t)dv;
        }
        __syncthreads();
        if (tid < nb) bslot[tid] = ((uint16_t *)bcnt)[FIN_BIG_MAX * FW - 1 - tid];
        __syncthreads();
        for (int q = tid; q < nb * FW; q += FT) bcnt[q] = 0;
        __syncthreads();
        const unsigned lt = lanemask_lt();
        auto slot_of = [&](int j) -> int {  // slot of item j's digit, -1 unless oversized
            const int d = (int)((dpk[j >> 1] >> (16 * (j & 1))) & 0xFFFF);
            if (d == 0xFFFF || !((bigmask[d >> 5] >> (d & 31)) & 1u)) return -1;
            int lo = 0, hi = nb - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (bslot[mid] < d) lo = mid + 1;
                else hi = mid;
            }
            return lo;
        };
#pragma unroll
        for (int j = 0; j < F; j++) {
            const int sl = slot_of(j);
            const unsigned peers = __match_any_sync(0xffffffffu, sl);
            if (sl >= 0 && (peers & lt) == 0) {
                const int q = sl * FW + w;
                atomicAdd((uint32_t *)bcnt + (q >> 1), (uint32_t)__popc(peers) << (16 * (q & 1)));
            }
        }
        __syncthreads();
        for (int q = tid; q < nb; q += FT) {  // exclusive prefix over warps from the digit's start
            uint16_t *cur_d = (uint16_t *)cw + bslot[q];
            uint32_t run = *cur_d;  // not advanced by the atomic placement: still the start
            for (int ww = 0; ww < FW; ww++) {
                const uint32_t c = bcnt[q * FW + ww];
                bcnt[q * FW + ww] = (uint16_t)run;
                run += c;
            }
            *cur_d = (uint16_t)run;  // end of the digit, like every other cursor
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < F; j++) {
            const int sl = slot_of(j);
            const unsigned peers = __match_any_sync(0xffffffffu, sl);
            const int leader = __ffs(peers) - 1;
            uint32_t b0 = 0;
            if (sl >= 0 && lane == leader) {
                b0 = bcnt[sl * FW + w];
                bcnt[sl * FW + w] = (uint16_t)(b0 + __popc(peers));
            }
            __syncwarp();
            b0 = __shfl_sync(0xffffffffu, b0, leader);
            if (sl >= 0) {
                const uint32_t pos = b0 + __popc(peers & lt);
                ZSB_CHECK(pos < (uint32_t)m);
                const uint32_t ri = (uint32_t)(base + j * 32);
                if (packed) {
                    Bo[pos] = ((o[j] - omin) << IB) | ri;
                } else {
                    Bo[pos] = o[j];
                    Ix[pos] = (uint16_t)ri;
                }
            }
        }
    }
    __syncthreads();
    FIN_MARK(5);
    // ---- rank inside each sub-bucket by (key, record index) and store to
    //      the final position; ties keep input order (stable)
    // (one loop per (packed, digit) combination: the flags are uniform per run)
    auto rank_t = [&](auto pk_t, auto vd_t, auto neg_t) {
        constexpr bool PK = decltype(pk_t)::value;
        // NEG = false: the run holds no -0.0 (checked once per run), so the
        // key bits are the inverse ordered image with no per-record test
        auto key_out = [&](uint64_t ov, int idx) -> uint64_t {
            if constexpr (decltype(neg_t)::value) return key_bits(ov, idx);
            else return key_from_ord<KK>(ov);
        };
        for (int i = tid; i < m; i += FT) {
            const uint64_t pv = Bo[i];
            const uint64_t ov = PK ? (pv >> IB) + omin : pv;
            const int idx = PK ? (int)(pv & ((1u << IB) - 1)) : (int)Ix[i];
            const int d = digit_t(vd_t, ov);
            const int a = d ? (int)((const uint16_t *)cw)[d - 1] : 0, z = ((const uint16_t *)cw)[d];
            const int c = z - a;
            int rank = i - a;
            if (c <= fin_ins) {
                if (c > 1 && c <= 4) {
                    // the common sizes (S >= m/2 sub-buckets: ~1-3 records):
                    // four masked compares, no loop; reads past z stay
                    // inside the shared-memory allocation and are masked
                    rank = 0;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint64_t ox = Bo[a + q];
                        if constexpr (PK) rank += (q < c) & (ox < pv);
                        else rank += (q < c) & ((ox < ov) || (ox == ov && Ix[a + q] < idx));
                    }
                } else if (c > 4) {
                    rank = 0;
                    for (int x = a; x < z; x++) {
                        const uint64_t ox = Bo[x];
                        if constexpr (PK) rank += ox < pv;
                        else rank += (ox < ov) || (ox == ov && Ix[x] < idx);
                    }
                }
            } else if (i == a) {  // oversized sub-bucket, placed stably: refine unless already ordered
                bool sorted = true;
                for (int x = a + 1; x < z && sorted; x++) sorted = Bo[x - 1] <= Bo[x];
                if (!sorted) {
                    unsigned long long r = atomicAdd(refine_count, 1ull);
                    refine[r] = Entry{e.start + a, c, 2};
                }
            }
            ZSB_CHECK(a + rank >= 0 && a + rank < m && idx >= 0 && idx < m && z <= m);
            ok[a + rank] = key_out(ov, idx);
            if constexpr (PB != 0) op[a + rank] = pin[idx];
        }
    };
    mbar_wait(&bar[1], parity);  // payload staged (landed while the keys were ranked)
    parity ^= 1u;
    const bool vd = KK == KEY_F64 && vdig;
    const bool neg = KK == KEY_F64 && anyneg;
    if (packed) {
        if (vd) rank_t(std::true_type{}, std::true_type{}, std::true_type{});
        else if (!neg) rank_t(std::true_type{}, std::false_type{}, std::false_type{});
        else rank_t(std::true_type{}, std::false_type{}, std::true_type{});
    } else {
        if (vd) rank_t(std::false_type{}, std::true_type{}, std::true_type{});
        else rank_t(std::false_type{}, std::false_type{}, std::true_type{});
    }
    FIN_MARK(6);
#undef FIN_MARK
}

// L2 prefetch of a finish run's keys and payload (aligned interiors).
template <int PB>
__device__ __forceinline__ void finish_prefetch(const Buffers &B, const Entry e) {
    using P = typename PayloadT<PB>::T;
    if (e.len <= 0) return;
    const StageSpan ks = stage_span(src_keys(B, e.src) + e.start, e.len, 8);
    if (ks.bytes) prefetch_l2_bulk((const void *)ks.a16, ks.bytes);
    if constexpr (PB != 0) {
        const StageSpan ps = stage_span(src_pay<PB>(B, e.src) + e.start, e.len, PB);
        if (ps.bytes) prefetch_l2_bulk((const void *)ps.a16, ps.bytes);
    }
}

// Persistent finish over one run list; dynamic scheduling with a lookahead
// of one run: a CTA holds the ticket of its next run while it finishes the
// current one and (`prefetch`: the level's records do not fit L2, so the
// scatter's evict_last runs are not all resident) has the copy engine
// prefetch that run's keys and payload into L2, so its staging copies hit L2
// instead of waiting on HBM.
template <int KK, int PB>
__device__ __forceinline__ void finish_list(const Buffers &B, const Entry *__restrict__ entries, int64_t ne, int cap,
                                            Entry *refine, unsigned long long *refine_count, int fin_ins,
                                            long long *prof, unsigned long long *ticket, int prefetch, uint64_t *bar,
                                            uint32_t &parity, const int32_t *order = nullptr) {
    __shared__ long long next, cur_s;
    long long cur = 0;
    if (threadIdx.x == 0) cur = (long long)atomicAdd(ticket, 1ull);
    while (true) {
        if (threadIdx.x == 0) {
            const long long nx = (long long)atomicAdd(ticket, 1ull);
            next = nx;
            if (nx < ne && prefetch) finish_prefetch<PB>(B, entries[order ? order[nx] : nx]);
        }
        if (threadIdx.x == 0) cur_s = cur;
        __syncthreads();
        const int64_t i = cur_s;
        cur = next;
        if (i >= ne) break;
        const int64_t ei = order ? order[i] : i;
        finish_entry<KK, PB>(B, entries[ei], ei, cap, refine, refine_count, fin_ins, prof, bar, parity);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K5t
// Team finish: a run of cap < m <= TEAM * cap records -- a bucket too large
// for one CTA's shared memory, which would otherwise cost another partition
// level -- is finished by a thread-block cluster of TEAM CTAs (sample sort
// of one run, the exchange through L2):
//   stage     CTA r stages the contiguous chunk r of ceil(m / TEAM) records
//             (TMA bulk copies, input order) and publishes TEAM_SAMP evenly
//             spaced samples and its extremes (DSMEM);
//   splitters every CTA sorts the cluster's 1024 samples (bitonic, warp
//             shuffles below 32) and takes TEAM - 1 splitters s_j at equal
//             sample ranks;
//   parts     2 TEAM - 1 parts in key order: (s_{j-1}, s_j) and {s_j}; an
//             equality part is final once its records are in input order;
//   exchange  every record goes to its part in the output buffer at part
//             start + part records of lower-ranked chunks + its rank among
//             its chunk's records of that part (ballot multi-split in record
//             order: stable); the stores stay in L2 for the next step;
//   finish    after a cluster barrier, CTA r finishes the open part 2r
//             (finish_entry in place, staged from L2).
// An open part that still holds more than cap records (the samples missed
// its mass) is pushed on the team's stack -- identical in every CTA -- and
// finished the same way; its keys exclude the splitter values, so every
// pass removes distinct values and this terminates.
#ifndef ZSB_TEAM
#define ZSB_TEAM 8  // CTAs per team; 0: no team runs
#endif
constexpr bool TEAM_ON = ZSB_TEAM > 0;
constexpr int TEAM = ZSB_TEAM > 0 ? ZSB_TEAM : 8;  // CTAs per team (thread-block cluster size)
constexpr int TEAM_NS = 1024;                     // samples of a run (one per thread of the sort)
constexpr int TEAM_SAMP = TEAM_NS / TEAM;         // samples per chunk
constexpr int TEAM_PARTS = 2 * TEAM - 1;          // open and equality parts
constexpr int TEAM_PBITS = TEAM <= 2 ? 2 : (TEAM <= 4 ? 3 : (TEAM <= 8 ? 4 : 5));  // ballots per record
constexpr int TEAM_STACK = 8 * TEAM;              // oversized open parts: < TEAM per run and level

struct TeamShared {
    unsigned long long omin, omax;          // this CTA's chunk extremes (read by the peers)
    unsigned long long rmin, rmax;          // the run's extremes
    unsigned long long wmin[FW], wmax[FW];  // warp partials
    unsigned long long split[TEAM];         // splitters s_0 .. s_{TEAM-2}
    long long ticket;                       // rank 0: the team's run ticket (read by the peers)
    long long tk;                           // local copy of rank 0's ticket
    uint32_t pcnt[TEAM_PARTS];              // this CTA's records per part (read by the peers)
    uint32_t pstart[TEAM_PARTS + 1];        // part starts (offsets in the run)
    uint32_t pbase[TEAM_PARTS];             // this CTA's first slot in each part
    int sp;                                 // stack depth (the same in every CTA)
    Entry stack[TEAM_STACK];
};

// Ascending sort of one u64 per thread across the 1024-thread CTA; a[] is
// 1024 words of shared scratch.  Returns the thread's element of the result.
__device__ __forceinline__ unsigned long long bitonic_1024(unsigned long long v, unsigned long long *a) {
    const int t = threadIdx.x;
#pragma unroll 1
    for (int k = 2; k <= 1024; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            unsigned long long y;
            if (j >= 32) {
                a[t] = v;
                __syncthreads();
                y = a[t ^ j];
                __syncthreads();
            } else {
                y = __shfl_xor_sync(0xffffffffu, v, j);
            }
            const bool up = (t & k) == 0, low = (t & j) == 0;
            v = (low == up) ? min(v, y) : max(v, y);
        }
    }
    return v;
}

template <int KK, int PB>
__device__ __forceinline__ int team_run(const Buffers &B, const Entry e, int cap, Entry *refine,
                                        unsigned long long *refine_count, int fin_ins, uint64_t *bar,
                                        uint32_t &parity, TeamShared &ts) {
    using P = typename PayloadT<PB>::T;
    constexpr int F = FinItems<PB>::F;
    static_assert(!TEAM_ON || FT == TEAM_NS, "one sample per thread of the splitter sort");
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cl = cg::this_cluster();
    const FinLayout L = fin_layout(cap, PB);
    unsigned long long *samp = (unsigned long long *)(smem + L.off_i);  // TEAM_SAMP samples (read by the peers)
    unsigned long long *sortbuf = samp + TEAM_SAMP;                     // bitonic scratch (1024 words)
    uint16_t *wcnt = (uint16_t *)(smem + L.off_bcnt);                   // [part][warp] counts, then cursors
    const int tid = threadIdx.x, w = tid >> 5, lane = lane_id();
    const unsigned lt = lanemask_lt();
    const int r = (int)cl.block_rank();
    const int m = e.len;
    ZSB_CHECK(m > 0 && m <= TEAM * cap && e.start >= 0 && e.start + m <= B.n);
    const int q = (m + TEAM - 1) / TEAM;
    const int c0 = min(m, r * q), mc = min(m, c0 + q) - c0;
    const uint64_t *kin = nullptr;
    const P *pin = nullptr;
    stage_run<P, PB>(smem + L.off_o, src_keys(B, e.src) + e.start + c0, smem + L.off_pb,
                     src_pay<PB>(B, e.src) + e.start + c0, mc, bar, kin, pin);
    for (int x = tid; x < TEAM_PARTS * FW; x += FT) wcnt[x] = 0;
    mbar_wait(&bar[0], parity);
    __syncthreads();
    const int base = w * 32 * F + lane;
    uint64_t o[F];
    unsigned long long mn = ~0ull, mx = 0ull;
#pragma unroll
    for (int j = 0; j < F; j++) {
        const int i = base + j * 32;
        o[j] = i < mc ? ord_key<KK>(kin[i]) : 0ull;
        if (i < mc) {
            mn = min(mn, (unsigned long long)o[j]);
            mx = max(mx, (unsigned long long)o[j]);
        }
    }
    if (tid < TEAM_SAMP)  // evenly spaced samples of the chunk (mc >= TEAM_SAMP for every team run)
        samp[tid] = mc ? ord_key<KK>(kin[min(mc - 1, (int)(((2 * tid + 1) * (int64_t)mc) / (2 * TEAM_SAMP)))]) : ~0ull;
    mn = warp_min_u64(mn);
    mx = warp_max_u64(mx);
    if (lane == 0) {
        ts.wmin[w] = mn;
        ts.wmax[w] = mx;
    }
    __syncthreads();
    if (w == 0) {
        mn = warp_min_u64(ts.wmin[lane]);
        mx = warp_max_u64(ts.wmax[lane]);
        if (lane == 0) {
            ts.omin = mn;
            ts.omax = mx;
        }
    }
    cl.sync();  // #1: extremes and samples published; every chunk is staged (the run may be overwritten in place)
    if (w == 0) {
        unsigned long long a = ~0ull, z = 0ull;
        if (lane < TEAM) {
            const TeamShared *peer = cl.map_shared_rank(&ts, lane);
            a = peer->omin;
            z = peer->omax;
        }
        a = warp_min_u64(a);
        z = warp_max_u64(z);
        if (lane == 0) {
            ts.rmin = a;
            ts.rmax = z;
        }
    }
    const unsigned long long sv = cl.map_shared_rank(samp, tid / TEAM_SAMP)[tid % TEAM_SAMP];
    __syncthreads();
    const uint64_t rmin = ts.rmin, rmax = ts.rmax;
    if (rmin == rmax) {  // all keys equal: already in stable order
        mbar_wait(&bar[1], parity);
        parity ^= 1u;
        if (e.src != 2) {
            uint64_t *ok = B.out_k + e.start + c0;
            P *op = (P *)B.out_p + e.start + c0;
            for (int i = tid; i < mc; i += FT) {
                ok[i] = kin[i];
                if constexpr (PB != 0) op[i] = pin[i];
            }
        }
        cl.sync();  // peers are done reading this CTA's samples
        return 0;
    }
    const unsigned long long sorted = bitonic_1024(sv, sortbuf);
    if (tid % TEAM_SAMP == 0 && tid) ts.split[tid / TEAM_SAMP - 1] = sorted;
    __syncthreads();
    unsigned long long spl[TEAM - 1];
#pragma unroll
    for (int j = 0; j < TEAM - 1; j++) spl[j] = ts.split[j];
    // part of each record (key order): 2c for (s_{c-1}, s_c), 2c + 1 for {s_c}
    uint32_t ppk[(F + 3) / 4];  // parts, four per register
#pragma unroll
    for (int j = 0; j < F; j++) {
        int c = 0;
        bool eq = false;
#pragma unroll
        for (int u = 0; u < TEAM - 1; u++) {
            c += spl[u] < o[j];
            eq |= spl[u] == o[j];
        }
        const uint32_t pj = (uint32_t)(2 * c + (eq ? 1 : 0));
        if ((j & 3) == 0) ppk[j >> 2] = pj;
        else ppk[j >> 2] |= pj << (8 * (j & 3));
    }
    // multi-split pass 1: per-(part, warp) counts
    unsigned gm[F];
#pragma unroll
    for (int j = 0; j < F; j++) {
        const bool valid = base + j * 32 < mc;
        const int p = (int)((ppk[j >> 2] >> (8 * (j & 3))) & 0xFFu);
        unsigned mm = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int bit = 0; bit < TEAM_PBITS; bit++) {
            const bool v = (p >> bit) & 1;
            const unsigned bb = __ballot_sync(0xffffffffu, v);
            mm &= v ? bb : ~bb;
        }
        gm[j] = mm;
        __syncwarp();
        if (valid && lane == __ffs(mm) - 1) wcnt[p * FW + w] += (uint16_t)__popc(mm);
    }
    __syncthreads();
    // per part: exclusive scan over the warps, chunk total (warp p scans part p)
    if (w < TEAM_PARTS) {
        const uint32_t c = wcnt[w * FW + lane];
        uint32_t s_ = c;
#pragma unroll
        for (int o_ = 1; o_ < 32; o_ <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, s_, o_);
            if (lane >= o_) s_ += y;
        }
        wcnt[w * FW + lane] = (uint16_t)(s_ - c);
        if (lane == 31) ts.pcnt[w] = s_;
    }
    cl.sync();  // #2: part counts published
    if (w == 0) {  // part starts and this CTA's slots: lane p (< TEAM_PARTS) reads every chunk's count of part p
        uint32_t tot = 0, below = 0;
        if (lane < TEAM_PARTS) {
#pragma unroll
            for (int rr = 0; rr < TEAM; rr++) {
                const uint32_t v = cl.map_shared_rank(ts.pcnt, rr)[lane];
                tot += v;
                below += rr < r ? v : 0u;
            }
        }
        uint32_t s_ = tot;
#pragma unroll
        for (int o_ = 1; o_ < 32; o_ <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, s_, o_);
            if (lane >= o_) s_ += y;
        }
        if (lane < TEAM_PARTS) {
            ts.pstart[lane] = s_ - tot;
            ts.pbase[lane] = s_ - tot + below;
        }
        if (lane == TEAM_PARTS - 1) ts.pstart[TEAM_PARTS] = s_;
    }
    __syncthreads();
    mbar_wait(&bar[1], parity);  // payload staged
    parity ^= 1u;
    // multi-split pass 2: rank in record order, store to the part
    uint64_t *ok = B.out_k + e.start;
    P *op = (P *)B.out_p + e.start;
    const uint64_t l2pol = l2_evict_last_policy();
#pragma unroll
    for (int j = 0; j < F; j++) {
        const int i = base + j * 32;
        const bool valid = i < mc;
        const int p = (int)((ppk[j >> 2] >> (8 * (j & 3))) & 0xFFu);
        const unsigned mm = gm[j];
        const int leader = valid ? __ffs(mm) - 1 : lane;
        uint32_t c = 0;
        __syncwarp();
        if (valid && lane == leader) {
            c = wcnt[p * FW + w];
            wcnt[p * FW + w] = (uint16_t)(c + __popc(mm));
        }
        c = __shfl_sync(0xffffffffu, c, leader);
        if (valid) {
            const uint32_t pos = ts.pbase[p] + c + (uint32_t)__popc(mm & lt);
            ZSB_CHECK(p < TEAM_PARTS && pos < (uint32_t)m && pos >= ts.pstart[p] && pos < ts.pstart[p + 1]);
            st_keep(ok + pos, kin[i], l2pol);
            if constexpr (PB != 0) st_keep(op + pos, pin[i], l2pol);
        }
    }
    // the open parts are re-staged by TMA bulk copies (async proxy) in other CTAs
    fence_proxy_async_global();
    cl.sync();  // #3: every record is in its part (equality parts are final)
    int nfin = 0;
    {
        const int ps = (int)ts.pstart[2 * r], pc = (int)ts.pstart[2 * r + 1] - ps;
        if (pc > 0 && pc <= cap) {
            finish_entry<KK, PB>(B, Entry{e.start + ps, pc, 2}, 0, cap, refine, refine_count, fin_ins, nullptr, bar,
                                 parity);
            nfin = 1;
        }
    }
    if (tid == 0) {  // oversized open parts: the team finishes them next (same order in every CTA)
        for (int pp = TEAM - 1; pp >= 0; pp--) {
            const int ps = (int)ts.pstart[2 * pp], pc = (int)ts.pstart[2 * pp + 1] - ps;
            if (pc > cap && ts.sp < TEAM_STACK) ts.stack[ts.sp++] = Entry{e.start + ps, pc, 2};
        }
    }
    __syncthreads();
    return nfin;
}

// Persistent team kernel: clusters of TEAM CTAs take team runs by ticket
// (rank 0 draws, the peers read it through DSMEM), oversized parts first.
template <int KK, int PB>
__global__ void __launch_bounds__(FT, 1) k_team(Buffers B, const Entry *__restrict__ runs,
                                                const unsigned long long *count, int64_t cap_runs, int cap,
                                                Entry *refine, unsigned long long *refine_count, int fin_ins,
                                                unsigned long long *ticket, unsigned long long *runs_total) {
    __shared__ uint64_t bar[2];
    __shared__ TeamShared ts;
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        ts.sp = 0;
    }
    __syncthreads();
    const int64_t ne = min((int64_t)*count, cap_runs);
    uint32_t parity = 0;
    int nfin = 0;
    while (true) {
        Entry e;
        if (ts.sp > 0) {
            e = ts.stack[ts.sp - 1];
            __syncthreads();
            if (threadIdx.x == 0) ts.sp--;
        } else {
            if (cl.block_rank() == 0 && threadIdx.x == 0) ts.ticket = (long long)atomicAdd(ticket, 1ull);
            cl.sync();
            if (threadIdx.x == 0) ts.tk = *cl.map_shared_rank(&ts.ticket, 0);
            __syncthreads();
            if (ts.tk >= ne) break;
            e = runs[ts.tk];
        }
        __syncthreads();
        nfin += team_run<KK, PB>(B, e, cap, refine, refine_count, fin_ins, bar, parity, ts);
    }
    cl.sync();  // no CTA leaves while a peer may still read its shared memory
    if (threadIdx.x == 0 && nfin) atomicAdd(runs_total, (unsigned long long)nfin);
}

// Refine iterations (every CTA of a cooperative grid): finishes the refine
// runs in list A (count *count_a) into list B, then B into A, ... until a
// pass leaves none, so oversized sub-buckets of refine runs never need the
// host.  Each pass's run count is added to *runs_total (SortStats).  Lists
// and counts are swapped between passes; a pass's input count and the
// ticket are reset by block 0 between the two grid barriers.
template <int KK, int PB>
__device__ void refine_loop(const Buffers &B, Entry *list_a, unsigned long long *count_a, Entry *list_b,
                            unsigned long long *count_b, int64_t cap_list, int cap, int fin_ins,
                            unsigned long long *ticket, unsigned long long *runs_total, int prefetch, uint64_t *bar,
                            uint32_t &parity) {
    cg::grid_group grid = cg::this_grid();
    Entry *lin = list_a, *lout = list_b;
    unsigned long long *cin = count_a, *cout = count_b;
    while (true) {
        const int64_t ne = min((int64_t)*(volatile unsigned long long *)cin, cap_list);
        if (ne == 0) break;  // every CTA reads the same value (written before the last grid barrier)
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(runs_total, (unsigned long long)ne);
        finish_list<KK, PB>(B, lin, ne, cap, lout, cout, fin_ins, nullptr, ticket, prefetch, bar, parity);
        // the next pass stages this pass's generic-proxy output stores with
        // TMA bulk copies (async proxy): fence them before the grid barrier
        fence_proxy_async_global();
        grid.sync();  // pass done: its refine runs are all in lout
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            *cin = 0ull;
            *ticket = 0ull;
        }
        grid.sync();
        Entry *tl = lin;
        lin = lout;
        lout = tl;
        unsigned long long *tc = cin;
        cin = cout;
        cout = tc;
    }
}

struct RefineArgs {  // the refine iterations a finish launch runs after its own list (list_b == nullptr: none)
    const int32_t *order;  // finish order of the launch's own list (nullptr: list order)
    Entry *list_b;
    unsigned long long *count_b;
    int64_t cap_list;
    unsigned long long *ticket_b;
    unsigned long long *runs_total;
};

// Persistent finish: the work count is read from device memory (written by
// the classify or a previous finish), so the host enqueues without a sync.
// With `ra.list_b` (cooperative launch) the same grid then runs the refine
// iterations of the runs it left in `refine`: one launch per level instead
// of two.
template <int KK, int PB>
__global__ void __launch_bounds__(FT, FIN_CTAS) k_finish(Buffers B, const Entry *__restrict__ entries,
                                                  const unsigned long long *count, int64_t count_const, int cap,
                                                  Entry *refine, unsigned long long *refine_count, int fin_ins,
                                                  long long *prof, unsigned long long *ticket, int prefetch,
                                                  RefineArgs ra) {
    __shared__ uint64_t bar[2];  // run staging (TMA bulk copies) completion: keys, payload
    uint32_t parity = 0;
    const int64_t ne = count ? min((int64_t)*count, count_const) : count_const;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    __syncthreads();
    if (!ticket) {  // one run per CTA (grid = exact count)
        if ((int64_t)blockIdx.x < ne) finish_entry<KK, PB>(B, entries[blockIdx.x], blockIdx.x, cap, refine, refine_count,
                                                           fin_ins, prof, bar, parity);
    } else {
        finish_list<KK, PB>(B, entries, ne, cap, refine, refine_count, fin_ins, prof, ticket, prefetch, bar, parity,
                            ra.order);
    }
    if (ra.list_b) {
        fence_proxy_async_global();  // refine runs are re-staged by TMA (async proxy) after the barrier
        cg::this_grid().sync();  // every refine run of the list is published
        refine_loop<KK, PB>(B, refine, refine_count, ra.list_b, ra.count_b, ra.cap_list, cap, fin_ins, ra.ticket_b,
                            ra.runs_total, prefetch, bar, parity);
    }
}

// Refine pass as a launch of its own (cooperative, every CTA resident).
template <int KK, int PB>
__global__ void __launch_bounds__(FT, FIN_CTAS) k_refine(Buffers B, Entry *list_a, unsigned long long *count_a, Entry *list_b,
                                                  unsigned long long *count_b, int64_t cap_list, int cap, int fin_ins,
                                                  unsigned long long *ticket, unsigned long long *runs_total,
                                                  int prefetch) {
    __shared__ uint64_t bar[2];
    uint32_t parity = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    __syncthreads();
    refine_loop<KK, PB>(B, list_a, count_a, list_b, count_b, cap_list, cap, fin_ins, ticket, runs_total, prefetch, bar,
                        parity);
}

// Entry builder for the small-n path (one finish over the whole input).
__global__ void k_single_entry(Entry *entries, int64_t n) { entries[0] = Entry{0, (int32_t)n, 0}; }

}  // namespace zsb
