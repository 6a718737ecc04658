// common.cuh -- shared device helpers for the B200 zSort kernels.
//
// Keys are moved as raw 8-byte words (int64 or float64 bit patterns); every
// comparison goes through an order-preserving uint64 image (ord_key) and
// every z-score evaluation through the key's fp64 value (key_value), so the
// output keys are bit-identical to the input words.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace zsb {

// Bounds-check build (-DZSB_CHECKS; tools/bounds_check.py): every shared and
// global index of the data path is range-checked and violations are counted
// in zsb_check_count (read by zsb_check_violations()).  compute-sanitizer is
// not available on this GPU pool; this is its stand-in.  Empty otherwise.
#ifdef ZSB_CHECKS
__device__ unsigned long long zsb_check_count;
#define ZSB_CHECK(cond)                                         \
    do {                                                        \
        if (!(cond)) atomicAdd(&::zsb::zsb_check_count, 1ull); \
    } while (0)
#else
#define ZSB_CHECK(cond) \
    do {                \
    } while (0)
#endif

constexpr uint64_t SIGN = 0x8000000000000000ull;
constexpr uint64_t ORD_PINF = 0xFFF0000000000000ull;  // ord_key<KEY_F64>(+inf); positive NaNs order above
constexpr uint64_t ORD_NINF = 0x000FFFFFFFFFFFFFull;  // ord_key<KEY_F64>(-inf); negative NaNs order below
constexpr int WARP = 32;

enum KeyKind { KEY_I64 = 0, KEY_F64 = 1 };

// Partition mapping mode of one segment.
enum SegMode : int32_t {
    MODE_ZSCORE = 0,   // Eq. 1 z-score bucket (fp64, IEEE-exact intrinsics)
    MODE_INTEGER = 1,  // exact MSD digit of (ord(key) - ord(min)): termination fallback (K7)
    MODE_COPY = 2,     // all keys equal: copy through (core.py:377-380, _kernels.py:339-343)
    MODE_DEST = 3,     // multi-GPU exchange: bucket = destination rank from the global cuts
    MODE_ZCDF = 4,     // level 1, fitted: z-score coordinate through the piecewise-linear empirical CDF
                       // (histogram equalisation over kf coarse z-bins) -> equal-population buckets
    MODE_ZLIN = 5,     // recursion levels, fitted: Eq. 1's line in fp32, fmaf((float)(x - center), za, zb)
                       // (monotone; no fp64 division per key)
};

// Global cuts of the multi-GPU exchange (paper_2605_14419_b200/dist.py).
// A record (key x, global index g) goes to the number of cuts c_j with
// (bucket(x), ord(x), g) >= (bucket_j, ord_j, gidx_j) lexicographically;
// bucket(x) is the global fitted z-score bucket, monotone in x, so this
// order is the global stable order (key, original index).
constexpr int MAX_CUTS = 15;
struct DestCuts {
    double center, std, zmin, scale;
    int32_t k;
    int32_t ncuts;
    int64_t gidx_base;
    int32_t bucket[MAX_CUTS];
    int32_t pad;
    uint64_t ord[MAX_CUTS];
    int64_t gidx[MAX_CUTS];
};

// Fused exchange (dist.py, exchange="p2p"): the MODE_DEST scatter writes a
// record of destination rank d straight into d's receive buffer (a CUDA IPC
// peer pointer: NVLink stores on a multi-GPU node) at position
// dst + delta[d], dst being its position in the local partitioned layout.
constexpr int MAX_PEERS = MAX_CUTS + 1;
struct PeerDest {
    uint64_t k[MAX_PEERS];   // destination key buffers (device addresses, peers' via IPC)
    uint64_t p[MAX_PEERS];   // destination payload buffers
    int64_t delta[MAX_PEERS];  // this rank's chunk offset in destination d minus d's local start
};

// Per-segment partition parameters (one partition problem of the batch).
// Level 1 is a batch of one segment covering the whole input.
struct SegParams {
    double center;     // mean (level 1) or estimated center (recursion), core.py:226 / _kernels.py:103-106
    double std;        // sqrt(mean squared deviation around center)
    double zmin;       // z-offset of the segment minimum
    double scale;      // buckets per z unit
    uint64_t umin;     // ordered image of the segment minimum (integer mode)
    int64_t start;     // first position of the segment in the array
    int64_t len;       // records in the segment
    int64_t tile_first;// first tile (CTA) of this segment in the batch
    int64_t mat_base;  // first entry of this segment's bucket-major count matrix
    int64_t scan_base; // sum of len over the preceding segments of the batch
    int64_t tile_len;  // records per tile (last tile may be shorter)
    int32_t k;         // buckets
    int32_t ntiles;    // tiles
    int32_t mode;      // SegMode
    int32_t level;     // partition depth (1 = first level)
    int32_t shift;     // integer mode: digit = (ord - umin) >> shift
    int32_t src;       // buffer holding the segment: 0 = input, 1 = tmp, 2 = out
    int32_t kf;        // MODE_ZCDF: coarse z-bins of the CDF table (scale is the coarse scale)
    int32_t win;       // finish window width of the segment's buckets (0: the level default)
    float za, zb;      // MODE_ZCDF: coarse coordinate = fmaf((float)(x - center), za, zb)
};

// Per-segment accumulator for the recursion moments pass (fused_stats_pass,
// _kernels.py:74-88): ordered min/max and sum of squared deviations.
struct SegAcc {
    unsigned long long omin;
    unsigned long long omax;
    double s2;
    double pad;
};

// Finish work item: a contiguous run of whole buckets, <= capacity records.
struct Entry {
    int64_t start;
    int32_t len;
    int32_t src;  // 1 = tmp, 2 = out, 0 = input
};

// Control block slots (uint64).
enum Ctrl {
    C_MOM_TICKET = 0,
    C_SCAN_TICKET = 1,
    C_NCHILD = 2,
    C_NENTRY = 3,
    C_TILES_NEXT = 4,
    C_MAT_NEXT = 5,
    C_ST_FALLBACKS = 6,
    C_ST_SCATTERS = 7,
    C_ST_MAXDEPTH = 8,
    C_STATUS = 9,
    C_ST_INSERTION = 10,
    C_KMAX_NEXT = 11,
    C_NEXT_BIG = 12,
    C_WIN_NEXT = 13,
    C_NREF0 = 14,
    C_NREF1 = 15,
    C_FTICK0 = 16,  // finish work tickets (dynamic scheduling), one per launch in a pair
    C_FTICK1 = 17,
    C_SAMP_TICKET = 18,  // sampled level-1 kernels
    C_SAMPLE_OK = 19,    // 1: level 1 mapped from the sample (exact K1 skipped)
    C_NREF2 = 20,        // refine lists of odd levels (C_NREF0/1: even levels)
    C_NREF3 = 21,
    C_FTICK2 = 22,
    C_FTICK3 = 23,
    C_NTEAM = 24,        // team runs of the level (cap < len <= TEAM * cap)
    C_TTICK = 25,        // team run ticket
    C_NEED_STATS = 26,   // some child of the level needs the moments pass (k_seg_moments) before its mapping
    C_REC_NEXT = 27,     // records of the level's children (the next level's histogram and scatter pass over them)
    C_SLOTS = 28
};

#ifndef ZSB_EXP_CHEAPMAP
#define ZSB_EXP_CHEAPMAP 0
#endif

// ------------------------------------------------------------ key traits

template <int KK>
__device__ __forceinline__ uint64_t ord_key(uint64_t b) {
    if constexpr (KK == KEY_I64) {
        return b ^ SIGN;
    } else {
        if (b == SIGN) b = 0;  // -0.0 == +0.0
        return (b & SIGN) ? ~b : (b | SIGN);
    }
}

template <int KK>
__device__ __forceinline__ double key_value(uint64_t b) {
    if constexpr (KK == KEY_I64) {
        return __ll2double_rn((long long)b);  // numba int64 -> float64 (round to nearest)
    } else {
        return __longlong_as_double((long long)b);
    }
}

template <int KK>
__device__ __forceinline__ uint64_t key_from_ord(uint64_t o) {
    if constexpr (KK == KEY_I64) {
        return o ^ SIGN;
    } else {
        return (o & SIGN) ? (o ^ SIGN) : ~o;
    }
}

// Eq. 1 (_kernels.py:91-100) with explicit round-to-nearest intrinsics so
// nvcc cannot contract or reassociate: identical to the reference's
// sequential IEEE evaluation.
__device__ __forceinline__ int32_t bucket_z(double x, double center, double std, double zmin, double scale,
                                            int32_t k) {
    double h = __dmul_rn(__dadd_rn(__ddiv_rn(__dsub_rn(x, center), std), zmin), scale);
    double f = floor(h);
    if (!(f > 0.0)) return 0;
    if (f >= (double)k) return k - 1;
    return (int32_t)f;
}

template <int KK>
__device__ __forceinline__ int32_t dest_of(uint64_t bits, int64_t pos, const DestCuts *c) {
    const int32_t b = bucket_z(key_value<KK>(bits), c->center, c->std, c->zmin, c->scale, c->k);
    const uint64_t o = ord_key<KK>(bits);
    const int64_t g = c->gidx_base + pos;
    int32_t d = 0;
    for (int j = 0; j < c->ncuts; j++) {
        const bool ge = b > c->bucket[j] ||
                        (b == c->bucket[j] && (o > c->ord[j] || (o == c->ord[j] && g >= c->gidx[j])));
        d += ge;
    }
    return d;
}

// Coefficients of the level-1 coarse coordinate h = ((x - center)/std + zmin)
// * scale_f, evaluated as fmaf((float)(x - center), za, zb): one fp64
// subtraction, a conversion and one fp32 FMA.  Every step is a rounded
// monotone map (za > 0), so h is non-decreasing in the key, which is all the
// equalised partition needs (the final order never depends on bucket ids,
// only on their monotonicity).  Returns false if the pair is unusable
// (degenerate std), in which case the level keeps the exact Eq. 1 mapping.
__device__ __forceinline__ bool zc_coeffs(const SegParams &p, int kf, float &za, float &zb) {
    const double sf = p.scale * ((double)kf / (double)p.k);
    za = (float)(sf / p.std);
    zb = (float)(p.zmin * sf);
    return za > 0.0f && za < 3.0e38f && fabsf(zb) < 3.0e38f;
}

__device__ __forceinline__ float zc_coord(double x, double center, float za, float zb) {
    return fmaf((float)__dsub_rn(x, center), za, zb);
}

__device__ __forceinline__ int zc_bin(float h, int kf) {
    const float f = floorf(h);
    return !(f > 0.0f) ? 0 : (f >= (float)kf ? kf - 1 : (int)f);
}

// Histogram-equalised bucket: within coarse bin s the bucket interpolates the
// empirical CDF linearly between knots kn[s] = (cdf[s], cdf[s+1]) (bucket
// units, cdf[0] = 0, cdf[kf] = k).  Clamping each bin to [floor(cdf[s]),
// floor(cdf[s+1])] keeps the map monotone in the key under any rounding.
__device__ __forceinline__ int32_t bucket_cdf(double x, const SegParams &p, const float2 *kn) {
    // h clamped into [0, kf): below 0 -> bin 0 at fr 0, at or above kf -> the
    // last bin at fr just below 1 (its keys keep their order: fr stays
    // monotone); NaN (rejected by K2's screen) lands in bin 0
    const float hmax = __int_as_float(__float_as_int((float)p.kf) - 1);  // largest float below kf
    const float hc = fminf(fmaxf(zc_coord(x, p.center, p.za, p.zb), 0.0f), hmax);
    const int s = (int)hc;
    const float fr = hc - (float)s;
    const float2 az = kn[s];
    // floor(a + fr*(z - a)) >= floor(a) always; the clamp at floor(z) keeps
    // rounding from stepping past the next bin's first bucket
    const float b = fminf(floorf(fmaf(fr, az.y - az.x, az.x)), floorf(az.y));
    const int bi = (int)b;
    return bi < p.k ? bi : p.k - 1;
}

// BM = 1: the caller guarantees MODE_ZCDF, BM = 3: MODE_ZSCORE (the kernels
// dispatch on the segment's mode once per CTA, so the hot loop carries one
// mapping, not five).
template <int KK, int BM = 0>
__device__ __forceinline__ int32_t seg_bucket(uint64_t bits, const SegParams &p, int64_t pos = 0,
                                              const DestCuts *cuts = nullptr, const float2 *cdf = nullptr) {
    auto zlin = [&]() -> int32_t {
        const float f = floorf(zc_coord(key_value<KK>(bits), p.center, p.za, p.zb));
        return !(f > 0.0f) ? 0 : (f >= (float)p.k ? p.k - 1 : (int32_t)f);
    };
#if ZSB_EXP_CHEAPMAP  // what-if (wrong output): a conversion-free bucket map, to time the mapping's share
    if constexpr (BM == 1 || BM == 4) return (int32_t)((bits >> 20) & (uint64_t)(p.k - 1));
#endif
    if constexpr (BM == 1) {
        return bucket_cdf(key_value<KK>(bits), p, cdf);
    } else if constexpr (BM == 3) {
        return bucket_z(key_value<KK>(bits), p.center, p.std, p.zmin, p.scale, p.k);
    } else if constexpr (BM == 4) {
        return zlin();
    } else if constexpr (BM == 5) {
        return dest_of<KK>(bits, pos, cuts);
    } else {
        if (p.mode == MODE_ZCDF) return bucket_cdf(key_value<KK>(bits), p, cdf);
        if (p.mode == MODE_ZLIN) return zlin();
        if (p.mode == MODE_ZSCORE) return bucket_z(key_value<KK>(bits), p.center, p.std, p.zmin, p.scale, p.k);
        if (p.mode == MODE_INTEGER) return (int32_t)((ord_key<KK>(bits) - p.umin) >> p.shift);
        if (p.mode == MODE_DEST) return dest_of<KK>(bits, pos, cuts);
        return 0;
    }
}

// ---------------------------------------------------------- warp helpers

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// 64-bit warp min/max from two 32-bit REDUX reductions (high words, then the
// low words of the lanes holding the extreme high word); full warp only
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32);
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? (unsigned)v : 0xffffffffu);
    return ((unsigned long long)mh << 32) | ml;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? (unsigned)v : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

// Sum of the 32-bit warp totals of the warps before warp w (one REDUX).
__device__ __forceinline__ uint32_t warps_before(const uint32_t *wsum, int w, int lane) {
    return __reduce_add_sync(0xffffffffu, lane < w ? wsum[lane] : 0u);
}

// Named barriers 1..15 (0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------ TMA bulk copy + mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Order earlier generic-proxy shared-memory accesses before async-proxy (TMA) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Order this thread's earlier generic-proxy global stores before later
// async-proxy (TMA bulk copy) reads of the same data by any thread that
// synchronises with it afterwards (PTX memory model, proxy fences).
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// One TMA bulk copy global -> shared (16-byte aligned addresses, size a multiple of 16).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// L2 prefetch of a 16-byte-aligned range (size a multiple of 16) by the copy
// engine: no registers, no shared memory, no completion to wait for.
__device__ __forceinline__ void prefetch_l2_bulk(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// Stores with an L2 evict_last policy (the scatter's runs: its output is the
// finish's input, and keeping it in L2 saves both DRAM write-back and the
// finish's re-read; measured 10 us on C2).
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_keep(uint64_t *p, uint64_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;\n" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(uint32_t *p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;\n" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

template <int PB>
struct PayloadT {
    using T = uint32_t;
};
template <>
struct PayloadT<8> {
    using T = uint64_t;
};

__device__ __forceinline__ int bitlen64(uint64_t x) { return x ? 64 - __clzll((long long)x) : 0; }

}  // namespace zsb
