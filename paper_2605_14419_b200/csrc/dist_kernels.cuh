// dist_kernels.cuh -- device side of the multi-GPU exchange (D1/D2 inputs).
//
// The collectives themselves run through torch.distributed (NCCL) in
// paper_2605_14419_b200/dist.py; these kernels produce the per-rank inputs:
//   k_local_moments   count, sum(x - c), sum((x - c)^2) around the shard's
//                     first key, ordered min/max (D1 all_gather payload, one pass);
//   k_bucket_hist     histogram of the global fitted z-score buckets (D2);
//   k_bucket_minmax   ordered min/max of keys in a few candidate buckets
//                     (all-equal test for cuts inside a bucket);
//   k_range_hist      digit histograms refining a cut inside a bucket;
//   k_occ_count/find  index of the t-th occurrence of a key (cut by position).
// The stable partition to destination ranks reuses K2/K3/K4 in MODE_DEST.
#pragma once

#include "sort_kernels.cuh"

namespace zsb {

__global__ void k_dist_init(double *out4, unsigned long long *bits2) {
    if (threadIdx.x < 4) out4[threadIdx.x] = 0.0;
    if (threadIdx.x == 0) {
        bits2[0] = ~0ull;
        bits2[1] = 0ull;
    }
}

// One pass over the shard: count, sum(x - c), sum((x - c)^2) with c = shift,
// or (self_shift) c = the shard's first key, plus the ordered extremes.  The
// ranks combine these exactly once (all_gather + Chan's merge, dist.py), so
// no second pass around a common shift is needed.  One set of atomics per
// CTA (block reduction in shared memory).
template <int KK>
__global__ void __launch_bounds__(NT) k_local_moments(const uint64_t *__restrict__ keys, int64_t n, double shift,
                                                      int self_shift, double *out4, unsigned long long *bits2) {
    __shared__ double ws1[NT / 32], ws2[NT / 32], wc[NT / 32];
    __shared__ unsigned long long wmn[NT / 32], wmx[NT / 32];
    const double c = self_shift ? key_value<KK>(keys[0]) : shift;
    unsigned long long omin = ~0ull, omax = 0ull;
    double s1 = 0.0, s2 = 0.0, cnt = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const uint64_t b = __ldcs(keys + i);
        const unsigned long long o = ord_key<KK>(b);
        omin = min(omin, o);
        omax = max(omax, o);
        const double d = key_value<KK>(b) - c;
        s1 += d;
        s2 += d * d;
        cnt += 1.0;
    }
    const int w = threadIdx.x >> 5, lane = lane_id();
    omin = warp_min_u64(omin);
    omax = warp_max_u64(omax);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    cnt = warp_sum(cnt);
    if (lane == 0) {
        ws1[w] = s1;
        ws2[w] = s2;
        wc[w] = cnt;
        wmn[w] = omin;
        wmx[w] = omax;
    }
    __syncthreads();
    if (w == 0) {
        constexpr int NW = NT / 32;
        omin = warp_min_u64(lane < NW ? wmn[lane] : ~0ull);
        omax = warp_max_u64(lane < NW ? wmx[lane] : 0ull);
        s1 = warp_sum(lane < NW ? ws1[lane] : 0.0);
        s2 = warp_sum(lane < NW ? ws2[lane] : 0.0);
        cnt = warp_sum(lane < NW ? wc[lane] : 0.0);
        if (lane == 0 && cnt > 0.0) {
            atomicMin(&bits2[0], omin);
            atomicMax(&bits2[1], omax);
            atomicAdd(&out4[0], cnt);
            atomicAdd(&out4[1], s1);
            atomicAdd(&out4[2], s2);
        }
        if (lane == 0 && blockIdx.x == 0) out4[3] = c;
    }
}

template <int KK>
__global__ void __launch_bounds__(NT) k_bucket_hist(const uint64_t *__restrict__ keys, int64_t n, double center,
                                                    double sd, double zmin, double scale, int k,
                                                    unsigned long long *counts) {
    extern __shared__ uint32_t h[];
    for (int b = threadIdx.x; b < k; b += NT) h[b] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
        atomicAdd(&h[bucket_z(key_value<KK>(__ldcs(keys + i)), center, sd, zmin, scale, k)], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < k; b += NT)
        if (h[b]) atomicAdd(&counts[b], (unsigned long long)h[b]);
}

// Ordered min/max of the keys of nb (<= 32) candidate buckets: shared
// atomics per record, one global atomic per CTA and candidate.
template <int KK>
__global__ void __launch_bounds__(NT) k_bucket_minmax(const uint64_t *__restrict__ keys, int64_t n, double center,
                                                      double sd, double zmin, double scale, int k, int nb,
                                                      const int32_t *__restrict__ buckets,
                                                      unsigned long long *omin, unsigned long long *omax) {
    __shared__ unsigned long long smn[32], smx[32];
    __shared__ int32_t sb[32];
    if (threadIdx.x < 32) {
        smn[threadIdx.x] = ~0ull;
        smx[threadIdx.x] = 0ull;
        sb[threadIdx.x] = (int)threadIdx.x < nb ? buckets[threadIdx.x] : -1;
    }
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const uint64_t b = __ldcs(keys + i);
        const int bk = bucket_z(key_value<KK>(b), center, sd, zmin, scale, k);
        for (int j = 0; j < nb; j++) {
            if (bk == sb[j]) {
                const unsigned long long o = ord_key<KK>(b);
                atomicMin(&smn[j], o);
                atomicMax(&smx[j], o);
            }
        }
    }
    __syncthreads();
    if ((int)threadIdx.x < nb && smx[threadIdx.x] >= smn[threadIdx.x]) {
        atomicMin(&omin[threadIdx.x], smn[threadIdx.x]);
        atomicMax(&omax[threadIdx.x], smx[threadIdx.x]);
    }
}

// Refinement histograms for cuts inside a bucket: query q counts the local
// records with bucket == qb[q] and ordered key in [qlo[q], qhi[q]] by the
// exact digit (ord - qlo) >> qsh[q] (nbins bins per query).  With `smem`
// the nq * nbins counters live in shared memory (one global add per CTA
// and nonzero bin), else in global memory.
template <int KK>
__global__ void __launch_bounds__(NT) k_range_hist(const uint64_t *__restrict__ keys, int64_t n, double center,
                                                   double sd, double zmin, double scale, int k, int nq,
                                                   const int32_t *__restrict__ qb, const uint64_t *__restrict__ qlo,
                                                   const uint64_t *__restrict__ qhi, const int32_t *__restrict__ qsh,
                                                   int nbins, unsigned long long *counts, int smem) {
    extern __shared__ uint32_t rh[];
    const int tot = nq * nbins;
    if (smem) {
        for (int q = threadIdx.x; q < tot; q += NT) rh[q] = 0;
        __syncthreads();
    }
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const uint64_t b = __ldcs(keys + i);
        const int bk = bucket_z(key_value<KK>(b), center, sd, zmin, scale, k);
        const uint64_t o = ord_key<KK>(b);
        for (int q = 0; q < nq; q++) {
            if (bk == qb[q] && o >= qlo[q] && o <= qhi[q]) {
                const uint64_t d = (o - qlo[q]) >> qsh[q];
                if (d < (uint64_t)nbins) {
                    if (smem) atomicAdd(&rh[q * nbins + (int)d], 1u);
                    else atomicAdd(&counts[(int64_t)q * nbins + d], 1ull);
                }
            }
        }
    }
    if (smem) {
        __syncthreads();
        for (int q = threadIdx.x; q < tot; q += NT)
            if (rh[q]) atomicAdd(&counts[q], (unsigned long long)rh[q]);
    }
}

__global__ void k_minmax_init(int nb, unsigned long long *omin, unsigned long long *omax) {
    if ((int)threadIdx.x < nb) {
        omin[threadIdx.x] = ~0ull;
        omax[threadIdx.x] = 0ull;
    }
}

// Occurrence search (the record that a cut inside a one-valued run falls
// on): local index of the t-th record whose ordered key equals `target`
// (-0.0 and +0.0 share one image).  Pass 1: per-chunk match counts; pass 2
// (one CTA): the chunk holding the t-th match, then that chunk in order
// (ballots per warp, warp prefix).  *out = index or -1.
constexpr int OCC_T = 1024;
template <int KK>
__global__ void __launch_bounds__(NT) k_occ_count(const uint64_t *__restrict__ keys, int64_t n, int64_t chunk,
                                                  uint64_t target, unsigned long long *cnt) {
    __shared__ unsigned long long ws[NT / 32];
    const int64_t c0 = (int64_t)blockIdx.x * chunk, c1 = min(n, c0 + chunk);
    unsigned long long c = 0;
    for (int64_t i = c0 + threadIdx.x; i < c1; i += NT) c += ord_key<KK>(__ldcs(keys + i)) == target;
    c = warp_sum(c);
    if (lane_id() == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < NT / 32; w++) t += ws[w];
        cnt[blockIdx.x] = t;
    }
}

template <int KK>
__global__ void __launch_bounds__(OCC_T) k_occ_find(const uint64_t *__restrict__ keys, int64_t n, int64_t chunk,
                                                    int nchunks, uint64_t target, int64_t t,
                                                    const unsigned long long *cnt, long long *out) {
    __shared__ long long s_chunk, s_before;
    __shared__ uint32_t wc[OCC_T / 32];
    __shared__ long long s_found;
    if (threadIdx.x == 0) {
        long long before = 0, ch = -1;
        for (int b = 0; b < nchunks; b++) {
            if (t < before + (long long)cnt[b]) {
                ch = b;
                break;
            }
            before += (long long)cnt[b];
        }
        s_chunk = ch;
        s_before = before;
        s_found = -1;
    }
    __syncthreads();
    if (s_chunk < 0) {
        if (threadIdx.x == 0) *out = -1;
        return;
    }
    const int w = threadIdx.x >> 5, lane = lane_id();
    const int64_t c0 = s_chunk * chunk, c1 = min(n, c0 + chunk);
    long long seen = s_before;
    for (int64_t base = c0; base < c1; base += OCC_T) {  // uniform trip count
        const int64_t i = base + threadIdx.x;
        const bool m = i < c1 && ord_key<KK>(keys[i]) == target;
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        if (lane == 0) wc[w] = (uint32_t)__popc(bal);
        __syncthreads();
        long long pre = seen;
        for (int q = 0; q < w; q++) pre += wc[q];
        if (m && pre + __popc(bal & lanemask_lt()) == t) s_found = i;
        long long tot = 0;
        for (int q = 0; q < OCC_T / 32; q++) tot += wc[q];
        __syncthreads();
        seen += tot;
        if (s_found >= 0 || seen > t) break;
    }
    __syncthreads();
    if (threadIdx.x == 0) *out = s_found;
}

}  // namespace zsb
