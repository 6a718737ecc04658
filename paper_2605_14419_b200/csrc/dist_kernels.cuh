// dist_kernels.cuh -- device side of the multi-GPU exchange (D1/D2 inputs).
//
// The collectives themselves run through torch.distributed (NCCL) in
// paper_2605_14419_b200/dist.py; these kernels produce the per-rank inputs:
//   k_local_moments   count, sum(x - shift), sum((x - shift)^2), ordered
//                     min/max of the local shard (D1 allreduce payload);
//   k_bucket_hist     histogram of the global fitted z-score buckets (D2);
//   k_bucket_minmax   ordered min/max of keys in a few candidate buckets
//                     (all-equal test for cuts inside a bucket).
// The stable partition to destination ranks reuses K2/K3/K4 in MODE_DEST.
#pragma once

#include "sort_kernels.cuh"

namespace zsb {

__global__ void k_dist_init(double *out3, unsigned long long *bits2) {
    if (threadIdx.x < 3) out3[threadIdx.x] = 0.0;
    if (threadIdx.x == 0) {
        bits2[0] = ~0ull;
        bits2[1] = 0ull;
    }
}

template <int KK>
__global__ void __launch_bounds__(NT) k_local_moments(const uint64_t *__restrict__ keys, int64_t n, double shift,
                                                      double *out3, unsigned long long *bits2) {
    unsigned long long omin = ~0ull, omax = 0ull;
    double s1 = 0.0, s2 = 0.0, cnt = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const uint64_t b = __ldcs(keys + i);
        const unsigned long long o = ord_key<KK>(b);
        omin = min(omin, o);
        omax = max(omax, o);
        const double d = key_value<KK>(b) - shift;
        s1 += d;
        s2 += d * d;
        cnt += 1.0;
    }
    omin = warp_min_u64(omin);
    omax = warp_max_u64(omax);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    cnt = warp_sum(cnt);
    if (lane_id() == 0) {
        atomicMin(&bits2[0], omin);
        atomicMax(&bits2[1], omax);
        atomicAdd(&out3[0], cnt);
        atomicAdd(&out3[1], s1);
        atomicAdd(&out3[2], s2);
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

template <int KK>
__global__ void __launch_bounds__(NT) k_bucket_minmax(const uint64_t *__restrict__ keys, int64_t n, double center,
                                                      double sd, double zmin, double scale, int k, int nb,
                                                      const int32_t *__restrict__ buckets,
                                                      unsigned long long *omin, unsigned long long *omax) {
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const uint64_t b = __ldcs(keys + i);
        const int bk = bucket_z(key_value<KK>(b), center, sd, zmin, scale, k);
        for (int j = 0; j < nb; j++) {
            if (bk == buckets[j]) {
                const unsigned long long o = ord_key<KK>(b);
                atomicMin(&omin[j], o);
                atomicMax(&omax[j], o);
            }
        }
    }
}

// Refinement histograms for cuts inside a bucket: query q counts the local
// records with bucket == qb[q] and ordered key in [qlo[q], qhi[q]] by the
// exact digit (ord - qlo) >> qsh[q] (nbins bins per query).
template <int KK>
__global__ void __launch_bounds__(NT) k_range_hist(const uint64_t *__restrict__ keys, int64_t n, double center,
                                                   double sd, double zmin, double scale, int k, int nq,
                                                   const int32_t *__restrict__ qb, const uint64_t *__restrict__ qlo,
                                                   const uint64_t *__restrict__ qhi, const int32_t *__restrict__ qsh,
                                                   int nbins, unsigned long long *counts) {
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const uint64_t b = __ldcs(keys + i);
        const int bk = bucket_z(key_value<KK>(b), center, sd, zmin, scale, k);
        const uint64_t o = ord_key<KK>(b);
        for (int q = 0; q < nq; q++) {
            if (bk == qb[q] && o >= qlo[q] && o <= qhi[q]) {
                const uint64_t d = (o - qlo[q]) >> qsh[q];
                if (d < (uint64_t)nbins) atomicAdd(&counts[(int64_t)q * nbins + d], 1ull);
            }
        }
    }
}

__global__ void k_minmax_init(int nb, unsigned long long *omin, unsigned long long *omax) {
    if ((int)threadIdx.x < nb) {
        omin[threadIdx.x] = ~0ull;
        omax[threadIdx.x] = 0ull;
    }
}

}  // namespace zsb
