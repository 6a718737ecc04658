// gen_kernels.cuh -- counter-based workload generator for the reference's
// key families (datagen.py:92-162 shapes), on the device.
//
// The reference draws its families sequentially from one MT19937-64 stream
// (_mt19937.py:24-48), which cannot be split across threads or GPUs.  Here
// key i is a pure function of (family, seed, i, params) through splitmix64
// of the global index, so every CTA, every GPU shard and any checker can
// produce any key independently:
//   0 uniform         the raw 64-bit word as int64 (full int64 range);
//   1 normal          rint(mu + sigma * z), z = Box-Muller radius(u1) * cos(2 pi u2),
//                     clipped to int64 (reference: both Box-Muller outputs of a pair);
//   2 skewed          floor(xm * u^(-1/alpha)), u in (0, 1] (Pareto);
//   3 nearly_sorted   an increasing sequence over the int64 range (position j:
//                     INT64_MIN + j * stride + jitter_j, jitter_j < stride), where a
//                     fraction 2 * swap_fraction of the positions take the key of a
//                     uniformly random position (reference: swap_fraction * n index
//                     swaps of a sorted uniform draw -- same shape, a sorted run with
//                     scattered out-of-place keys; here displaced keys repeat);
//   4 high_duplicate  raw % dup_range.
// Uniform draws follow the reference's conventions: (0, 1] = ((r >> 11) + 1) * 2^-53,
// [0, 1) = (r >> 11) * 2^-53 (datagen.py:92-99).
#pragma once

#include "sort_kernels.cuh"

namespace zsb {

enum GenFamily { GEN_UNIFORM = 0, GEN_NORMAL = 1, GEN_SKEWED = 2, GEN_NEARLY_SORTED = 3, GEN_HIGH_DUP = 4 };

struct GenParams {
    double normal_mu, normal_sigma, pareto_alpha, pareto_xm, swap_fraction;
    uint64_t dup_range;
};

__host__ __device__ __forceinline__ uint64_t splitmix64_u(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int64_t clip_i64(double x) {
    if (!(x > -9.2233720368547758e18)) return INT64_MIN;  // also NaN
    if (x >= 9.2233720368547758e18) return INT64_MAX;
    return (int64_t)x;
}

// Stream s of the family's seed at global index g.
__device__ __forceinline__ uint64_t gen_word(uint64_t base, int s, uint64_t g) {
    return splitmix64_u(base + ((uint64_t)s << 58) + g);
}

__device__ __forceinline__ int64_t nearly_sorted_key(uint64_t base, uint64_t j, uint64_t stride) {
    return (int64_t)(0x8000000000000000ull + j * stride + gen_word(base, 3, j) % stride);
}

__global__ void __launch_bounds__(NT) k_generate(int family, uint64_t base, int64_t offset, int64_t n,
                                                 int64_t n_total, GenParams gp, int64_t *out) {
    constexpr double TWO_M53 = 1.1102230246251565e-16;  // 2^-53
    const uint64_t stride = n_total > 0 ? ~0ull / (uint64_t)n_total : 1ull;
    const double inv_alpha = 1.0 / gp.pareto_alpha;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        const uint64_t g = (uint64_t)(offset + i);
        const uint64_t r0 = gen_word(base, 0, g);
        int64_t key;
        switch (family) {
            case GEN_UNIFORM: key = (int64_t)r0; break;
            case GEN_NORMAL: {
                const double u1 = (double)((r0 >> 11) + 1) * TWO_M53;
                const double u2 = (double)(gen_word(base, 1, g) >> 11) * TWO_M53;
                const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
                key = clip_i64(rint(gp.normal_mu + gp.normal_sigma * z));
                break;
            }
            case GEN_SKEWED: {
                const double u = (double)((r0 >> 11) + 1) * TWO_M53;
                key = clip_i64(floor(gp.pareto_xm * pow(u, -inv_alpha)));
                break;
            }
            case GEN_NEARLY_SORTED: {
                const double u = (double)(gen_word(base, 2, g) >> 11) * TWO_M53;
                uint64_t j = g;
                if (u < 2.0 * gp.swap_fraction) j = gen_word(base, 4, g) % (uint64_t)n_total;
                key = nearly_sorted_key(base, j, stride);
                break;
            }
            default: key = (int64_t)(r0 % (gp.dup_range ? gp.dup_range : 1ull)); break;
        }
        out[i] = key;
    }
}

}  // namespace zsb
