// Microbenchmark: throughput of __match_any_sync vs ballot multisplit on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ballot_match(int id, int nbits) {
    unsigned m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 10; b++) {
        const unsigned bit = ((unsigned)id >> b) & 1u;
        const unsigned v = __ballot_sync(0xffffffffu, bit);
        m &= v ^ (bit - 1u);
    }
    return m;
}
template <int MODE>
__global__ void k(const int *ids, unsigned *out, int iters, int mask) {
    int v[16];
    for (int j = 0; j < 16; j++) {
        int x = ids[(blockIdx.x * blockDim.x + threadIdx.x) * 16 + j];
        v[j] = mask >= 0 ? (x & mask) : ((x & 31) << (-mask));  // negative: 32 distinct values spread by a shift
    }
    unsigned acc = 0;
    for (int it = 0; it < iters; it++) {
        unsigned m[16];
#pragma unroll
        for (int j = 0; j < 16; j++) m[j] = MODE == 0 ? __match_any_sync(0xffffffffu, v[j]) : ballot_match(v[j], 10);
#pragma unroll
        for (int j = 0; j < 16; j++) { acc += __popc(m[j]); v[j] ^= (int)(m[j] & 0x80000000u) >> 31 & 0; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    const int T = 512, B = 148, N = T * B * 16, iters = 200;
    int *ids; unsigned *out;
    cudaMalloc(&ids, N * 4); cudaMalloc(&out, T * B * 4);
    int *h = new int[N];
    unsigned s = 12345;
    for (int i = 0; i < N; i++) { s = s * 1664525u + 1013904223u; h[i] = (int)(s >> 8); }
    cudaMemcpy(ids, h, N * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mask : {31, 63, 127, 255, 511, 1023, 2047, -5, -10, -20}) {
        for (int mode = 0; mode < 1; mode++) {
            for (int rep = 0; rep < 2; rep++) {
                cudaEventRecord(a);
                if (mode == 0) k<0><<<B, T>>>(ids, out, iters, mask); else k<1><<<B, T>>>(ids, out, iters, mask);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("mask %4d %s: %.3f ms  -> %.1f cycles/op/SMSP (1.9GHz)\n", mask, mode ? "ballot" : "match ", ms,
                       ms * 1e-3 * 1.9e9 / (iters * 16.0 * (T / 32) / 4));
            }
        }
    }
    return 0;
}
