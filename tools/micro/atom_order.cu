// Does a warp's shared-memory atomicAdd hand out old values in lane order
// when several lanes hit the same address?  Counts violations over many
// random collision patterns (u16 halves of 32-bit words, as in k_scatter).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const unsigned *rnd, unsigned long long *viol, unsigned long long *groups, int iters, int nb) {
    __shared__ unsigned cnt[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long v = 0, g = 0;
    for (int it = 0; it < iters; it++) {
        const unsigned r = rnd[(blockIdx.x * 64 + it) * blockDim.x + threadIdx.x];
        const int b = r % nb;                 // bucket
        const int q = w * 1024 + b;           // per-(warp, bucket) u16 counter
        const unsigned sh = 16 * (q & 1);
        const unsigned old = (atomicAdd(&cnt[(q >> 1) & 2047], 1u << sh) >> sh) & 0xFFFFu;
        const unsigned m = __match_any_sync(0xffffffffu, b);
        // lanes of my group below me must have smaller old values
        for (int l = 0; l < 32; l++) {
            const unsigned o2 = __shfl_sync(0xffffffffu, old, l);
            if (((m >> l) & 1u) && l < lane && o2 > old) v++;
        }
        if ((m & ((1u << lane) - 1)) == 0 && __popc(m) > 1) g++;
    }
    atomicAdd(viol, v);
    atomicAdd(groups, g);
}
int main() {
    const int B = 148, T = 512, iters = 64;
    size_t N = (size_t)B * 64 * T;
    unsigned *h = new unsigned[N];
    unsigned s = 7;
    for (size_t i = 0; i < N; i++) { s = s * 1664525u + 1013904223u; h[i] = s >> 4; }
    unsigned *d; unsigned long long *dv, *dg;
    cudaMalloc(&d, N * 4); cudaMalloc(&dv, 8); cudaMalloc(&dg, 8);
    cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
    for (int nb : {2, 8, 64, 1024}) {
        cudaMemset(dv, 0, 8); cudaMemset(dg, 0, 8);
        k<<<B, T>>>(d, dv, dg, iters, nb);
        unsigned long long v, g; cudaMemcpy(&v, dv, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&g, dg, 8, cudaMemcpyDeviceToHost);
        printf("buckets %5d: tie groups %llu, lane-order violations %llu\n", nb, g, v);
    }
    return 0;
}
