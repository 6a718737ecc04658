// Shared-memory atomic throughput on B200: cycles per warp-instruction of
// atomicAdd to random addresses among K counters (32-bit and packed 16-bit),
// versus plain LDS+STS, with 1024 threads per CTA, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(int iters, int kmask, unsigned long long *out, uint32_t *sink) {
    __shared__ uint32_t h[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint32_t r = threadIdx.x * 0x9E3779B9u + blockIdx.x * 7919u + 1;
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            r = r * 1664525u + 1013904223u;
            const uint32_t b = (r >> 8) & kmask;
            if (MODE == 0) atomicAdd(&h[b], 1u);                          // ATOMS 32-bit, result unused
            else if (MODE == 1) acc += atomicAdd(&h[b], 1u);             // ATOMS with result
            else if (MODE == 2) atomicAdd(&h[b >> 1], 1u << (16 * (b & 1)));  // packed u16 pair
            else if (MODE == 3) acc += h[b];                              // LDS only
            else if (MODE == 4) h[b] = r;                                 // STS only
            else if (MODE == 5) acc += __popc(__match_any_sync(0xffffffffu, b));  // MATCH.ANY
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    if (acc == 0x12345678u) sink[0] = h[0];
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *d;
    uint32_t *sink;
    cudaMalloc(&d, sms * 8);
    cudaMalloc(&sink, 64);
    const int iters = 256;
    const char *names[] = {"ATOMS (no ret)", "ATOMS (ret)", "ATOMS packed u16", "LDS", "STS", "MATCH.ANY"};
    for (int mode = 0; mode < 6; mode++)
        for (int km : {1023, 4095}) {
            unsigned long long h[256];
            for (int rep = 0; rep < 2; rep++) {
                switch (mode) {
                    case 0: k<0><<<sms, 1024>>>(iters, km, d, sink); break;
                    case 1: k<1><<<sms, 1024>>>(iters, km, d, sink); break;
                    case 2: k<2><<<sms, 1024>>>(iters, km, d, sink); break;
                    case 3: k<3><<<sms, 1024>>>(iters, km, d, sink); break;
                    case 4: k<4><<<sms, 1024>>>(iters, km, d, sink); break;
                    case 5: k<5><<<sms, 1024>>>(iters, km, d, sink); break;
                }
                cudaDeviceSynchronize();
            }
            cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < sms; i++) avg += h[i];
            avg /= sms;
            const double warp_instr = 32.0 * iters * 8;  // per SM: 32 warps x iters x 8
            printf("%-18s K=%4d: %.2f cycles per warp-instruction per SM (%.3f per lane)\n", names[mode], km + 1,
                   avg / warp_instr, avg / warp_instr / 32);
        }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
