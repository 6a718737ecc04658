// Cluster occupancy and DSMEM/cluster-barrier probe for the team finish:
// how many clusters of T CTAs (1024 threads, ~214 KB dynamic shared memory
// each, one CTA per SM) the B200 keeps resident, and what one cluster.sync
// and a 16-byte DSMEM read cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_probe cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_probe(unsigned long long *out, int iters) {
    extern __shared__ uint4 sm[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned r = cl.block_rank();
    sm[threadIdx.x] = make_uint4(r, threadIdx.x, 0, 0);
    cl.sync();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) cl.sync();
    long long t1 = clock64();
    const uint4 *peer = cl.map_shared_rank(sm, (r + 1) % cl.num_blocks());
    unsigned acc = 0;
    long long t2 = clock64();
    for (int i = 0; i < iters; i++) acc += peer[(threadIdx.x + i) & 1023].y;
    long long t3 = clock64();
    cl.sync();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (threadIdx.x == 0) {
        out[blockIdx.x * 4 + 0] = (t1 - t0) / iters;
        out[blockIdx.x * 4 + 1] = (t3 - t2) / iters;
        out[blockIdx.x * 4 + 2] = smid;
        out[blockIdx.x * 4 + 3] = acc;
    }
}

int main() {
    const size_t smem = 214 * 1024;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    unsigned long long *d;
    cudaMalloc(&d, 4096 * 32);
    for (int T : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = T;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(T * 64);
        int ncl = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void *)k_probe, &cfg);
        printf("T=%2d max active clusters %d (%d SMs) %s\n", T, ncl, ncl * T, cudaGetErrorString(e));
        if (ncl <= 0) continue;
        cfg.gridDim = dim3(ncl * T);
        e = cudaLaunchKernelEx(&cfg, k_probe, d, 200);
        cudaError_t e2 = cudaDeviceSynchronize();
        unsigned long long h[4 * 160];
        cudaMemcpy(h, d, sizeof(unsigned long long) * 4 * ncl * T, cudaMemcpyDeviceToHost);
        printf("   launch %s/%s cluster.sync %llu cyc, DSMEM read %llu cyc; smids of cluster 0:", cudaGetErrorString(e),
               cudaGetErrorString(e2), h[0], h[1]);
        for (int i = 0; i < T; i++) printf(" %llu", h[i * 4 + 2]);
        printf("\n");
    }
    return 0;
}
