// Cost of a cooperative launch with 0/1/2 grid barriers vs a plain launch (B200).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_plain(int *x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0]++; }
template <int NS>
__global__ void k_coop(int *x) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < NS; i++) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) x[0]++;
}
int main() {
    int *x; cudaMalloc(&x, 4);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid : {2, 148}) {
        for (int mode = 0; mode < 4; mode++) {
            void *args[] = {&x};
            auto launch = [&]() {
                if (mode == 0) k_plain<<<grid, 1024, 0, s>>>(x);
                else if (mode == 1) cudaLaunchCooperativeKernel((void *)k_coop<0>, grid, 1024, args, 0, s);
                else if (mode == 2) cudaLaunchCooperativeKernel((void *)k_coop<1>, grid, 1024, args, 0, s);
                else cudaLaunchCooperativeKernel((void *)k_coop<2>, grid, 1024, args, 0, s);
            };
            for (int i = 0; i < 10; i++) launch();
            cudaStreamSynchronize(s);
            cudaEventRecord(a, s);
            for (int i = 0; i < 200; i++) launch();
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("grid %3d %-22s %.2f us per launch (back to back)\n", grid,
                   mode == 0 ? "plain" : mode == 1 ? "cooperative, 0 syncs" : mode == 2 ? "cooperative, 1 sync" : "cooperative, 2 syncs",
                   ms * 1000 / 200);
        }
    }
    return 0;
}
