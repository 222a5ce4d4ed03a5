// Cost of one cooperative grid barrier with one 512-thread CTA per SM (the Taylor kernel's
// launch shape).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gsp tools/gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *sink = iters;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    for (int blocks : {148, 128, 96, 64, 32, 16}) {
        if (blocks > sms) continue;
        int iters = 1000;
        void* args[] = {&iters, &d};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)k, blocks, 512, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k, blocks, 512, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("blocks=%d grid.sync %.3f us\n", blocks, ms * 1000.0 / iters);
    }
    return 0;
}
