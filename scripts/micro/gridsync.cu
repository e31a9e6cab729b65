// Microbenchmark: cost of a grid-wide barrier in a persistent cooperative
// kernel on B200 (cooperative_groups grid.sync vs a sense-reversing barrier).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* sink) {
    cg::grid_group g = cg::this_grid();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x ^ i;
        g.sync();
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

__device__ __forceinline__ void bar(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == g0) { __nanosleep(32); }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_own(int iters, unsigned* count, unsigned* gen, unsigned* sink) {
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x ^ i;
        bar(count, gen, gridDim.x);
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *sink, *cnt, *gen;
    cudaMalloc(&sink, 4); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bps : {1, 2, 4, 8}) {
        int iters = 2000;
        dim3 grid(sms * bps), block(256);
        void* args[] = {&iters, &sink};
        cudaLaunchCooperativeKernel((void*)k_cg, grid, block, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_cg, grid, block, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        void* args2[] = {&iters, &cnt, &gen, &sink};
        cudaLaunchCooperativeKernel((void*)k_own, grid, block, args2, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_own, grid, block, args2, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        printf("blocks/SM=%d grid=%d cg.sync=%.3f us own=%.3f us err=%s\n", bps, grid.x,
               ms * 1e3 / iters, ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    // empty-kernel launch-to-launch cost in a stream, for comparison
    cudaEventRecord(a);
    for (int i = 0; i < 2000; ++i) k_cg<<<sms * 4, 256>>>(0, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("back-to-back empty launches: %.3f us each\n", ms * 1e3 / 2000);
    return 0;
}
