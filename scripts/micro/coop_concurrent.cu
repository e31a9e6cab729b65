// Can two cooperative kernels (each half of the SM slots) run concurrently on
// one GPU, on two streams of one process? Each signals a flag and waits for
// the other's (bounded spin), then reports whether it saw the partner.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_pair(volatile unsigned* mine, volatile unsigned* other, unsigned* result) {
    cg::grid_group g = cg::this_grid();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *mine = 1;
        __threadfence_system();
        long long t0 = clock64();
        unsigned seen = 0;
        while (clock64() - t0 < 4000000000ll) { // ~2 s
            if (*other) { seen = 1; break; }
        }
        *result = seen;
    }
    g.sync();
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pair, 256, 0);
    unsigned *flags, *res;
    cudaMalloc(&flags, 16); cudaMalloc(&res, 16);
    cudaStream_t s0, s1;
    cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    for (int frac : {2, 4}) {
        cudaMemset(flags, 0, 16); cudaMemset(res, 0, 16);
        cudaDeviceSynchronize();
        int grid = per_sm * sms / frac;
        unsigned *f0 = flags, *f1 = flags + 1, *r0 = res, *r1 = res + 1;
        void* a0[] = {&f0, &f1, &r0};
        void* a1[] = {&f1, &f0, &r1};
        cudaError_t e0 = cudaLaunchCooperativeKernel((void*)k_pair, grid, 256, a0, 0, s0);
        cudaError_t e1 = cudaLaunchCooperativeKernel((void*)k_pair, grid, 256, a1, 0, s1);
        cudaDeviceSynchronize();
        unsigned h[2];
        cudaMemcpy(h, res, 8, cudaMemcpyDeviceToHost);
        printf("grid=%d (1/%d of %d slots): launch %s/%s, saw partner %u/%u, err=%s\n", grid, frac,
               per_sm * sms, cudaGetErrorString(e0), cudaGetErrorString(e1), h[0], h[1],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
