// Microbenchmark: random 8-byte gathers from arrays of growing size on B200
// (L2-resident -> HBM-resident), U independent loads in flight per thread.
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

template <int U>
__global__ void k_gather(const long long* __restrict__ a, uint64_t n, uint64_t loads, long long* sink) {
    long long acc = 0;
    const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x, nth = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = tid * U; i < loads; i += nth * U) {
        long long v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(&a[mix(i + u) % n]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 42) *sink = acc;
}

int main(int argc, char** argv) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *a, *sink;
    const uint64_t maxn = (8ull << 30) / 8; // 8 GB
    if (cudaMalloc(&a, maxn * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&sink, 8);
    cudaMemset(a, 1, maxn * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const uint64_t loads = 1ull << 28;
    // sizes in MB from the command line (default: L2-resident to HBM-resident)
    uint64_t sizes[32] = {8, 64, 256, 1024, 2048, 4096, 8192};
    int ns = 7;
    if (argc > 1) {
        ns = 0;
        for (int i = 1; i < argc && ns < 32; ++i) sizes[ns++] = strtoull(argv[i], nullptr, 10);
    }
    for (int si = 0; si < ns; ++si) {
        const uint64_t bytes = sizes[si] << 20;
        const uint64_t n = bytes / 8;
        for (int blocks_per_sm : {4, 8}) {
            k_gather<8><<<sms * blocks_per_sm, 256>>>(a, n, loads, sink);
            cudaEventRecord(e0);
            k_gather<8><<<sms * blocks_per_sm, 256>>>(a, n, loads, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("array %6llu MB blocks/SM %d: %.2f Ggather/s (%.0f GB/s of 32B sectors)\n",
                   (unsigned long long)(bytes >> 20), blocks_per_sm, loads / ms / 1e6, loads * 32.0 / ms / 1e6);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
