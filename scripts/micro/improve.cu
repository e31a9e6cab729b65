// Microbenchmark: the exact-lane improvement pass (howard_par.hpp:146
// spf_pass_iter) in isolation, on a uniform random digraph held in HBM:
// candidate = key[target] + w*den per edge, lexicographic (candidate, edge)
// argmin per vertex, policy written where it strictly improves.
//
//   A  thread per vertex, edges loaded with __ldg, 4 in flight (the r01 k_solve pass)
//   B  the same with all 8 edges in flight
//   C  edges and row offsets staged into shared memory by 1-D bulk TMA
//      (cp.async.bulk + mbarrier, double-buffered chunks of <= 256 vertices /
//      2048 edges), then thread per vertex with 8 key gathers in flight
//
// usage: improve <n> <deg> [passes] [cold]
//   cold = 1: before every pass flush L2 (256 MB write) and re-touch the key
//   array, as inside k_solve (keys just written by the value phases, edge
//   stream evicted by them)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr unsigned NONE = 0xffffffffu;
constexpr int kBlock = 256;
constexpr int kChV = 256;   // vertices per chunk
constexpr int kChE = 2064;  // edges per chunk (16.5 KB; 2 stages x 4 CTAs fit one SM)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

__global__ void k_init(uint32_t n, uint32_t deg, uint32_t* row, int2* ew, long long* key, uint32_t* succ_e) {
    const uint64_t m = uint64_t(n) * deg;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m; i += uint64_t(gridDim.x) * blockDim.x) {
        ew[i] = make_int2(int(mix(i) % n), int(1 + mix(i ^ 0x5555) % 100));
        if (i <= n) row[i] = uint32_t(i * deg);
        if (i < n) { key[i] = (long long)(mix(i * 7 + 1) % 100000); succ_e[i] = uint32_t(i * deg + mix(i * 3) % deg); }
    }
}

template <int U>
__global__ void __launch_bounds__(kBlock, 4) k_direct(uint32_t n, const uint32_t* __restrict__ row,
        const int2* __restrict__ ew, const long long* key, uint32_t* succ_e, uint32_t* succ_v, long long den, unsigned* changes) {
    unsigned ch = 0;
    for (uint32_t v = blockIdx.x * kBlock + threadIdx.x; v < n; v += gridDim.x * kBlock) {
        const uint32_t b = __ldg(&row[v]), e_end = __ldg(&row[v + 1]);
        const uint32_t cur = succ_e[v];
        long long best = 0, curc = 0; uint32_t be = NONE;
        for (uint32_t e0 = b; e0 < e_end; e0 += U) {
            int2 ed[U]; long long kk[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ed[u] = __ldg(&ew[min(e0 + u, e_end - 1)]);
#pragma unroll
            for (int u = 0; u < U; ++u) kk[u] = __ldcg(&key[ed[u].x]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = e0 + u;
                if (e < e_end) {
                    const long long c = kk[u] + (long long)ed[u].y * den;
                    if (be == NONE || c < best) { best = c; be = e; }
                    if (e == cur) curc = c;
                }
            }
        }
        if (be != NONE && best < curc) {
            succ_e[v] = be; succ_v[v] = uint32_t(__ldg(&ew[be]).x); ++ch;
        }
    }
    if (ch) atomicAdd(changes, ch);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                    "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(parity) : "memory");
}

struct Chunk { uint32_t v0, v1; };

// issue the bulk copies of chunk c into stage s (one thread)
__device__ __forceinline__ void stage_chunk(const Chunk& c, const uint32_t* row, const int2* ew,
                                            uint32_t* srow, int2* sedge, uint64_t* bar, uint32_t& ebase, uint32_t& rbase) {
    // 16-byte aligned windows: rows from v0 rounded down to 4 entries, edges
    // from row[v0] rounded down to 2 records
    rbase = c.v0 & ~3u;
    const uint32_t rcount = ((c.v1 + 1 - rbase) + 3) & ~3u;
    const uint32_t e0 = __ldg(&row[c.v0]) & ~1u, e1 = (__ldg(&row[c.v1]) + 1) & ~1u;
    ebase = e0;
    const unsigned rb = rcount * 4, eb = (e1 - e0) * 8;
    mbar_expect(bar, rb + eb);
    bulk_g2s(srow, row + rbase, rb, bar);
    if (eb) bulk_g2s(sedge, ew + e0, eb, bar);
}

__global__ void __launch_bounds__(kBlock, 4) k_tma(const Chunk* chunks, uint32_t nchunks, const uint32_t* __restrict__ row,
        const int2* __restrict__ ew, const long long* key, uint32_t* succ_e, uint32_t* succ_v, long long den, unsigned* changes) {
    __shared__ alignas(16) int2 sedge[2][kChE + 2];
    __shared__ alignas(16) uint32_t srow[2][kChV + 8];
    __shared__ alignas(8) uint64_t bar[2];
    __shared__ uint32_t s_ebase[2], s_rbase[2];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1); mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned ch = 0;
    uint32_t c = blockIdx.x;
    int s = 0; unsigned phase[2] = {0, 0};
    if (threadIdx.x == 0 && c < nchunks) stage_chunk(chunks[c], row, ew, srow[0], sedge[0], &bar[0], s_ebase[0], s_rbase[0]);
    for (; c < nchunks; c += gridDim.x, s ^= 1) {
        const uint32_t cn = c + gridDim.x;
        if (threadIdx.x == 0 && cn < nchunks)
            stage_chunk(chunks[cn], row, ew, srow[s ^ 1], sedge[s ^ 1], &bar[s ^ 1], s_ebase[s ^ 1], s_rbase[s ^ 1]);
        mbar_wait(&bar[s], phase[s]);
        phase[s] ^= 1;
        __syncthreads(); // s_ebase visible
        const Chunk k = chunks[c];
        const uint32_t v = k.v0 + threadIdx.x;
        if (v < k.v1) {
            const uint32_t eb = s_ebase[s], rb = s_rbase[s];
            const uint32_t b = srow[s][v - rb], e_end = srow[s][v + 1 - rb];
            const uint32_t cur = succ_e[v];
            long long best = 0, curc = 0; uint32_t be = NONE;
            for (uint32_t e0 = b; e0 < e_end; e0 += 8) {
                long long kk[8]; int2 ed[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) ed[u] = sedge[s][min(e0 + u, e_end - 1) - eb];
#pragma unroll
                for (int u = 0; u < 8; ++u) kk[u] = __ldcg(&key[ed[u].x]);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t e = e0 + u;
                    if (e < e_end) {
                        const long long cc = kk[u] + (long long)ed[u].y * den;
                        if (be == NONE || cc < best) { best = cc; be = e; }
                        if (e == cur) curc = cc;
                    }
                }
            }
            if (be != NONE && best < curc) {
                succ_e[v] = be; succ_v[v] = uint32_t(sedge[s][be - eb].x); ++ch;
            }
        }
        __syncthreads(); // stage s is free for the next-but-one chunk
    }
    if (ch) atomicAdd(changes, ch);
}

__global__ void k_touch(const long long* key, uint32_t n, long long* sink) {
    long long acc = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += key[i];
    if (acc == 42) *sink = acc;
}

int main(int argc, char** argv) {
    const uint32_t n = argc > 1 ? strtoul(argv[1], nullptr, 10) : 1000000;
    const uint32_t deg = argc > 2 ? strtoul(argv[2], nullptr, 10) : 8;
    const int passes = argc > 3 ? atoi(argv[3]) : 20;
    const int cold = argc > 4 ? atoi(argv[4]) : 0;
    char* flush; CK(cudaMalloc(&flush, 256u << 20));
    long long* sink; CK(cudaMalloc(&sink, 8));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t m = uint64_t(n) * deg;
    uint32_t *row, *succ_e, *succ_v, *succ_e0; int2* ew; long long* key; unsigned* changes;
    CK(cudaMalloc(&row, (n + 1ull) * 4)); CK(cudaMalloc(&ew, m * 8)); CK(cudaMalloc(&key, n * 8ull));
    CK(cudaMalloc(&succ_e, n * 4ull)); CK(cudaMalloc(&succ_e0, n * 4ull)); CK(cudaMalloc(&succ_v, n * 4ull)); CK(cudaMalloc(&changes, 4));
    k_init<<<sms * 8, 256>>>(n, deg, row, ew, key, succ_e0);
    // chunks: <= kChV vertices and <= kChE - 2 edges each (host, from the uniform row)
    std::vector<Chunk> hc;
    for (uint32_t v = 0; v < n;) {
        uint32_t v1 = v, e = 0;
        while (v1 < n && v1 - v < kChV && e + deg <= kChE - 2) { e += deg; ++v1; }
        hc.push_back({v, v1}); v = v1;
    }
    Chunk* chunks; CK(cudaMalloc(&chunks, hc.size() * sizeof(Chunk)));
    CK(cudaMemcpy(chunks, hc.data(), hc.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int grid = sms * 4;
    unsigned ref = 0;
    for (int var = 0; var < 3; ++var) {
        float best = 1e9, tot = 0;
        unsigned got = 0;
        for (int it = 0; it < passes + 2; ++it) {
            CK(cudaMemcpy(succ_e, succ_e0, n * 4ull, cudaMemcpyDeviceToDevice));
            CK(cudaMemset(changes, 0, 4));
            if (cold) {
                CK(cudaMemset(flush, it, 256u << 20));
                k_touch<<<sms * 8, 256>>>(key, n, sink);
            }
            cudaEventRecord(a);
            if (var == 0) k_direct<4><<<grid, kBlock>>>(n, row, ew, key, succ_e, succ_v, 7, changes);
            if (var == 1) k_direct<8><<<grid, kBlock>>>(n, row, ew, key, succ_e, succ_v, 7, changes);
            if (var == 2) k_tma<<<grid, kBlock>>>(chunks, hc.size(), row, ew, key, succ_e, succ_v, 7, changes);
            cudaEventRecord(b); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (it >= 2) { tot += ms; if (ms < best) best = ms; }
            CK(cudaMemcpy(&got, changes, 4, cudaMemcpyDeviceToHost));
        }
        if (var == 0) ref = got;
        printf("%s n=%u deg=%u variant %c: avg %.1f us  best %.1f us  %.1f Ggather/s  changes %u%s\n", cold ? "cold" : "warm",
               n, deg, "ABC"[var], tot / passes * 1e3, best * 1e3, m / (tot / passes) / 1e6, got, got == ref ? "" : " MISMATCH");
    }
    CK(cudaGetLastError());
    return 0;
}
