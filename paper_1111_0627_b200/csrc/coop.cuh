// Grid-cooperative building blocks shared by the persistent solver kernel
// (solve_kernel.cuh) and the cooperative preparation kernels (prep.cu):
// relaxed control loads, cumulative ping-pong append counters (Ring) and
// block-aggregated appends/counts/flags.
//
// Ring protocol: an append phase reserves slots on counter `cur`; after the
// phase's grid barrier every thread calls take(), which reads how many were
// appended and flips to the other counter. That counter is not touched again
// until two append phases later, so every thread reads the same value; bases
// are thread-private copies that stay identical grid-wide. Every CTA must
// have read the bases (Ring::init) before any CTA appends.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "devcommon.cuh"

namespace ocmb {
namespace {

__device__ __forceinline__ std::size_t gtid() {
    return blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
}
__device__ __forceinline__ std::size_t gstride() { return std::size_t(gridDim.x) * blockDim.x; }

// Control values (counters, flags) read after a grid barrier: relaxed
// gpu-scope loads, coherent at L2 and never hoisted across the barrier.
__device__ __forceinline__ unsigned long long ldr(const unsigned long long& x) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&x) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ldr(const unsigned& x) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&x) : "memory");
    return v;
}
__device__ __forceinline__ int ldr(const int& x) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(&x) : "memory");
    return v;
}
// Four consecutive 16-byte aligned control ints in one relaxed load.
__device__ __forceinline__ int4 ldr4(const int* x) {
    int4 v;
    asm volatile("ld.relaxed.gpu.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(x)
                 : "memory");
    return v;
}
// Data another thread may write in the same phase.
template <class T> __device__ __forceinline__ T ldv(const T& x) {
    return *reinterpret_cast<const volatile T*>(&x);
}

// Plain loads are used for everything written in an earlier phase: the
// grid barrier's fences make those writes visible.
__device__ __forceinline__ bool working(const KP& p, std::uint32_t v) {
    return p.active[__ldg(&p.reg[v])] != 0;
}

// Set *flag to val unless it already is (read first: avoids store storms).
template <class T> __device__ __forceinline__ void set_once(T* flag, T val) {
    if (ldr(*flag) != val)
        *flag = val;
}

// Block-wide OR of a predicate, then one store per block.
template <class T> __device__ __forceinline__ void block_flag(bool pred, T* flag, T val) {
    if (__syncthreads_or(pred) && threadIdx.x == 0)
        set_once(flag, val);
}

// Cumulative append counters used in ping-pong pairs. An append phase
// reserves slots on counter `cur`; after the phase's grid barrier every
// thread calls take(), which reads how many were appended (the counter is
// not touched again until two append phases later, so all threads read the
// same value) and flips to the other counter. Every thread keeps identical
// private copies of the bases.
struct Ring {
    unsigned long long* ctr; // ctl->ring[i]
    unsigned long long base[2];
    int cur;
    __device__ void init(unsigned long long* c) {
        ctr = c;
        base[0] = ldr(c[0]);
        base[1] = ldr(c[1]);
        cur = 0;
    }
    __device__ __forceinline__ unsigned long long* counter() const { return &ctr[cur]; }
    __device__ __forceinline__ unsigned long long origin() const { return base[cur]; }
    __device__ std::uint64_t take() {
        const unsigned long long v = ldr(ctr[cur]);
        const std::uint64_t n = v - base[cur];
        base[cur] = v;
        cur ^= 1;
        return n;
    }
};

// Block-wide append: every thread of the block must call it (block-uniform
// loops). Returns this thread's slot relative to the ring's phase origin.
__device__ __forceinline__ std::uint64_t block_append(bool take, const Ring& ring) {
    __shared__ unsigned s_cnt[kBlock / 32];
    __shared__ unsigned long long s_base;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(FULL, take);
    if (lane == 0)
        s_cnt[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (unsigned w = 0; w < blockDim.x / 32; ++w) {
            const unsigned c = s_cnt[w];
            s_cnt[w] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(ring.counter(), static_cast<unsigned long long>(tot)) - ring.origin()
                     : 0ull;
    }
    __syncthreads();
    const std::uint64_t slot = s_base + s_cnt[warp] + __popc(bal & ((1u << lane) - 1u));
    __syncthreads();
    return slot;
}

// Two appends (to two rings) with one set of block barriers.
__device__ __forceinline__ void block_append2(bool ta, const Ring& ra, std::uint64_t& sa, bool tb,
                                              const Ring& rb, std::uint64_t& sb) {
    __shared__ unsigned s_a[kBlock / 32], s_b[kBlock / 32];
    __shared__ unsigned long long s_base_a, s_base_b;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bal_a = __ballot_sync(FULL, ta), bal_b = __ballot_sync(FULL, tb);
    if (lane == 0) {
        s_a[warp] = __popc(bal_a);
        s_b[warp] = __popc(bal_b);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot_a = 0, tot_b = 0;
        for (unsigned w = 0; w < blockDim.x / 32; ++w) {
            const unsigned ca = s_a[w], cb = s_b[w];
            s_a[w] = tot_a;
            s_b[w] = tot_b;
            tot_a += ca;
            tot_b += cb;
        }
        s_base_a = tot_a ? atomicAdd(ra.counter(), static_cast<unsigned long long>(tot_a)) - ra.origin()
                         : 0ull;
        s_base_b = tot_b ? atomicAdd(rb.counter(), static_cast<unsigned long long>(tot_b)) - rb.origin()
                         : 0ull;
    }
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
    sa = s_base_a + s_a[warp] + __popc(bal_a & below);
    sb = s_base_b + s_b[warp] + __popc(bal_b & below);
    __syncthreads();
}

// Block-wide reservation of per-thread counts on two rings (every thread
// of the block must call it): thread slots are consecutive in thread order,
// one atomic per ring per call.
__device__ __forceinline__ void block_reserve2(unsigned na, const Ring& ra, std::uint64_t& sa, unsigned nb,
                                               const Ring& rb, std::uint64_t& sb) {
    __shared__ unsigned s_a[kBlock / 32], s_b[kBlock / 32];
    __shared__ unsigned long long s_base_a, s_base_b;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // inclusive warp scans of both counts, packed 16|16 (counts <= 65535 per warp)
    unsigned x = na | (nb << 16);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, x, off);
        if (static_cast<int>(lane) >= off)
            x += y;
    }
    if (lane == 31) {
        s_a[warp] = x & 0xffffu;
        s_b[warp] = x >> 16;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot_a = 0, tot_b = 0;
        for (unsigned w = 0; w < blockDim.x / 32; ++w) {
            const unsigned ca = s_a[w], cb = s_b[w];
            s_a[w] = tot_a;
            s_b[w] = tot_b;
            tot_a += ca;
            tot_b += cb;
        }
        s_base_a = tot_a ? atomicAdd(ra.counter(), static_cast<unsigned long long>(tot_a)) - ra.origin()
                         : 0ull;
        s_base_b = tot_b ? atomicAdd(rb.counter(), static_cast<unsigned long long>(tot_b)) - rb.origin()
                         : 0ull;
    }
    __syncthreads();
    sa = s_base_a + s_a[warp] + (x & 0xffffu) - na;
    sb = s_base_b + s_b[warp] + (x >> 16) - nb;
    __syncthreads();
}

// Warp-aggregated append of the calling (active) lanes: one atomic per warp.
__device__ __forceinline__ std::uint64_t warp_append(const Ring& ring) {
    const unsigned m = __activemask();
    const int leader = __ffs(m) - 1;
    const unsigned lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (static_cast<int>(lane) == leader)
        base = atomicAdd(ring.counter(), static_cast<unsigned long long>(__popc(m))) - ring.origin();
    base = __shfl_sync(m, base, leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

// Block-reduced count added to the ring's current counter.
__device__ __forceinline__ void block_count(unsigned mine, const Ring& ring) {
    __shared__ unsigned s_sum;
    if (threadIdx.x == 0)
        s_sum = 0;
    __syncthreads();
    unsigned w = mine;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
        w += __shfl_xor_sync(FULL, w, off);
    if ((threadIdx.x & 31) == 0 && w)
        atomicAdd(&s_sum, w);
    __syncthreads();
    if (threadIdx.x == 0 && s_sum)
        atomicAdd(ring.counter(), static_cast<unsigned long long>(s_sum));
    __syncthreads(); // s_sum is reset by the block's next call (racecheck-clean)
}

} // namespace
} // namespace ocmb
