// Device-side preparation: upload the host CSR once, split it into solver
// regions (strongly connected components, proj/src/scc.cpp), drop trivial
// regions and cross-region edges, and pack the intra-region CSR the solver
// streams every policy iteration.
//
// SCC on the device (the reference's --scc parallel lane, scc.cpp:105, does
// the same decomposition with trim + pivoted forward/backward reachability on
// its CPU engine; any correct partition gives the same solver result):
//   1. queue-based trimming of vertices with no in- or out-neighbour
//      (self-loops ignored) -- each is its own singleton component;
//   2. forward/backward BFS from the max-degree pivot: the intersection is
//      the pivot's component (the giant one on the benchmark graphs);
//   3. whatever remains is finished by max-label colouring: labels flow
//      forward to a fixpoint, each colour's root collects its component by a
//      backward closure inside the colour, repeat (re-trimming first).
// Vertices keep their original ids; trivial vertices get region R (never
// active) and empty intra-region edge lists.

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <atomic>
#include <cstring>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <condition_variable>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ocm_b200.h"
#include "coop.cuh"
#include "devcommon.cuh"
#include "graph.hpp"

namespace ocmb {

void device_prepare(const HostCsr& g, const ocm_solve_options& opt, DeviceState& d, PrepInfo& info);
void device_prepare_csr(std::uint32_t n, std::uint64_t m, DBuf<std::uint32_t>& row,
                        DBuf<std::uint32_t>& tgt, DBuf<double>& w, int exactness,
                        const ocm_solve_options& opt, DeviceState& d, PrepInfo& info,
                        cudaEvent_t w_ready = nullptr,
                        const std::function<void()>& w_host_done = nullptr);

namespace {

// One atomicMax per warp (warp-reduced, skipped when it cannot win): a
// whole grid max-reducing into one word otherwise serialises at L2.
__device__ __forceinline__ void warp_atomic_max(unsigned long long* dst, unsigned long long v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, off);
        v = o > v ? o : v;
    }
    if ((threadIdx.x & 31) == 0 && v && v > __ldcg(dst))
        atomicMax(dst, v);
}

__device__ __forceinline__ std::size_t tid_() {
    return blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
}
__device__ __forceinline__ std::size_t stride_() { return std::size_t(gridDim.x) * blockDim.x; }

struct PrepCounters {
    unsigned q[2];       // frontier sizes
    unsigned remaining;  // unassigned vertices
    int changed;
    int bad_weight;      // exact weight outside int32
    int non_integral;    // some weight is not an integer below 2^53 (checked graphs)
    unsigned long long bad_weight_edge; // least edge id with a non-finite weight (checked graphs)
    unsigned long long max_abs_bits; // max |w| as double bits
    unsigned long long pivot;        // (score << 32) | ~v
    unsigned max_region;
    unsigned regions_total;
    unsigned R;
    unsigned long long bfs_ring[4]; // cumulative append counters (kp_scc_coop: fwd, bwd; kp_trim_coop)
    long long clk[4];               // kp_scc_coop block-0 SM clocks: trim, pivot, reachability, assign
    unsigned levels;                // reachability levels
};

__global__ void kp_row32(const std::uint64_t* r64, std::uint32_t* r32, std::size_t n1) {
    for (std::size_t i = tid_(); i < n1; i += stride_())
        r32[i] = static_cast<std::uint32_t>(r64[i]);
}

// Out-degree / in-degree without self-loops, self-loop flags, max |w|.
// max |w| over all edges (as double bits: non-negative doubles order like
// their bit patterns).
// max |w|; with `check` also build_graph's weight contract for caller-provided
// arrays (graph.cpp:33-36): the least edge with a non-finite weight, and
// whether every weight is an integer below 2^53 (Graph::integer_exact)
__global__ void kp_max_abs(std::uint64_t m, const double* w, PrepCounters* pc, int check) {
    unsigned long long mx = 0;
    bool frac = false;
    for (std::uint64_t e = tid_(); e < m; e += stride_()) {
        const double x = w[e];
        const unsigned long long bits = __double_as_longlong(fabs(x));
        if (check) {
            if (!isfinite(x)) {
                atomicMin(&pc->bad_weight_edge, static_cast<unsigned long long>(e));
                continue;
            }
            frac |= floor(x) != x || fabs(x) >= 9007199254740992.0;
        }
        mx = bits > mx ? bits : mx;
    }
    warp_atomic_max(&pc->max_abs_bits, mx);
    if (check && __syncthreads_or(frac) && threadIdx.x == 0)
        pc->non_integral = 1;
}

// Thread-per-vertex edge loops would leave a power-law hub's 10^4..10^5
// edges to one thread: these kernels take 32 vertices per warp, a lane walks
// its own vertex's edges, and the warp walks every wide vertex's (> 32
// edges) together.
#define OCM_WARP_VERTICES(n, BODY_NARROW, BODY_WIDE)                                             \
    {                                                                                            \
        const unsigned lane = threadIdx.x & 31;                                                  \
        const std::size_t nw_ = stride_() >> 5;                                                  \
        for (std::size_t base_ = (tid_() >> 5) * 32; base_ < (n); base_ += nw_ * 32) {           \
            const bool on = base_ + lane < (n);                                                  \
            const std::uint32_t v = static_cast<std::uint32_t>(base_ + lane);                    \
            std::uint32_t b = 0, e_end = 0;                                                      \
            if (on) {                                                                            \
                b = row[v];                                                                      \
                e_end = row[v + 1];                                                              \
            }                                                                                    \
            const bool wide = e_end - b > 32;                                                    \
            if (on && !wide) {                                                                   \
                BODY_NARROW                                                                      \
            }                                                                                    \
            for (unsigned hv_ = __ballot_sync(FULL, wide); hv_; hv_ &= hv_ - 1) {                \
                const int j_ = __ffs(hv_) - 1;                                                   \
                const std::uint32_t hvx = static_cast<std::uint32_t>(base_ + j_);                \
                const std::uint32_t hb = __shfl_sync(FULL, b, j_), he = __shfl_sync(FULL, e_end, j_); \
                BODY_WIDE                                                                        \
            }                                                                                    \
        }                                                                                        \
    }

__global__ void kp_degrees(std::uint32_t n, const std::uint32_t* row, const std::uint32_t* tgt,
                           std::uint32_t* outd, std::uint32_t* ind, std::uint8_t* self) {
    OCM_WARP_VERTICES(n, {
        std::uint32_t o = 0;
        std::uint8_t sl = 0;
        for (std::uint32_t e = b; e < e_end; ++e) {
            const std::uint32_t t = tgt[e];
            if (t == v) {
                sl = 1;
            } else {
                ++o;
                atomicAdd(&ind[t], 1u);
            }
        }
        outd[v] = o;
        self[v] = sl;
    }, {
        std::uint32_t o = 0;
        bool sl = false;
        for (std::uint32_t e = hb + lane; e < he; e += 32) {
            const std::uint32_t t = tgt[e];
            if (t == hvx) {
                sl = true;
            } else {
                ++o;
                atomicAdd(&ind[t], 1u);
            }
        }
        o = __reduce_add_sync(FULL, o);
        sl = __any_sync(FULL, sl);
        if (lane == 0) {
            outd[hvx] = o;
            self[hvx] = sl ? 1 : 0;
        }
    })
}

// Backward CSR (no self-loops): bsrc grouped by target.
__global__ void kp_bwd_fill(std::uint32_t n, const std::uint32_t* row, const std::uint32_t* tgt,
                            std::uint32_t* cursor, std::uint32_t* bsrc) {
    OCM_WARP_VERTICES(n, {
        for (std::uint32_t e = b; e < e_end; ++e) {
            const std::uint32_t t = tgt[e];
            if (t != v)
                bsrc[atomicAdd(&cursor[t], 1u)] = v;
        }
    }, {
        for (std::uint32_t e = hb + lane; e < he; e += 32) {
            const std::uint32_t t = tgt[e];
            if (t != hvx)
                bsrc[atomicAdd(&cursor[t], 1u)] = hvx;
        }
    })
}

// Initial trim frontier among unassigned vertices: in- or out-degree 0.

// Process one trim frontier: each trimmed vertex removes its edges from the
// neighbours' counters; a neighbour reaching zero is trimmed next.

// Recount degrees inside the unassigned subgraph (pull, no atomics).
__global__ void kp_recount(std::uint32_t n, const std::uint32_t* row, const std::uint32_t* tgt,
                           const std::uint32_t* brow, const std::uint32_t* bsrc,
                           const std::uint32_t* lab, std::uint32_t* ind, std::uint32_t* outd,
                           PrepCounters* pc) {
    unsigned rem = 0;
    for (std::size_t vv = tid_(); vv < n; vv += stride_()) {
        const std::uint32_t v = static_cast<std::uint32_t>(vv);
        if (lab[v] != NONE)
            continue;
        ++rem;
        std::uint32_t o = 0, i = 0;
        for (std::uint32_t e = row[v]; e < row[v + 1]; ++e) {
            const std::uint32_t t = tgt[e];
            o += (t != v && lab[t] == NONE);
        }
        for (std::uint32_t s = brow[v]; s < brow[v + 1]; ++s)
            i += lab[bsrc[s]] == NONE;
        outd[v] = o;
        ind[v] = i;
    }
    rem = __reduce_add_sync(FULL, rem);
    if ((threadIdx.x & 31) == 0 && rem)
        atomicAdd(&pc->remaining, rem);
}


// Queue-based trimming (vertices left with no in- or out-neighbour among the
// unassigned ones are singleton components) to its fixpoint in one
// cooperative launch: seed pass, then one grid barrier per level.
__device__ __forceinline__ void trim_fixpoint(cooperative_groups::grid_group& grid, std::uint32_t n,
                                              const std::uint32_t* row, const std::uint32_t* tgt,
                                              const std::uint32_t* brow, const std::uint32_t* bsrc,
                                              std::uint32_t* ind, std::uint32_t* outd, std::uint32_t* lab,
                                              std::uint32_t* q0, std::uint32_t* q1, Ring& ring) {
    for (std::size_t base = blockIdx.x * std::size_t(kBlock); base < n;
         base += gridDim.x * std::size_t(kBlock)) {
        const std::size_t v = base + threadIdx.x;
        bool take = false;
        if (v < n && lab[v] == NONE && (ind[v] == 0 || outd[v] == 0)) {
            lab[v] = static_cast<std::uint32_t>(v);
            take = true;
        }
        const std::uint64_t slot = block_append(take, ring);
        if (take)
            q0[slot] = static_cast<std::uint32_t>(v);
    }
    grid.sync();
    std::uint64_t nin = ring.take();
    int cur = 0;
    while (nin) {
        const std::uint32_t* qin = cur ? q1 : q0;
        std::uint32_t* qout = cur ? q0 : q1;
        for (std::uint64_t i = gtid(); i < nin; i += gstride()) {
            const std::uint32_t v = qin[i];
            for (std::uint32_t e = row[v]; e < row[v + 1]; ++e) {
                const std::uint32_t t = tgt[e];
                if (t == v || lab[t] != NONE)
                    continue;
                if (atomicSub(&ind[t], 1u) == 1u && atomicCAS(&lab[t], NONE, t) == NONE)
                    qout[warp_append(ring)] = t;
            }
            for (std::uint32_t e = brow[v]; e < brow[v + 1]; ++e) {
                const std::uint32_t u = bsrc[e];
                if (lab[u] != NONE)
                    continue;
                if (atomicSub(&outd[u], 1u) == 1u && atomicCAS(&lab[u], NONE, u) == NONE)
                    qout[warp_append(ring)] = u;
            }
        }
        grid.sync();
        nin = ring.take();
        cur ^= 1;
    }
}

__global__ void __launch_bounds__(kBlock) kp_trim_coop(std::uint32_t n, const std::uint32_t* row,
                                                       const std::uint32_t* tgt, const std::uint32_t* brow,
                                                       const std::uint32_t* bsrc, std::uint32_t* ind,
                                                       std::uint32_t* outd, std::uint32_t* lab,
                                                       std::uint32_t* q0, std::uint32_t* q1,
                                                       unsigned long long* ring_ctr) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    Ring ring;
    ring.init(ring_ctr);
    grid.sync(); // every CTA has read the ring bases
    trim_fixpoint(grid, n, row, tgt, brow, bsrc, ind, outd, lab, q0, q1, ring);
}

// One BFS level (restricted to unassigned vertices; vis[v] = the level that
// reached v, 0 = not reached). Top-down pushes every frontier edge through a
// CAS and lists the newly reached vertices (warp-aggregated appends: the
// frontier is short here). Bottom-up -- used while the frontier is a sizeable
// share of the graph -- lets every unreached vertex scan its in-edges
// (rrow/rcol) and stop at the first reached one; it lists nothing (one
// contended append per hit would serialise on the counter) and only counts
// the hits per block. Reachability only (vis is monotone), so racing readers
// of vis[] stay correct.
__device__ __forceinline__ void bfs_level(const std::uint32_t* row, const std::uint32_t* col,
                                          const std::uint32_t* rrow, const std::uint32_t* rcol,
                                          std::uint32_t n, const std::uint32_t* lab, std::uint32_t* vis,
                                          std::uint32_t level, bool bottom_up, const std::uint32_t* qin,
                                          std::uint64_t nin, std::uint32_t* qout, const Ring& ring) {
    if (bottom_up) {
        unsigned got = 0;
        for (std::uint64_t v = gtid(); v < n; v += gstride()) {
            if (lab[v] != NONE || vis[v] != 0)
                continue;
            const std::uint32_t b = rrow[v], e_end = rrow[v + 1];
            // 8 in-neighbours and their marks in flight at a time
            for (std::uint32_t e0 = b; e0 < e_end; e0 += 8) {
                std::uint32_t src[8];
                bool hit = false;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    src[u] = rcol[min(e0 + u, e_end - 1)];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    hit |= ldv(vis[src[u]]) != 0;
                if (hit) {
                    vis[v] = level;
                    ++got;
                    break;
                }
            }
        }
        block_count(got, ring);
    } else {
        // 32 frontier vertices per warp: a lane walks its own vertex's
        // edges, the warp walks a high-degree vertex's together (a hub's
        // 10^4..10^5 edges would otherwise be one thread's serial loop)
        const unsigned lane = threadIdx.x & 31;
        const std::uint64_t nw = gstride() >> 5;
        for (std::uint64_t base = (gtid() >> 5) * 32; base < nin; base += nw * 32) {
            std::uint32_t b = 0, e_end = 0;
            if (base + lane < nin) {
                const std::uint32_t u = qin[base + lane];
                b = row[u];
                e_end = row[u + 1];
            }
            const bool wide = e_end - b > 32;
            if (!wide)
                for (std::uint32_t e = b; e < e_end; ++e) {
                    const std::uint32_t t = col[e];
                    if (lab[t] != NONE || vis[t] != 0)
                        continue;
                    if (atomicCAS(&vis[t], 0u, level) == 0u)
                        qout[warp_append(ring)] = t;
                }
            for (unsigned hv = __ballot_sync(FULL, wide); hv; hv &= hv - 1) {
                const int j = __ffs(hv) - 1;
                const std::uint32_t hb = __shfl_sync(FULL, b, j), he = __shfl_sync(FULL, e_end, j);
                for (std::uint32_t e = hb + lane; e < he; e += 32) {
                    const std::uint32_t t = col[e];
                    if (lab[t] != NONE || vis[t] != 0)
                        continue;
                    if (atomicCAS(&vis[t], 0u, level) == 0u)
                        qout[warp_append(ring)] = t;
                }
            }
        }
    }
}

// The frontier of a top-down level that follows a bottom-up one: the
// vertices the bottom-up level reached (block-aggregated appends).
__device__ __forceinline__ void bfs_collect(std::uint32_t n, const std::uint32_t* vis, std::uint32_t level,
                                            std::uint32_t* qout, const Ring& ring) {
    for (std::size_t base = blockIdx.x * std::size_t(kBlock); base < n;
         base += gridDim.x * std::size_t(kBlock)) {
        const std::size_t v = base + threadIdx.x;
        const bool take = v < n && vis[v] == level;
        const std::uint64_t slot = block_append(take, ring);
        if (take)
            qout[slot] = static_cast<std::uint32_t>(v);
    }
}


// The whole first pass of the region split in one cooperative launch:
// trimming to its fixpoint, the pivot (max (1+in)(1+out) among the
// survivors, least id on ties), forward and backward reachability, the
// pivot's component, and the count of vertices still unassigned (which
// decides whether the colouring fallback runs). One host read follows.
__global__ void __launch_bounds__(kBlock) kp_scc_coop(std::uint32_t n, const std::uint32_t* row,
                                                      const std::uint32_t* col, const std::uint32_t* brow,
                                                      const std::uint32_t* bcol, std::uint32_t* ind,
                                                      std::uint32_t* outd, std::uint32_t* lab,
                                                      std::uint32_t* visf, std::uint32_t* visb,
                                                      std::uint32_t* qf0, std::uint32_t* qf1,
                                                      std::uint32_t* qb0, std::uint32_t* qb1,
                                                      PrepCounters* pc) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    Ring rf, rb;
    rf.init(pc->bfs_ring);
    rb.init(pc->bfs_ring + 2);
    grid.sync(); // every CTA has read the ring bases
    const bool clk0 = blockIdx.x == 0 && threadIdx.x == 0;
    long long t = clk0 ? clock64() : 0;
    auto lap = [&](int i) {
        if (clk0) {
            const long long u = clock64();
            pc->clk[i] = u - t;
            t = u;
        }
    };
    trim_fixpoint(grid, n, row, col, brow, bcol, ind, outd, lab, qf0, qf1, rf);
    lap(0);
    // trimming kept ind/outd exact for the surviving subgraph
    {
        unsigned long long best = 0;
        unsigned rem = 0;
        for (std::size_t v = gtid(); v < n; v += gstride()) {
            if (lab[v] != NONE)
                continue;
            ++rem;
            const unsigned long long score = min(0xffffffffull, (1ull + ind[v]) * (1ull + outd[v]));
            const unsigned long long key = (score << 32) | (0xffffffffull - v);
            best = key > best ? key : best;
        }
        warp_atomic_max(&pc->pivot, best);
        block_count(rem, rb);
    }
    grid.sync();
    if (rb.take() == 0) {
        if (gtid() == 0)
            pc->remaining = 0;
        return;
    }
    const std::uint32_t start = 0xffffffffu - static_cast<std::uint32_t>(ldr(pc->pivot) & 0xffffffffull);
    if (gtid() == 0) {
        qf0[0] = start;
        qb0[0] = start;
        visf[start] = 1;
        visb[start] = 1;
    }
    grid.sync(); // the seed is visible
    lap(1);
    std::uint64_t nf = 1, nb = 1;
    bool f_was_bu = false, b_was_bu = false;
    int cf = 0, cb = 0; // which queue holds the current frontier
    const std::uint64_t bu_from = n >> 6;
    std::uint32_t level = 2;
    for (; nf || nb; ++level) {
        const bool f_bu = nf > bu_from, b_bu = nb > bu_from;
        const bool f_cmp = nf && !f_bu && f_was_bu, b_cmp = nb && !b_bu && b_was_bu;
        if (f_cmp || b_cmp) {
            if (f_cmp)
                bfs_collect(n, visf, level - 1, cf ? qf1 : qf0, rf);
            if (b_cmp)
                bfs_collect(n, visb, level - 1, cb ? qb1 : qb0, rb);
            grid.sync();
            if (f_cmp)
                nf = rf.take();
            if (b_cmp)
                nb = rb.take();
        }
        if (nf)
            bfs_level(row, col, brow, bcol, n, lab, visf, level, f_bu, cf ? qf1 : qf0, nf, cf ? qf0 : qf1, rf);
        if (nb)
            bfs_level(brow, bcol, row, col, n, lab, visb, level, b_bu, cb ? qb1 : qb0, nb, cb ? qb0 : qb1, rb);
        grid.sync();
        if (nf) {
            f_was_bu = f_bu;
            nf = rf.take();
            cf ^= 1;
        }
        if (nb) {
            b_was_bu = b_bu;
            nb = rb.take();
            cb ^= 1;
        }
    }
    if (clk0)
        pc->levels = level - 2;
    lap(2);
    // the pivot's component; count what is left for the colouring
    unsigned rem = 0;
    for (std::size_t v = gtid(); v < n; v += gstride()) {
        if (lab[v] != NONE)
            continue;
        if (visf[v] != 0 && visb[v] != 0)
            lab[v] = start;
        else
            ++rem;
    }
    block_count(rem, rf);
    grid.sync();
    const std::uint64_t left = rf.take();
    lap(3);
    if (gtid() == 0)
        pc->remaining = static_cast<unsigned>(left);
}


// Colouring: colour = max id among vertices reaching v (in-place, pull).
__global__ void kp_color_init(std::uint32_t n, const std::uint32_t* lab, std::uint32_t* color) {
    for (std::size_t v = tid_(); v < n; v += stride_())
        if (lab[v] == NONE)
            color[v] = static_cast<std::uint32_t>(v);
}

__global__ void kp_color_prop(std::uint32_t n, const std::uint32_t* brow, const std::uint32_t* bsrc,
                              const std::uint32_t* lab, std::uint32_t* color, PrepCounters* pc) {
    bool ch = false;
    for (std::size_t vv = tid_(); vv < n; vv += stride_()) {
        if (lab[vv] != NONE)
            continue;
        std::uint32_t c = color[vv];
        const std::uint32_t c0 = c;
        for (std::uint32_t s = brow[vv]; s < brow[vv + 1]; ++s) {
            const std::uint32_t u = bsrc[s];
            if (lab[u] == NONE) {
                const std::uint32_t cu = *(volatile std::uint32_t*)&color[u];
                c = cu > c ? cu : c;
            }
        }
        if (c != c0) {
            color[vv] = c;
            ch = true;
        }
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0)
        pc->changed = 1;
}

// Backward closure inside each colour from its root (in-place, pull).
__global__ void kp_color_roots(std::uint32_t n, const std::uint32_t* lab, const std::uint32_t* color,
                               std::uint32_t* in_scc, std::uint32_t stamp) {
    for (std::size_t v = tid_(); v < n; v += stride_())
        if (lab[v] == NONE && color[v] == v)
            in_scc[v] = stamp;
}

__global__ void kp_color_close(std::uint32_t n, const std::uint32_t* row, const std::uint32_t* tgt,
                               const std::uint32_t* lab, const std::uint32_t* color,
                               std::uint32_t* in_scc, std::uint32_t stamp, PrepCounters* pc) {
    bool ch = false;
    for (std::size_t vv = tid_(); vv < n; vv += stride_()) {
        if (lab[vv] != NONE || in_scc[vv] == stamp)
            continue;
        const std::uint32_t c = color[vv];
        for (std::uint32_t e = row[vv]; e < row[vv + 1]; ++e) {
            const std::uint32_t t = tgt[e];
            if (lab[t] == NONE && color[t] == c &&
                *(volatile std::uint32_t*)&in_scc[t] == stamp) {
                in_scc[vv] = stamp;
                ch = true;
                break;
            }
        }
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0)
        pc->changed = 1;
}

__global__ void kp_color_assign(std::uint32_t n, const std::uint32_t* color,
                                const std::uint32_t* in_scc, std::uint32_t stamp,
                                std::uint32_t* lab) {
    for (std::size_t v = tid_(); v < n; v += stride_())
        if (lab[v] == NONE && in_scc[v] == stamp)
            lab[v] = color[v];
}

// Component sizes at the representatives (lab[r] == r).
__global__ void kp_sizes(std::uint32_t n, const std::uint32_t* lab, std::uint32_t* size) {
    // warp-aggregated: lanes sharing a label add once (the giant component
    // would otherwise serialise every vertex on one word)
    for (std::size_t base = (tid_() & ~std::size_t(31)); base < n; base += stride_()) {
        const std::size_t v = base + (threadIdx.x & 31);
        const bool on = v < n;
        const std::uint32_t l = on ? lab[v] : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, l);
        if (on && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1))
            atomicAdd(&size[l], static_cast<unsigned>(__popc(peers)));
    }
}

__global__ void kp_nontrivial(std::uint32_t n, const std::uint32_t* lab, const std::uint32_t* size,
                              const std::uint8_t* self, std::uint32_t* flag, PrepCounters* pc) {
    unsigned mx = 0, reps = 0;
    for (std::size_t v = tid_(); v < n; v += stride_()) {
        std::uint32_t f = 0;
        if (lab[v] == v) {
            ++reps;
            f = (size[v] > 1 || self[v]) ? 1u : 0u;
            if (f)
                mx = size[v] > mx ? size[v] : mx;
        }
        flag[v] = f;
    }
    reps = __reduce_add_sync(FULL, reps);
    mx = __reduce_max_sync(FULL, mx);
    if ((threadIdx.x & 31) == 0) {
        if (reps)
            atomicAdd(&pc->regions_total, reps);
        if (mx)
            atomicMax(&pc->max_region, mx);
    }
}

__global__ void kp_region_ids(std::uint32_t n, const std::uint32_t* lab, const std::uint32_t* flag,
                              const std::uint32_t* rid, std::uint32_t R, std::uint32_t* reg) {
    for (std::size_t v = tid_(); v < n; v += stride_()) {
        const std::uint32_t r = lab[v];
        reg[v] = flag[r] ? rid[r] : R;
    }
}

__global__ void kp_count_intra(std::uint32_t n, std::uint32_t R, const std::uint32_t* row,
                               const std::uint32_t* tgt, const std::uint32_t* reg,
                               std::uint32_t* cnt) {
    OCM_WARP_VERTICES(n, {
        const std::uint32_t r = reg[v];
        std::uint32_t c = 0;
        if (r != R)
            for (std::uint32_t e = b; e < e_end; ++e)
                c += reg[tgt[e]] == r;
        cnt[v] = c;
    }, {
        const std::uint32_t r = reg[hvx];
        std::uint32_t c = 0;
        if (r != R)
            for (std::uint32_t e = hb + lane; e < he; e += 32)
                c += reg[tgt[e]] == r;
        c = __reduce_add_sync(FULL, c);
        if (lane == 0)
            cnt[hvx] = c;
    })
}

// ew_hi != nullptr: the wide exact lane (64-bit weights, the high half in
// ew_hi); otherwise a weight outside int32 is reported.
template <bool EXACT>
__device__ __forceinline__ bool pack_one(std::uint32_t t, double x, std::uint32_t k, int2* ew,
                                         int* ew_hi, FEdge* fe) {
    if constexpr (EXACT) {
        if (ew_hi) {
            const long long wv = static_cast<long long>(x);
            ew[k] = make_int2(static_cast<int>(t), static_cast<int>(static_cast<unsigned>(wv)));
            ew_hi[k] = static_cast<int>(wv >> 32);
            return false;
        }
        ew[k] = make_int2(static_cast<int>(t), static_cast<int>(x));
        return !(fabs(x) <= 2147483647.0);
    } else {
        fe[k] = FEdge{x, t, 0u};
        return false;
    }
}

template <bool EXACT>
__global__ void kp_pack(std::uint32_t n, std::uint32_t R, const std::uint32_t* row,
                        const std::uint32_t* tgt, const double* w, const std::uint32_t* reg,
                        const std::uint32_t* nrow, double sign, int2* ew, int* ew_hi, FEdge* fe,
                        PrepCounters* pc) {
    bool bad = false;
    OCM_WARP_VERTICES(n, {
        const std::uint32_t r = reg[v];
        if (r != R) {
            std::uint32_t k = nrow[v];
            for (std::uint32_t e = b; e < e_end; ++e) {
                const std::uint32_t t = tgt[e];
                if (reg[t] == r)
                    bad |= pack_one<EXACT>(t, sign * w[e], k++, ew, ew_hi, fe);
            }
        }
    }, {
        // edge order kept: 32 edges at a time, slots from a ballot prefix
        const std::uint32_t r = reg[hvx];
        if (r != R) {
            std::uint32_t k = nrow[hvx];
            for (std::uint32_t e0 = hb; e0 < he; e0 += 32) {
                const std::uint32_t e = e0 + lane;
                std::uint32_t t = 0;
                bool in = false;
                if (e < he) {
                    t = tgt[e];
                    in = reg[t] == r;
                }
                const unsigned m = __ballot_sync(FULL, in);
                if (in)
                    bad |= pack_one<EXACT>(t, sign * w[e], k + __popc(m & ((1u << lane) - 1u)), ew,
                                           ew_hi, fe);
                k += __popc(m);
            }
        }
    })
    if (__syncthreads_or(bad) && threadIdx.x == 0)
        pc->bad_weight = 1;
}

// Hamiltonian augmentation (graph.cpp:105) packed directly: vertex v keeps
// its edges and gains v -> v+1 mod n with weight big_w (already in the
// minimised orientation), appended last so edge order is preserved.
template <bool EXACT>
__global__ void kp_pack_hamiltonian(std::uint32_t n, const std::uint32_t* row,
                                    const std::uint32_t* tgt, const double* w, double sign,
                                    double big_w, int2* ew, int* ew_hi, FEdge* fe,
                                    std::uint32_t* nrow, std::uint32_t* reg, PrepCounters* pc) {
    bool bad = false;
    for (std::size_t vv = tid_(); vv <= n; vv += stride_()) {
        const std::uint32_t v = static_cast<std::uint32_t>(vv);
        nrow[v] = row[v] + v;
        if (v == n)
            continue;
        reg[v] = 0;
        std::uint32_t k = row[v] + v;
        for (std::uint32_t e = row[v]; e <= row[v + 1]; ++e) {
            const bool extra = e == row[v + 1];
            const std::uint32_t t = extra ? (v + 1) % n : tgt[e];
            const double x = extra ? big_w : sign * w[e];
            bad |= pack_one<EXACT>(t, x, k, ew, ew_hi, fe);
            ++k;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0)
        pc->bad_weight = 1;
}

template <class T> void exclusive_scan(const T* in, T* out, std::size_t n, cudaStream_t s) {
    std::size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    DBuf<unsigned char> tmp;
    tmp.alloc(std::max<std::size_t>(bytes, 1), s);
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, s));
}

} // namespace

namespace {

// Host->device copies from memory the library did not allocate. Page-locked
// (or registered) sources go straight to the copy engine; pageable ones are
// staged through a per-process ring of pinned buffers: the host copies chunk
// i+1 into one slot (several threads) while the copy engine drains chunk i
// from the other, so the transfer runs at PCIe speed instead of the driver's
// pageable-copy path, and the caller's arrays are never registered or
// modified. One ring per process, serialised by a lock.
// out[i] = (int)in[i]; true if any in[i] is not an integer in int32 range
// (or not finite). SSE2 truncation returns INT_MIN for out-of-range and NaN
// inputs, so "converts back to itself" is the whole test (-0.0 passes as 0).
bool narrow_i32(int* out, const double* in, std::size_t n) {
    std::size_t i = 0;
    bool bad = false;
#if defined(__SSE2__)
    __m128d acc = _mm_setzero_pd();
    for (; i + 4 <= n; i += 4) {
        const __m128d a = _mm_loadu_pd(in + i), b = _mm_loadu_pd(in + i + 2);
        const __m128i ia = _mm_cvttpd_epi32(a), ib = _mm_cvttpd_epi32(b);
        acc = _mm_or_pd(acc, _mm_cmpneq_pd(_mm_cvtepi32_pd(ia), a));
        acc = _mm_or_pd(acc, _mm_cmpneq_pd(_mm_cvtepi32_pd(ib), b));
        _mm_storeu_si128(reinterpret_cast<__m128i*>(out + i), _mm_unpacklo_epi64(ia, ib));
    }
    bad = _mm_movemask_pd(acc) != 0;
#endif
    for (; i < n; ++i) {
        const double x = in[i];
        const bool inr = x >= -2147483648.0 && x <= 2147483647.0; // false for NaN
        const int v = inr ? static_cast<int>(x) : 0;
        bad |= !inr || static_cast<double>(v) != x;
        out[i] = v;
    }
    return bad;
}

class StagingRing {
  public:
    // chunk size (OCM_STAGE_MB) and host copy threads (OCM_COPY_THREADS) are
    // read once per process
    std::size_t kChunk = 8u << 20; // 8 MB: +2.7% e2e over 16 MB (profiles/r02/e2e_staging_r02.log)
    static constexpr int kSlots = 3;

    static StagingRing& get() {
        static StagingRing r;
        return r;
    }

    void copy(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
        if (bytes == 0)
            return;
        if (pinned(src)) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
            return;
        }
        std::lock_guard<std::mutex> lock(mu_);
        ensure();
        const char* from = static_cast<const char*>(src);
        char* to = static_cast<char*>(dst);
        for (std::size_t off = 0; off < bytes; off += kChunk) {
            const std::size_t len = std::min(kChunk, bytes - off);
            const int k = static_cast<int>(next_++ % kSlots);
            CK(cudaEventSynchronize(done_[k])); // the slot's previous copy has left
            host_copy(buf_[k], from + off, len);
            CK(cudaMemcpyAsync(to + off, buf_[k], len, cudaMemcpyHostToDevice, s));
            CK(cudaEventRecord(done_[k], s));
        }
    }

    // Weights that are all integers in int32 range cross PCIe as int32 --
    // half the bytes -- into `tmp`, converted (and checked) by the host
    // threads filling the staging slots. Returns false at the first chunk
    // holding any other value (non-integral, too large, non-finite): the
    // caller then copies the doubles. Pinned sources return false at once
    // (the copy engine reads them directly, faster than a host pass).
    bool copy_narrow(int* tmp, const double* src, std::size_t count, cudaStream_t s) {
        if (count == 0 || pinned(src))
            return false;
        std::lock_guard<std::mutex> lock(mu_);
        ensure();
        const std::size_t kPer = kChunk / sizeof(int);
        for (std::size_t off = 0; off < count; off += kPer) {
            const std::size_t len = std::min(kPer, count - off);
            const int k = static_cast<int>(next_++ % kSlots);
            CK(cudaEventSynchronize(done_[k]));
            int* out = reinterpret_cast<int*>(buf_[k]);
            const double* in = src + off;
            std::atomic<bool> bad{false};
            host_parts(len, [out, in, &bad](std::size_t lo, std::size_t hi) {
                if (narrow_i32(out + lo, in + lo, hi - lo))
                    bad.store(true, std::memory_order_relaxed);
            });
            if (bad.load())
                return false;
            CK(cudaMemcpyAsync(tmp + off, out, len * sizeof(int), cudaMemcpyHostToDevice, s));
            CK(cudaEventRecord(done_[k], s));
        }
        return true;
    }

  private:
    static bool pinned(const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    }
    void ensure() {
        if (buf_[0])
            return;
        if (const char* mb = std::getenv("OCM_STAGE_MB"))
            if (std::atoi(mb) > 0)
                kChunk = std::size_t(std::atoi(mb)) << 20;
        for (int k = 0; k < kSlots; ++k) {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&buf_[k]), kChunk, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&done_[k], cudaEventDisableTiming));
            CK(cudaEventRecord(done_[k], nullptr));
        }
    }
    // memcpy split over a persistent pool of host threads (one thread copies
    // ~10 GB/s, below the PCIe rate; threads are started once per process)
    class CopyPool {
      public:
        explicit CopyPool(int n) : n_(n) {
            for (int t = 1; t < n_; ++t)
                th_.emplace_back([this, t] { run(t); });
        }
        ~CopyPool() {
            {
                std::lock_guard<std::mutex> l(m_);
                quit_ = true;
                ++gen_;
            }
            cv_.notify_all();
            for (auto& x : th_)
                x.join();
        }
        void copy(char* dst, const char* src, std::size_t len) {
            run_parts(len, [dst, src](std::size_t lo, std::size_t hi) {
                std::memcpy(dst + lo, src + lo, hi - lo);
            });
        }
        // fn(lo, hi) over [0, len) in n_ parts of multiples of 64
        void run_parts(std::size_t len, const std::function<void(std::size_t, std::size_t)>& fn) {
            if (len < (1u << 20) || n_ == 1) {
                fn(0, len);
                return;
            }
            {
                std::lock_guard<std::mutex> l(m_);
                fn_ = &fn;
                len_ = len;
                pending_ = n_ - 1;
                ++gen_;
            }
            cv_.notify_all();
            part(0);
            std::unique_lock<std::mutex> l(m_);
            done_cv_.wait(l, [this] { return pending_ == 0; });
        }

      private:
        void part(int t) {
            const std::size_t per = ((len_ + n_ - 1) / n_ + 63) & ~std::size_t(63);
            const std::size_t lo = std::min(len_, per * t), hi = std::min(len_, per * (t + 1));
            if (hi > lo)
                (*fn_)(lo, hi);
        }
        void run(int t) {
            unsigned long long seen = 0;
            for (;;) {
                {
                    std::unique_lock<std::mutex> l(m_);
                    cv_.wait(l, [&] { return gen_ != seen; });
                    seen = gen_;
                    if (quit_)
                        return;
                }
                part(t);
                std::lock_guard<std::mutex> l(m_);
                if (--pending_ == 0)
                    done_cv_.notify_one();
            }
        }
        int n_;
        std::vector<std::thread> th_;
        std::mutex m_;
        std::condition_variable cv_, done_cv_;
        unsigned long long gen_ = 0;
        int pending_ = 0;
        bool quit_ = false;
        const std::function<void(std::size_t, std::size_t)>* fn_ = nullptr;
        std::size_t len_ = 0;
    };
    void host_copy(char* dst, const char* src, std::size_t len) {
        if (!pool_) {
            const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
            int nt = static_cast<int>(std::min(8u, std::max(1u, hw / 2)));
            if (const char* e = std::getenv("OCM_COPY_THREADS"))
                if (std::atoi(e) > 0)
                    nt = std::atoi(e);
            pool_ = std::make_unique<CopyPool>(nt);
        }
        pool_->copy(dst, src, len);
    }
    void host_parts(std::size_t len, const std::function<void(std::size_t, std::size_t)>& fn) {
        if (!pool_)
            host_copy(nullptr, nullptr, 0); // starts the pool
        pool_->run_parts(len, fn);
    }
    std::unique_ptr<CopyPool> pool_;
    std::mutex mu_;
    char* buf_[kSlots] = {};
    cudaEvent_t done_[kSlots] = {};
    unsigned long long next_ = 0;
};

// Checks a caller-provided CSR's offsets and targets on the device (the
// reference's build_graph contract, src/graph.cpp:29-32, plus well-formed
// offsets) before the region split reads them; the weights stream in on
// the side stream meanwhile and are checked where they are first read
// (kp_max_abs with check = 1).
__global__ void kp_widen_w(std::uint64_t m, const int* wi, double* w) {
    for (std::uint64_t e = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; e < m;
         e += std::uint64_t(gridDim.x) * blockDim.x)
        w[e] = static_cast<double>(wi[e]);
}

struct CsrCheck {
    unsigned long long bad_target;
    unsigned long long bad_weight;
    int non_integral;
    int bad_offsets;
};

__global__ void kp_check_csr(std::uint32_t n, std::uint64_t m, const std::uint32_t* row,
                             const std::uint32_t* tgt, const double* w, CsrCheck* out) {
    const std::uint64_t tid = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
    const std::uint64_t nth = std::uint64_t(gridDim.x) * blockDim.x;
    bool bad_row = false;
    for (std::uint64_t v = tid; v < n; v += nth)
        bad_row |= row[v] > row[v + 1];
    if (tid == 0)
        bad_row |= row[0] != 0 || row[n] != m;
    for (std::uint64_t e = tid; e < m; e += nth) {
        if (tgt[e] >= n)
            atomicMin(&out->bad_target, static_cast<unsigned long long>(e));
        if (w && !isfinite(w[e])) // only when a bad target needs the weights' order too
            atomicMin(&out->bad_weight, static_cast<unsigned long long>(e));
    }
    if (__syncthreads_or(bad_row) && threadIdx.x == 0)
        out->bad_offsets = 1;
}

} // namespace

void device_prepare(const HostCsr& g, const ocm_solve_options& opt, DeviceState& d, PrepInfo& info) {
    cudaStream_t s = d.stream;
    const std::uint32_t n = g.n;
    const std::uint64_t m = g.m;
    StagingRing& ring = StagingRing::get();
    // ---- upload
    DBuf<std::uint32_t> row, tgt;
    DBuf<double> w;
    row.alloc(std::size_t(n) + 1, s);
    tgt.alloc(std::max<std::uint64_t>(m, 1), s);
    w.alloc(std::max<std::uint64_t>(m, 1), s);
    DBuf<std::uint64_t> row64;
    if (g.index64) {
        row64.alloc(std::size_t(n) + 1, s);
        ring.copy(row64.p, g.index64, (std::size_t(n) + 1) * 8, s);
    } else {
        ring.copy(row.p, g.index32, (std::size_t(n) + 1) * 4, s);
    }
    // the weights (2/3 of the bytes) are first needed by the packing at the
    // end of the region split: they stream in on a side stream meanwhile
    cudaEvent_t w_ready = nullptr;
    // declared after w: on any exit (incl. exceptions) the side-stream copy
    // finishes before w's stream-ordered free
    struct SideGuard {
        DeviceState& d;
        ~SideGuard() {
            if (d.side)
                cudaStreamSynchronize(d.side);
        }
    } side_guard{d};
    bool exact = g.integer_exact;
    // the weights (2/3 of the bytes) are staged by a host thread of their own
    // while this one goes on to launch the region split; whoever first needs
    // them joins it (the event is recorded by then). Declared after w and
    // the side-stream guard: on any exit the thread is joined first.
    struct WeightStager {
        std::thread th;
        std::exception_ptr err;
        bool narrow = false; // the weights crossed PCIe as int32
        void join() {
            if (th.joinable())
                th.join();
            if (err) {
                auto e = err;
                err = nullptr;
                std::rethrow_exception(e);
            }
        }
        ~WeightStager() {
            if (th.joinable())
                th.join();
        }
    } wstage;
    if (m) {
        ring.copy(tgt.p, g.target, m * 4, s);
        if (!d.side) {
            CK(cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&d.side_done, cudaEventDisableTiming));
        }
        CK(cudaStreamWaitEvent(d.side, d.ev_alloc_done(s), 0)); // w allocated on s
        const int dev = d.device;
        cudaStream_t side = d.side;
        cudaEvent_t done = d.side_done;
        const int sms = d.sms;
        wstage.th = std::thread([&ring, &wstage, &w, &g, m, dev, sms, side, done] {
            try {
                CK(cudaSetDevice(dev));
                DBuf<int> wi; // freed in order on the side stream
                wi.alloc(m, side);
                if (!std::getenv("OCM_NO_NARROW") && ring.copy_narrow(wi.p, g.weight, m, side)) {
                    kp_widen_w<<<grid_for(m, sms, 8), kBlock, 0, side>>>(m, wi.p, w.p);
                    CK(cudaGetLastError());
                    wstage.narrow = true;
                } else {
                    ring.copy(w.p, g.weight, m * 8, side);
                }
                CK(cudaEventRecord(done, side));
            } catch (...) {
                wstage.err = std::current_exception();
            }
        });
        w_ready = d.side_done;
    }
    if (g.index64) {
        kp_row32<<<grid_for(n + 1, d.sms), kBlock, 0, s>>>(row64.p, row.p, std::size_t(n) + 1);
        row64.release();
    }
    int exactness = exact ? 1 : 0;
    if (!g.validated) {
        exactness = -1; // derived from the weights where they are first read
        DBuf<CsrCheck> chk;
        chk.alloc(1, s);
        auto run_check = [&](const double* wp) {
            CK(cudaMemsetAsync(chk.p, 0, sizeof(CsrCheck), s));
            CK(cudaMemsetAsync(chk.p, 0xff, 2 * sizeof(unsigned long long), s));
            kp_check_csr<<<grid_for(std::max<std::uint64_t>(m, n), d.sms, 16), kBlock, 0, s>>>(
                n, m, row.p, tgt.p, wp, chk.p);
            CK(cudaGetLastError());
            CsrCheck h{};
            CK(cudaMemcpyAsync(&h, chk.p, sizeof h, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            return h;
        };
        CsrCheck h = run_check(nullptr);
        if (h.bad_offsets)
            throw std::invalid_argument("CSR offsets are not a non-decreasing sequence from 0 to m");
        if (h.bad_target != ~0ull) {
            // report the first bad edge in id order, as build_graph's loop
            // does: a non-finite weight on an earlier edge comes first
            wstage.join();
            if (w_ready)
                CK(cudaStreamWaitEvent(s, w_ready, 0));
            h = run_check(w.p);
            if (h.bad_weight < h.bad_target)
                throw std::invalid_argument("edge " + std::to_string(h.bad_weight) +
                                            " has non-finite weight");
            throw std::invalid_argument("edge " + std::to_string(h.bad_target) +
                                        " endpoint out of range");
        }
    }
    if (std::getenv("OCM_PREP_TIMING")) {
        const auto t0 = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(s));
        std::fprintf(stderr, "{\"upload_wait_ms\": %.3f}\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    device_prepare_csr(n, m, row, tgt, w, exactness, opt, d, info, w_ready,
                       [&wstage] { wstage.join(); });
    wstage.join();
    info.h2d_bytes = (std::size_t(n) + 1) * (g.index64 ? 8 : 4) + m * (wstage.narrow ? 8 : 12);
}

void device_prepare_csr(std::uint32_t n, std::uint64_t m, DBuf<std::uint32_t>& row,
                        DBuf<std::uint32_t>& tgt, DBuf<double>& w, int exactness,
                        const ocm_solve_options& opt, DeviceState& d, PrepInfo& info,
                        cudaEvent_t w_ready, const std::function<void()>& w_host_done) {
    cudaStream_t s = d.stream;
    const int sms = d.sms;
    info.n = n;
    info.scc_off = opt.scc == OCM_SCC_OFF;
    // exactness: 1 integer weights, 0 float, -1 unknown (caller-provided
    // arrays: derived, with the non-finite check, where the weights are
    // first read)
    info.exact = exactness == 1;
    info.h2d_bytes = 0;
    const double sign = opt.objective == OCM_MAXIMIZE ? -1.0 : 1.0;
    const int gv = grid_for(n, sms);

    DBuf<PrepCounters> pcd;
    pcd.alloc(1, s);
    PrepCounters pc{};
    CK(cudaMemsetAsync(pcd.p, 0, sizeof(PrepCounters), s));
    DBuf<std::uint32_t> outd, ind;
    DBuf<std::uint8_t> self;
    outd.alloc(std::max<std::uint32_t>(n, 1), s);
    ind.alloc(std::max<std::uint32_t>(n, 1), s);
    self.alloc(std::max<std::uint32_t>(n, 1), s);
    CK(cudaMemsetAsync(ind.p, 0, std::size_t(n) * 4, s));
    kp_degrees<<<gv, kBlock, 0, s>>>(n, row.p, tgt.p, outd.p, ind.p, self.p);
    auto read_pc = [&] {
        CK(cudaMemcpyAsync(&pc, pcd.p, sizeof pc, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    };
    // weights: wait for their upload only where they are first read
    bool have_max_abs = false;
    double max_abs = 0.0;
    auto need_weights = [&] {
        if (have_max_abs)
            return;
        if (w_host_done)
            w_host_done(); // the host thread staging the weights has enqueued them
        if (w_ready)
            CK(cudaStreamWaitEvent(s, w_ready, 0));
        if (exactness < 0)
            CK(cudaMemsetAsync(&pcd.p->bad_weight_edge, 0xff, sizeof(unsigned long long), s));
        if (m)
            kp_max_abs<<<grid_for(m, sms, 16), kBlock, 0, s>>>(m, w.p, pcd.p, exactness < 0);
        read_pc();
        if (exactness < 0) {
            if (pc.bad_weight_edge != ~0ull)
                throw std::invalid_argument("edge " + std::to_string(pc.bad_weight_edge) +
                                            " has non-finite weight");
            info.exact = pc.non_integral == 0;
        }
        unsigned long long bits = pc.max_abs_bits;
        std::memcpy(&max_abs, &bits, sizeof max_abs);
        have_max_abs = true;
    };

    // Exact lane width: 32-bit weights and 64-bit keys while every weight
    // fits int32 (the session promotes itself to the wide lane if a key
    // could leave +-2^62 later), else 64-bit weights and 128-bit keys -- the
    // reference's whole ExactMode range (|w| < 2^53). Doubling sums stay
    // 64-bit, so the wide lane needs max_region * max|w| < 2^62 (the
    // reference's own int64 path sums overflow near there as well).
    // OCM_WIDE=1 forces the wide lane (tests).
    auto choose_wide = [&](double amax) {
        const char* force = std::getenv("OCM_WIDE");
        info.wide = amax > 2147483647.0 || (force && force[0] == '1');
        if (!info.wide)
            return;
        if (static_cast<long double>(amax) * info.max_region >= 4611686018427387904.0L)
            throw RangeError("exact weight sums would exceed 62 bits (max |w| x largest region)");
        const std::size_t cnt = std::max<std::uint64_t>(info.M, 1) + 2;
        d.ew_hi.alloc(cnt, s);
        CK(cudaMemsetAsync(d.ew_hi.p, 0, cnt * 4, s));
    };

    d.reg.alloc(std::max<std::uint32_t>(n, 1), s);
    // +7: the staged improvement pass copies 16-byte aligned windows of the
    // offsets and edge records (zeroed padding, never used as data)
    d.row.alloc(std::size_t(n) + 8, s);
    CK(cudaMemsetAsync(d.row.p + n + 1, 0, 7 * 4, s));

    if (info.scc_off) {
        // ---- single region: the Hamiltonian-augmented graph (solve.cpp:53)
        need_weights();
        const double big_w = 2.0 * double(n) * (max_abs + 1.0) + 1.0;
        if (!std::isfinite(big_w) || big_w >= 9007199254740992.0)
            throw std::overflow_error("hamiltonian weight too large to stay exact");
        info.no_cycle_above = max_abs;
        info.R = 1;
        info.regions_total = 1;
        info.trivial = 0;
        info.max_region = n;
        info.M = m + n;
        if (info.M >= 0xffffffffull)
            throw UnsupportedError("more than 2^32-1 edges after augmentation");
        if (info.exact) {
            d.ew.alloc(info.M + 2, s);
            CK(cudaMemsetAsync(d.ew.p + info.M, 0, 2 * sizeof(int2), s));
            choose_wide(std::max(max_abs, big_w));
        } else {
            d.fe.alloc(info.M, s);
        }
        if (info.exact)
            kp_pack_hamiltonian<true><<<grid_for(n + 1, sms), kBlock, 0, s>>>(
                n, row.p, tgt.p, w.p, sign, big_w, d.ew.p, d.ew_hi.p, nullptr, d.row.p, d.reg.p,
                pcd.p);
        else
            kp_pack_hamiltonian<false><<<grid_for(n + 1, sms), kBlock, 0, s>>>(
                n, row.p, tgt.p, w.p, sign, big_w, nullptr, nullptr, d.fe.p, d.row.p, d.reg.p, pcd.p);
        info.max_abs_w = static_cast<long long>(std::max(max_abs, big_w));
        read_pc();
        if (info.exact && pc.bad_weight)
            throw std::logic_error("weight packing: a weight outside the chosen lane's range");
        return;
    }

    // ---- backward CSR (no self-loops)
    const auto t_scc = std::chrono::steady_clock::now();
    // OCM_PREP_TIMING: per-step wall times of the region split (syncs the
    // stream at each mark; diagnostics only)
    static const bool timing = std::getenv("OCM_PREP_TIMING") != nullptr;
    std::string tmarks;
    auto t_last = t_scc;
    auto mark = [&](const char* what) {
        if (!timing)
            return;
        CK(cudaStreamSynchronize(s));
        const auto t = std::chrono::steady_clock::now();
        char buf[96];
        std::snprintf(buf, sizeof buf, "%s\"%s\": %.3f", tmarks.empty() ? "" : ", ", what,
                      std::chrono::duration<double, std::milli>(t - t_last).count());
        tmarks += buf;
        t_last = t;
    };
    DBuf<std::uint32_t> brow, bsrc, cursor;
    brow.alloc(std::size_t(n) + 1, s);
    CK(cudaMemsetAsync(brow.p + n, 0, 4, s));
    // brow[0..n] = exclusive scan of ind (ind[n] treated as 0 via n+1 scan)
    {
        DBuf<std::uint32_t> ind1;
        ind1.alloc(std::size_t(n) + 1, s);
        CK(cudaMemsetAsync(ind1.p + n, 0, 4, s));
        CK(cudaMemcpyAsync(ind1.p, ind.p, std::size_t(n) * 4, cudaMemcpyDeviceToDevice, s));
        exclusive_scan(ind1.p, brow.p, std::size_t(n) + 1, s);
    }
    // sized by m (an upper bound: self-loops are left out) instead of a
    // host read of brow[n]
    bsrc.alloc(std::max<std::uint64_t>(m, 1), s);
    cursor.alloc(std::max<std::uint32_t>(n, 1), s);
    CK(cudaMemcpyAsync(cursor.p, brow.p, std::size_t(n) * 4, cudaMemcpyDeviceToDevice, s));
    kp_bwd_fill<<<gv, kBlock, 0, s>>>(n, row.p, tgt.p, cursor.p, bsrc.p);
    cursor.release();
    mark("bwd_csr");

    // ---- SCC
    DBuf<std::uint32_t> lab, q0, q1, visf, visb, aux;
    lab.alloc(std::max<std::uint32_t>(n, 1), s);
    q0.alloc(std::max<std::uint32_t>(n, 1), s);
    q1.alloc(std::max<std::uint32_t>(n, 1), s);
    visf.alloc(std::max<std::uint32_t>(n, 1), s);
    visb.alloc(std::max<std::uint32_t>(n, 1), s);
    CK(cudaMemsetAsync(lab.p, 0xff, std::size_t(n) * 4, s));
    CK(cudaMemsetAsync(visf.p, 0, std::size_t(n) * 4, s));
    CK(cudaMemsetAsync(visb.p, 0, std::size_t(n) * 4, s));
    std::uint32_t stamp = 0;

    auto trim = [&] {
        static int trim_per_sm = 0;
        if (!trim_per_sm) {
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&trim_per_sm, kp_trim_coop, kBlock, 0));
            trim_per_sm = std::max(1, std::min(trim_per_sm, 8));
        }
        std::uint32_t nn = n;
        const std::uint32_t *r = row.p, *t = tgt.p, *br = brow.p, *bs = bsrc.p;
        std::uint32_t *ip = ind.p, *op = outd.p, *lp = lab.p, *a0 = q0.p, *a1 = q1.p;
        unsigned long long* rc = pcd.p->bfs_ring;
        void* args[] = {&nn, &r, &t, &br, &bs, &ip, &op, &lp, &a0, &a1, &rc};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&kp_trim_coop),
                                       dim3(std::min(trim_per_sm * sms, grid_for(n, sms, 8))),
                                       dim3(kBlock), args, 0, s));
    };
    auto remaining = [&] {
        CK(cudaMemsetAsync(&pcd.p->remaining, 0, 4, s));
        kp_recount<<<gv, kBlock, 0, s>>>(n, row.p, tgt.p, brow.p, bsrc.p, lab.p, ind.p, outd.p, pcd.p);
        read_pc();
        return pc.remaining;
    };
    // trimming, pivot, both reachability searches and the pivot's component
    // in one cooperative launch
    {
        static int scc_per_sm = 0; // cooperative occupancy of kp_scc_coop
        if (!scc_per_sm) {
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&scc_per_sm, kp_scc_coop, kBlock, 0));
            scc_per_sm = std::max(1, std::min(scc_per_sm, 8));
        }
        DBuf<std::uint32_t> qb0, qb1; // backward-search frontiers
        qb0.alloc(std::max<std::uint32_t>(n, 1), s);
        qb1.alloc(std::max<std::uint32_t>(n, 1), s);
        CK(cudaMemsetAsync(&pcd.p->pivot, 0, 8, s));
        std::uint32_t nn = n;
        const std::uint32_t *r = row.p, *c = tgt.p, *br = brow.p, *bc = bsrc.p;
        std::uint32_t *ip = ind.p, *op = outd.p, *lp = lab.p, *vf = visf.p, *vb = visb.p, *f0 = q0.p,
                      *f1 = q1.p, *b0 = qb0.p, *b1 = qb1.p;
        PrepCounters* pp = pcd.p;
        void* args[] = {&nn, &r, &c, &br, &bc, &ip, &op, &lp, &vf, &vb, &f0, &f1, &b0, &b1, &pp};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&kp_scc_coop),
                                       dim3(std::min(scc_per_sm * sms, grid_for(n, sms, 8))), dim3(kBlock),
                                       args, 0, s));
        qb0.release();
        qb1.release();
    }
    read_pc();
    mark("trim_bfs");
    if (timing)
        std::fprintf(stderr, "{\"scc_coop_Mclk\": [%.2f, %.2f, %.2f, %.2f], \"levels\": %u}\n", pc.clk[0] * 1e-6,
                     pc.clk[1] * 1e-6, pc.clk[2] * 1e-6, pc.clk[3] * 1e-6, pc.levels);
    if (pc.remaining) {
        // visf holds BFS levels: clear it for the colouring's stamps
        CK(cudaMemsetAsync(visf.p, 0, std::size_t(n) * 4, s));
        // finish the rest by colouring, re-trimming between rounds
        for (;;) {
            if (!remaining())
                break;
            trim();
            if (!remaining())
                break;
            aux.alloc(std::max<std::uint32_t>(n, 1), s); // colours
            kp_color_init<<<gv, kBlock, 0, s>>>(n, lab.p, aux.p);
            do {
                CK(cudaMemsetAsync(&pcd.p->changed, 0, 4, s));
                kp_color_prop<<<gv, kBlock, 0, s>>>(n, brow.p, bsrc.p, lab.p, aux.p, pcd.p);
                read_pc();
            } while (pc.changed);
            const std::uint32_t sc = ++stamp;
            kp_color_roots<<<gv, kBlock, 0, s>>>(n, lab.p, aux.p, visf.p, sc);
            do {
                CK(cudaMemsetAsync(&pcd.p->changed, 0, 4, s));
                kp_color_close<<<gv, kBlock, 0, s>>>(n, row.p, tgt.p, lab.p, aux.p, visf.p, sc, pcd.p);
                read_pc();
            } while (pc.changed);
            kp_color_assign<<<gv, kBlock, 0, s>>>(n, aux.p, visf.p, sc, lab.p);
        }
    }
    brow.release();
    bsrc.release();
    q0.release();
    q1.release();
    visb.release();

    // ---- regions: sizes, non-trivial flags, dense ids
    DBuf<std::uint32_t>& size = visf; // reuse
    CK(cudaMemsetAsync(size.p, 0, std::size_t(n) * 4, s));
    mark("rest");
    kp_sizes<<<gv, kBlock, 0, s>>>(n, lab.p, size.p);
    DBuf<std::uint32_t> flag, rid;
    flag.alloc(std::size_t(n) + 1, s);
    rid.alloc(std::size_t(n) + 1, s);
    CK(cudaMemsetAsync(flag.p + n, 0, 4, s));
    kp_nontrivial<<<gv, kBlock, 0, s>>>(n, lab.p, size.p, self.p, flag.p, pcd.p);
    exclusive_scan(flag.p, rid.p, std::size_t(n) + 1, s);
    CK(cudaMemcpyAsync(&pcd.p->R, rid.p + n, 4, cudaMemcpyDeviceToDevice, s));
    read_pc();
    const std::uint32_t R = pc.R;
    info.R = R;
    info.regions_total = pc.regions_total;
    info.trivial = pc.regions_total - R;
    info.max_region = pc.max_region;
    kp_region_ids<<<gv, kBlock, 0, s>>>(n, lab.p, flag.p, rid.p, R, d.reg.p);
    info.scc_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_scc).count();
    const auto t_pack = std::chrono::steady_clock::now();

    // ---- intra-region CSR
    DBuf<std::uint32_t>& cnt = rid; // reuse (n+1)
    mark("regions");
    kp_count_intra<<<gv, kBlock, 0, s>>>(n, R, row.p, tgt.p, d.reg.p, cnt.p);
    CK(cudaMemsetAsync(cnt.p + n, 0, 4, s));
    exclusive_scan(cnt.p, d.row.p, std::size_t(n) + 1, s);
    std::uint32_t M = 0; // stream-ordered read (the session stream does not sync with stream 0)
    CK(cudaMemcpyAsync(&M, d.row.p + n, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    info.M = M;
    need_weights();
    if (info.exact) {
        d.ew.alloc(std::size_t(M) + 2, s);
        CK(cudaMemsetAsync(d.ew.p + M, 0, 2 * sizeof(int2), s));
        choose_wide(max_abs);
    } else {
        d.fe.alloc(std::max<std::uint32_t>(M, 1), s);
    }
    CK(cudaMemsetAsync(&pcd.p->bad_weight, 0, 4, s));
    if (info.exact)
        kp_pack<true><<<gv, kBlock, 0, s>>>(n, R, row.p, tgt.p, w.p, d.reg.p, d.row.p, sign, d.ew.p,
                                            d.ew_hi.p, nullptr, pcd.p);
    else
        kp_pack<false><<<gv, kBlock, 0, s>>>(n, R, row.p, tgt.p, w.p, d.reg.p, d.row.p, sign,
                                             nullptr, nullptr, d.fe.p, pcd.p);
    read_pc();
    if (info.exact && pc.bad_weight)
        throw std::logic_error("weight packing: a weight outside the chosen lane's range");
    info.max_abs_w = static_cast<long long>(max_abs);
    mark("pack");
    if (std::getenv("OCM_PREP_TIMING"))
        std::fprintf(stderr, "{%s}\n{\"scc_ms\": %.3f, \"pack_ms\": %.3f, \"R\": %u}\n", tmarks.c_str(), info.scc_ms,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_pack).count(),
                     R);
}

} // namespace ocmb
