// The persistent policy-iteration kernel (included by solver.cu only).
//
// One cooperative launch runs a whole solve: every Howard iteration of
// proj/include/ocm/howard_par.hpp:544 run() with its kernels as phases of
// one grid, separated by grid-wide barriers. The host only launches and
// reads the result; convergence, the doubling round count, the winning-cycle
// round count and the re-attachment layers are all decided on the device.
//
//   phase                    replaces (howard_par.hpp)
//   improve                  :146 spf_pass_iter (+ policy in-degree count)
//   classify                 :189 finished_regions / :208 deactivate_regions,
//                            leaf/core split + first doubling round
//   rounds (2 steps/pass),   :249 elimination_fixpoint + :301 cycle_identification
//   last round + mark, check (exact round-count verification), :319 records
//   vote (block 0 when few   :56 vote_min, :339 vote_and_adopt,
//     cycle vertices; adopt, :494 value_propagate_fixpoint on the cycle
//     winning-cycle values)
//   keep                     :370 set_min_cycle, :393 mark_min_component,
//                            value propagation of kept vertices
//   attach layers            :433 connect_gpi_fixpoint (+ values)
//   float levels             :494 value_propagate_fixpoint (float lane)
//
// Cycle detection is leaves-then-double: the leaves of the functional policy
// graph (in-degree 0: never on a cycle, never anyone's successor; ~46% of the
// vertices on the benchmark graphs) are split off, the remaining core (closed
// under succ) is pointer-doubled, and leaves take anchor and value from their
// (core) successor in the keep pass.
//
// Parity: every phase computes the same function as the reference step it
// replaces; the policy, anchors, lambdas, integer keys and
// iteration counts are pinned against the reference bit for bit by the GPU
// parity suite.
//
// Memory model: arrays written inside the kernel are read with plain or
// L1-bypassing loads (never __ldg); only the CSR (row, ew, fe) and region
// ids are read-only for the whole launch. cooperative_groups grid.sync()
// orders all global memory between phases.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "coop.cuh"
#include "devcommon.cuh"

namespace ocmb {
namespace {

namespace cg = cooperative_groups;

#ifndef OCM_MINB
#define OCM_MINB 4
#endif
constexpr int kSolveMinBlocks = OCM_MINB; // 4: register cap 64 at 256 threads
#ifndef OCM_HOIST_DEN
#define OCM_HOIST_DEN 1
#endif
#ifndef OCM_KSHRINK
#define OCM_KSHRINK 2
#endif
// consecutive first-try verifications before the doubling depth is tried one
// step shallower
constexpr unsigned kKShrink = OCM_KSHRINK;

// Policy in-degree is only ever tested for zero (leaf split). OCM_PRED_FLAG
// selects how a vertex records that it has a predecessor:
//   0  atomic u32 counter (round 1), reset per core vertex in keep;
//   1  byte flag, plain store, reset per core vertex in keep;
//   2  bit in a packed bitmap (N/8 bytes: L2-resident even at 2.5*10^8
//      vertices), atomicOr, whole bitmap cleared by keep;
//   3  as 2, but the bit is read first and the atomic skipped when set
//      (hub targets).
#ifndef OCM_PRED_FLAG
#define OCM_PRED_FLAG 2
#endif
__device__ __forceinline__ void mark_pred(const KP& p, std::uint32_t t) {
#if OCM_PRED_FLAG == 0
    atomicAdd(&p.indeg[t], 1u);
#elif OCM_PRED_FLAG == 1
    reinterpret_cast<unsigned char*>(p.indeg)[t] = 1;
#else
    const unsigned bit = 1u << (t & 31);
#if OCM_PRED_FLAG == 3
    if (ldv(p.indeg[t >> 5]) & bit)
        return;
#endif
    atomicOr(&p.indeg[t >> 5], bit);
#endif
}
__device__ __forceinline__ bool has_pred(const KP& p, std::uint32_t v) {
#if OCM_PRED_FLAG == 0
    return p.indeg[v] != 0;
#elif OCM_PRED_FLAG == 1
    return reinterpret_cast<const unsigned char*>(p.indeg)[v] != 0;
#else
    return (p.indeg[v >> 5] >> (v & 31)) & 1u;
#endif
}
// per core vertex in keep (modes 0, 1)
__device__ __forceinline__ void clear_pred(const KP& p, std::uint32_t v) {
#if OCM_PRED_FLAG == 0
    p.indeg[v] = 0;
#elif OCM_PRED_FLAG == 1
    reinterpret_cast<unsigned char*>(p.indeg)[v] = 0;
#else
    (void)p;
    (void)v;
#endif
}
// whole-array clear in keep (modes 2, 3)
__device__ __forceinline__ void clear_pred_all(const KP& p) {
#if OCM_PRED_FLAG >= 2
    for (std::size_t w = gtid(); w < (std::size_t(p.N) + 31) / 32; w += gstride())
        p.indeg[w] = 0;
#else
    (void)p;
#endif
}

// Connected-vertex bitmap (OCM_CBITS=1, default): bit v is set once v is
// connected to its region's winning cycle (kept, or attached in a layer).
// Attach tests an edge's head with one bit of this N/8-byte array -- L2-
// resident even at 2.5*10^8 vertices -- instead of a 4-byte gather of conn[]
// from HBM, and confirms only set bits against conn[] (a head attached in
// the current layer has its bit set but conn == layer). Cleared by classify.
// Used when conn[] outgrows L2 (p.cbits != null: N >= 2^24 by default,
// OCM_CBITS_MIN_N): -10% per solve at configs 4 and 5, +4% at config 2,
// where conn[] is L2-resident and keep's extra atomics cost more than
// attach saves (profiles/r02/ab_cbits_r02.log).
#ifndef OCM_CBITS
#define OCM_CBITS 1
#endif
__device__ __forceinline__ void cbit_set(const KP& p, std::uint32_t v, bool on) {
    // one atomicOr per bitmap word per warp
    const unsigned act = __activemask();
    const unsigned want = __ballot_sync(act, on);
    if (!on)
        return;
    const unsigned peers = __match_any_sync(want, v >> 5);
    const unsigned bits = __reduce_or_sync(peers, 1u << (v & 31));
    if (static_cast<unsigned>(__ffs(peers) - 1) == (threadIdx.x & 31))
        atomicOr(&p.cbits[v >> 5], bits);
}

// ------------------------------------------------------------ modes
//
// Arithmetic mode of a k_solve instantiation (template parameter MODE):
//   0  FloatMode (policy.hpp) in doubles;
//   1  ExactMode with 64-bit keys K = value*den and 32-bit edge weights --
//      the fast lane, used while every key provably stays inside +-2^62;
//   2  ExactMode "wide": 128-bit keys and 64-bit weights (the low half in
//      the int2 edge record, the high half in ew_hi / succ_whi), covering
//      the reference's whole exact range (integral |w| < 2^53, graph.cpp:15,
//      compared as (wsum, steps) with 128-bit products, policy.hpp:71-79).
template <int MODE> struct ModeT;
template <> struct ModeT<0> { using Key = double; };
template <> struct ModeT<1> { using Key = long long; };
template <> struct ModeT<2> { using Key = __int128; };
template <int MODE> using KeyT = typename ModeT<MODE>::Key;

template <int MODE> __device__ __forceinline__ KeyT<MODE> key_ld(const KP& p, std::uint32_t v) {
    if constexpr (MODE == 0)
        return p.key_f[v];
    else if constexpr (MODE == 1)
        return p.key_i[v];
    else
        return p.key_w[v];
}
// key gather for the improvement pass (L2, bypassing L1)
template <int MODE> __device__ __forceinline__ KeyT<MODE> key_gather(const KP& p, std::uint32_t v) {
    if constexpr (MODE == 0)
        return __ldcg(&p.key_f[v]);
    else if constexpr (MODE == 1)
        return __ldcg(&p.key_i[v]);
    else {
        const longlong2 x = __ldcg(reinterpret_cast<const longlong2*>(p.key_w) + v);
        return (static_cast<__int128>(x.y) << 64) | static_cast<unsigned long long>(x.x);
    }
}
template <int MODE> __device__ __forceinline__ void key_st(const KP& p, std::uint32_t v, KeyT<MODE> k) {
    if constexpr (MODE == 0)
        p.key_f[v] = k;
    else if constexpr (MODE == 1)
        p.key_i[v] = k;
    else
        p.key_w[v] = k;
}
// exact weight of edge e (its int2 record ed)
template <int MODE> __device__ __forceinline__ long long edge_w(const KP& p, std::uint32_t e, int2 ed) {
    if constexpr (MODE == 2)
        return (static_cast<long long>(__ldg(&p.ew_hi[e])) << 32) | static_cast<unsigned>(ed.y);
    else
        return ed.y;
}
// exact weight of v's policy edge
template <int MODE> __device__ __forceinline__ long long succ_w(const KP& p, std::uint32_t v) {
    if constexpr (MODE == 2)
        return (static_cast<long long>(p.succ_whi[v]) << 32) | static_cast<unsigned>(p.succ_wi[v]);
    else
        return p.succ_wi[v];
}
// policy weight of v whose new head is t; the fast exact lane also keeps the
// packed {head, weight} shadow the leaf split reads at random (one sector
// instead of two)
template <int MODE>
__device__ __forceinline__ void succ_w_st(const KP& p, std::uint32_t v, std::uint32_t t, long long w) {
    p.succ_wi[v] = static_cast<int>(w);
    if constexpr (MODE == 2)
        p.succ_whi[v] = static_cast<int>(w >> 32);
    if constexpr (MODE == 1)
        if (p.succ_vw)
            p.succ_vw[v] = make_int2(static_cast<int>(t), static_cast<int>(w));
}
// keys are proven to stay inside this bound at every adoption
template <int MODE> __device__ __forceinline__ bool key_in_range(__int128 k) {
    const __int128 lim = static_cast<__int128>(1) << (MODE == 2 ? 120 : 62);
    return k < lim && k > -lim;
}
__device__ __forceinline__ long long shfl_key(unsigned m, long long x, int off, int w) {
    return __shfl_xor_sync(m, x, off, w);
}
__device__ __forceinline__ double shfl_key(unsigned m, double x, int off, int w) {
    return __shfl_xor_sync(m, x, off, w);
}
__device__ __forceinline__ __int128 shfl_key(unsigned m, __int128 x, int off, int w) {
    const long long lo = __shfl_xor_sync(m, static_cast<long long>(static_cast<unsigned long long>(x)), off, w);
    const long long hi = __shfl_xor_sync(m, static_cast<long long>(x >> 64), off, w);
    return (static_cast<__int128>(hi) << 64) | static_cast<unsigned long long>(lo);
}

// ------------------------------------------------------------ improvement
//
// howard_par.hpp:146 spf_pass_iter / howard.hpp:63 improve_policy.
// G lanes cooperate on one vertex and each lane keeps U edges in flight:
// lane j streams edges row[v]+j, +G, ... (8-byte {target, weight} records),
// gathers the U target keys together, and the group reduces the
// lexicographic minimum (candidate, edge id) -- exactly the sequential
// "first strictly smaller" scan. The incumbent's candidate is picked up on
// the way (the incumbent is one of v's edges), so the replacement test costs
// no extra gather; the lane owning the winning edge writes the new policy.
// Every processed vertex also adds 1 to the in-degree of its (new or kept)
// successor for the peeling that follows.

template <int G> __device__ __forceinline__ unsigned group_mask() {
    if constexpr (G == 32)
        return FULL;
    else
        return ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
}

// Raise region r's "changed" flag; in the fused sharded lane the peers'
// replicas of the flag too (stored during the pass, ordered before the
// cross-rank arrival by the same system fence as the policy pushes).
__device__ __forceinline__ void raise_changed(const KP& p, int* changed, std::uint32_t r) {
    set_once(&changed[r], 1);
    if (p.fused) {
        const int par = changed == p.changed[1] ? 1 : 0;
        for (int q = 0; q < p.world; ++q)
            if (q != p.rank)
                p.peer_changed[par][q][r] = 1;
    }
}

// Region "changed" bookkeeping with at most one store per block per region.
struct ChangedMarks {
    std::uint32_t first = NONE;
    std::uint32_t last_direct = NONE;
    __device__ __forceinline__ void note(const KP& p, int* changed, std::uint32_t r) {
        if (first == NONE)
            first = r;
        else if (r != first && r != last_direct) {
            last_direct = r;
            raise_changed(p, changed, r);
        }
    }
    __device__ __forceinline__ void flush(const KP& p, int* changed) {
        __shared__ std::uint32_t s_r;
        if (threadIdx.x == 0)
            s_r = NONE;
        __syncthreads();
        if (first != NONE) {
            const std::uint32_t prev = atomicCAS(&s_r, NONE, first);
            if (prev != NONE && prev != first)
                raise_changed(p, changed, first);
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_r != NONE)
            raise_changed(p, changed, s_r);
    }
};

// Read-only 8/16-byte edge records through the non-coherent path (an
// evict-first L2 policy on this stream measured no gain: the phases after
// the improvement pass are bound by random-sector throughput, not capacity).
__device__ __forceinline__ int2 ld_edge(const int2* e) { return __ldg(e); }
__device__ __forceinline__ FEdge ld_edge(const FEdge* e) {
    const double2 raw = __ldg(reinterpret_cast<const double2*>(e));
    FEdge f;
    f.w = raw.x;
    f.t = static_cast<std::uint32_t>(__double_as_longlong(raw.y));
    f.pad = 0;
    return f;
}

// Fused sharded lane: a vertex whose policy changed is stored straight into
// every peer's replica (NVLink stores into peer memory; ordered before the
// cross-rank barrier by a system-scope fence). Unchanged vertices are
// already identical everywhere, so only changes travel.
template <int MODE, class Edge>
__device__ __forceinline__ void push_policy(const KP& p, std::uint32_t v, std::uint32_t e,
                                            std::uint32_t t, const Edge& ed) {
    constexpr bool EXACT = MODE != 0;
    for (int q = 0; q < p.world; ++q) {
        if (q == p.rank)
            continue;
        p.peer_succ_e[q][v] = e;
        p.peer_succ_v[q][v] = t;
        if constexpr (EXACT)
            static_cast<int*>(p.peer_succ_w[q])[v] = reinterpret_cast<const int2&>(ed).y;
        else
            static_cast<double*>(p.peer_succ_w[q])[v] = reinterpret_cast<const FEdge&>(ed).w;
    }
}

// Hub keys staged in shared memory (north_star item 5): every CTA copies the
// keys of the graph's highest in-degree vertices into an open-addressed
// table {vertex, key} at the start of the pass (the keys do not change
// during it); an edge into a hub reads its key there instead of gathering
// it from L2/HBM, where every SM would hit the same few sectors.
constexpr int kHotProbe = 4;
// table layout in dynamic shared memory: slots x i64 key, then slots x u32
// vertex (NONE = empty); slots = 2^(32 - p.hot_shift). Addressed from the
// kernel parameters so the pass keeps no extra live registers.
extern __shared__ __align__(16) unsigned char dyn_smem[];
__device__ __forceinline__ unsigned hot_hash(std::uint32_t t, unsigned shift) {
    return (t * 2654435761u) >> shift;
}
__device__ __forceinline__ long long* hot_keys() { return reinterpret_cast<long long*>(dyn_smem); }
__device__ __forceinline__ std::uint32_t* hot_verts(const KP& p) {
    return reinterpret_cast<std::uint32_t*>(dyn_smem + (std::size_t(8) << (32 - p.hot_shift)));
}
__device__ __forceinline__ bool hot_find(const KP& p, std::uint32_t t, long long& key) {
    const unsigned mask = (1u << (32 - p.hot_shift)) - 1u;
    const std::uint32_t* hv = hot_verts(p);
    unsigned i = hot_hash(t, p.hot_shift);
#pragma unroll
    for (int j = 0; j < kHotProbe; ++j) {
        const std::uint32_t x = hv[i];
        if (x == t) {
            key = hot_keys()[i];
            return true;
        }
        if (x == NONE)
            return false;
        i = (i + 1) & mask;
    }
    return false;
}

// STAGED: the vertex's row offsets and edges were copied into shared memory
// by the bulk-TMA producer of improve_staged (exact lane); sedge[i] holds
// edge ebase + i, and b / e_end are the vertex's offsets read from there.
template <int MODE, int G, int U, bool HOT, bool STAGED = false>
__device__ __forceinline__ void improve_vertex(const KP& p, int* changed, ChangedMarks& marks,
                                               std::uint32_t v, long long den1,
                                               const int2* sedge = nullptr,
                                               std::uint32_t ebase = 0, std::uint32_t sb = 0,
                                               std::uint32_t se = 0) {
    // Register budget matters here (64 at 4 CTAs/SM): edges stay packed as
    // they were loaded, the winner's head and weight are re-read (an L1 hit)
    // only when the policy changes, and the exact candidate drops the
    // per-vertex constant -num (compares are offset-invariant in integers).
    constexpr bool EXACT = MODE != 0;
    const unsigned lane = threadIdx.x & (G - 1);
    const unsigned gm = group_mask<G>();
    using Key = KeyT<MODE>;
    using Edge = typename std::conditional<EXACT, int2, FEdge>::type;
    const Edge* __restrict__ edges = EXACT ? reinterpret_cast<const Edge*>(p.ew)
                                           : reinterpret_cast<const Edge*>(p.fe);
    // one non-trivial region (the common case): no per-vertex region
    // lookup -- trivial vertices are exactly those with no intra-region edge
    const std::uint32_t r = p.R == 1 ? 0u : __ldg(&p.reg[v]);
    if (p.R != 1 && !p.active[r])
        return;
    std::uint32_t b, e_end;
    if constexpr (STAGED) {
        b = sb;
        e_end = se;
    } else {
        b = __ldg(&p.row[v]);
        e_end = __ldg(&p.row[v + 1]);
    }
    if (e_end == b || e_end - b >= p.heavy_deg)
        return; // trivial, or the block-cooperative path (improve_heavy)
    auto edge_at = [&](std::uint32_t e) -> Edge {
        if constexpr (STAGED)
            return reinterpret_cast<const Edge*>(sedge)[e - ebase];
        else
            return ld_edge(&edges[e]);
    };
    const std::uint32_t cur = p.succ_e[v];
    long long den = 1;
    double lam = 0.0;
    if constexpr (EXACT)
        den = OCM_HOIST_DEN && p.R == 1 ? den1 : p.lam_den[r]; // den1: region 0's, read once
    else
        lam = p.lam_f[r];
    Key best = 0, curc = 0;
    std::uint32_t be = NONE;
    bool have_cur = false;
    for (std::uint32_t e0 = b + lane; e0 < e_end; e0 += G * U) {
        Edge ed[U];
        Key kk[U];
        // unconditional loads at a clamped edge id (always a valid edge of
        // v; the tail is masked below): predicated array writes would send
        // ed[]/kk[] to local memory
#pragma unroll
        for (int u = 0; u < U; ++u)
            ed[u] = edge_at(min(e0 + u * G, e_end - 1));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            std::uint32_t t;
            if constexpr (EXACT)
                t = static_cast<std::uint32_t>(ed[u].x);
            else
                t = ed[u].t;
            if constexpr (MODE == 1 && HOT) {
                long long hk;
                if (hot_find(p, t, hk))
                    kk[u] = hk;
                else
                    kk[u] = key_gather<MODE>(p, t);
            } else {
                kk[u] = key_gather<MODE>(p, t);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const std::uint32_t e = e0 + u * G;
            if (e < e_end) {
                Key c;
                if constexpr (MODE == 2)
                    c = kk[u] + static_cast<Key>(edge_w<MODE>(p, e, ed[u])) * den; // + const -num
                else if constexpr (EXACT)
                    c = kk[u] + static_cast<long long>(ed[u].y) * den; // + const -num
                else
                    c = (kk[u] + ed[u].w) - lam; // FloatMode::extend (policy.hpp:105)
                if (be == NONE || c < best) {
                    best = c;
                    be = e;
                }
                if (e == cur) {
                    curc = c;
                    have_cur = true;
                }
            }
        }
    }
    const bool saw_cur = have_cur; // this lane scanned the incumbent edge
    Key gbest = best;
    std::uint32_t gbe = be;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        const Key ob = shfl_key(gm, gbest, off, G);
        const std::uint32_t oe = __shfl_xor_sync(gm, gbe, off, G);
        if (oe != NONE && (gbe == NONE || ob < gbest || (ob == gbest && oe < gbe))) {
            gbest = ob;
            gbe = oe;
        }
        const Key oc = shfl_key(gm, curc, off, G);
        const bool oh = __shfl_xor_sync(gm, have_cur ? 1 : 0, off, G) != 0;
        if (oh) {
            curc = oc;
            have_cur = true;
        }
    }
    if (gbe == NONE) {
        if (lane == 0)
            p.c->error = 1;
        return;
    }
    bool rep = cur == NONE;
    if (!rep) {
        if constexpr (EXACT) {
            rep = gbest < curc;
        } else { // FloatMode::strictly_better (policy.hpp:116)
            const double tol = 1e-9 * fmax(1.0, fmax(fabs(gbest), fabs(curc)));
            rep = gbest < curc - tol;
        }
    }
    if (rep) {
        if (gbe == be) { // owner lane of the winning edge
            const Edge ed = edge_at(be);
            p.succ_e[v] = be;
            std::uint32_t t;
            if constexpr (EXACT) {
                t = static_cast<std::uint32_t>(ed.x);
                succ_w_st<MODE>(p, v, t, edge_w<MODE>(p, be, ed));
            } else {
                t = ed.t;
                p.succ_wf[v] = ed.w;
            }
            p.succ_v[v] = t;
            if (p.fused)
                push_policy<MODE>(p, v, be, t, ed);
            if (p.indeg_in_improve)
                mark_pred(p, t);
            marks.note(p, changed, r);
        }
    } else if (saw_cur && p.indeg_in_improve) {
        std::uint32_t t;
        if constexpr (EXACT)
            t = static_cast<std::uint32_t>(edge_at(cur).x);
        else
            t = edge_at(cur).t;
        mark_pred(p, t);
    }
}

// Heavy vertices (intra-region degree >= heavy_deg, listed at session
// creation): one block per vertex, 256 threads striding its edges, then a
// block-wide lexicographic (candidate, edge id) reduction -- the same
// "first strictly smaller" result as the sequential scan.
template <int MODE>
__device__ __forceinline__ void improve_heavy(const KP& p, int* changed) {
    constexpr bool EXACT = MODE != 0;
    using Key = KeyT<MODE>;
    __shared__ Key s_best[kBlock / 32];
    __shared__ std::uint32_t s_be[kBlock / 32];
    __shared__ Key s_cur;
    __shared__ int s_have_cur;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (std::uint32_t h = blockIdx.x; h < p.nheavy; h += gridDim.x) {
        const std::uint32_t v = p.heavy[h];
        const std::uint32_t r = __ldg(&p.reg[v]);
        if (!p.active[r] || v < p.own_lo || v >= p.own_hi)
            continue; // block-uniform
        const std::uint32_t b = __ldg(&p.row[v]), e_end = __ldg(&p.row[v + 1]);
        const std::uint32_t cur = p.succ_e[v];
        long long num = 0, den = 1;
        double lam = 0.0;
        if constexpr (EXACT) {
            num = p.lam_num[r];
            den = p.lam_den[r];
        } else {
            lam = p.lam_f[r];
        }
        if (threadIdx.x == 0)
            s_have_cur = 0;
        __syncthreads();
        Key best = 0;
        std::uint32_t be = NONE;
        for (std::uint32_t e0 = b + threadIdx.x; e0 < e_end; e0 += 4 * kBlock) {
            std::uint32_t tt[4];
            Key kk[4];
            long long wi[4];
            double wf[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const std::uint32_t e = min(e0 + u * kBlock, e_end - 1); // tail masked below
                if constexpr (EXACT) {
                    const int2 ed = __ldg(&p.ew[e]);
                    tt[u] = static_cast<std::uint32_t>(ed.x);
                    wi[u] = edge_w<MODE>(p, e, ed);
                } else {
                    const FEdge ed = ld_edge(&p.fe[e]);
                    tt[u] = ed.t;
                    wf[u] = ed.w;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                kk[u] = key_gather<MODE>(p, tt[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const std::uint32_t e = e0 + u * kBlock;
                if (e < e_end) {
                    Key c;
                    if constexpr (EXACT)
                        c = kk[u] + static_cast<Key>(wi[u]) * den - num;
                    else
                        c = (kk[u] + wf[u]) - lam;
                    if (be == NONE || c < best) { // ascending e per thread: first wins ties
                        best = c;
                        be = e;
                    }
                    if (e == cur) {
                        s_cur = c;
                        s_have_cur = 1;
                    }
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const Key ob = shfl_key(FULL, best, off, 32);
            const std::uint32_t oe = __shfl_xor_sync(FULL, be, off);
            if (oe != NONE && (be == NONE || ob < best || (ob == best && oe < be))) {
                best = ob;
                be = oe;
            }
        }
        if (lane == 0) {
            s_best[warp] = best;
            s_be[warp] = be;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            Key gb = s_best[0];
            std::uint32_t ge = s_be[0];
            for (int w = 1; w < kBlock / 32; ++w) {
                const std::uint32_t oe = s_be[w];
                if (oe != NONE && (ge == NONE || s_best[w] < gb || (s_best[w] == gb && oe < ge))) {
                    gb = s_best[w];
                    ge = oe;
                }
            }
            if (ge == NONE) {
                p.c->error = 1;
            } else {
                bool rep = cur == NONE || !s_have_cur;
                if (!rep) {
                    const Key curc = s_cur;
                    if constexpr (EXACT) {
                        rep = gb < curc;
                    } else {
                        const double tol = 1e-9 * fmax(1.0, fmax(fabs(gb), fabs(curc)));
                        rep = gb < curc - tol;
                    }
                }
                if (rep) {
                    p.succ_e[v] = ge;
                    if constexpr (EXACT) {
                        const int2 ed = __ldg(&p.ew[ge]);
                        p.succ_v[v] = static_cast<std::uint32_t>(ed.x);
                        succ_w_st<MODE>(p, v, static_cast<std::uint32_t>(ed.x), edge_w<MODE>(p, ge, ed));
                        if (p.fused)
                            push_policy<MODE>(p, v, ge, static_cast<std::uint32_t>(ed.x), ed);
                        if (p.indeg_in_improve)
                            mark_pred(p, ed.x);
                    } else {
                        const FEdge ed = ld_edge(&p.fe[ge]);
                        p.succ_v[v] = ed.t;
                        p.succ_wf[v] = ed.w;
                        if (p.fused)
                            push_policy<MODE>(p, v, ge, ed.t, ed);
                        if (p.indeg_in_improve)
                            mark_pred(p, ed.t);
                    }
                    raise_changed(p, changed, r);
                } else if (p.indeg_in_improve) {
                    mark_pred(p, p.succ_v[v]);
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------- propagation-blocked improvement
//
// Exact lane, key arrays too large for L2: a random 8-byte
// key gather per edge from HBM runs at ~40 G/s on B200, from L2 at ~210 G/s.
// The edges are kept a second time ordered by target bin (pb_nb bins of
// pb_bin vertices, a bin's keys ~16 MB) and in CSR order inside a bin, so
//   pass 1 streams the bin-ordered {target, weight} records in order -- at any
//          moment the grid gathers keys from one bin, which L2 holds -- and
//          streams each candidate key[t] + w*den out (the per-vertex -num
//          is dropped, as in improve_vertex);
//   pass 2 takes vertex blocks of pb_vb vertices: a block's candidates are
//          one contiguous segment per bin (pb_off), reduced to the
//          lexicographic minimum (candidate, edge id) per vertex in shared
//          memory -- the sequential "first strictly smaller" scan -- and the
//          incumbent's candidate is read back through pb_inv.
// Everything after the choice (replacement test, policy, in-degree, region
// flags) is improve_vertex's. Heavy vertices keep the block-cooperative path.
__device__ __forceinline__ void pb_pass1(const KP& p) {
    const int2* __restrict__ tw = p.pb_tw;
    const long long* __restrict__ key = p.key_i;
    long long* __restrict__ cand = p.pb_cand;
    const long long den0 = p.R == 1 ? p.lam_den[0] : 1;
    constexpr int kU = 4; // 8 and 16 measured slower (register pressure)
    const std::uint64_t nth = gstride();
    for (std::uint64_t i0 = gtid(); i0 < p.pb_m; i0 += kU * nth) {
        int2 e[kU];
        long long k[kU], d[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            e[u] = __ldcs(&tw[min(i0 + u * nth, p.pb_m - 1)]); // streamed: evict first
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            k[u] = __ldcg(&key[static_cast<std::uint32_t>(e[u].x)]);
            d[u] = p.R == 1 ? den0 : p.lam_den[__ldg(&p.reg[static_cast<std::uint32_t>(e[u].x)])];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * nth < p.pb_m)
                __stcs(&cand[i0 + u * nth], k[u] + static_cast<long long>(e[u].y) * d[u]);
    }
}

constexpr int kPbVB = 1024; // vertices per pass-2 block
constexpr std::size_t kPbSmem = kPbVB * 8 + (3 * kPbVB + 2 + 2 * kMaxPbBins) * 4;

__device__ __forceinline__ void pb_pass2(const KP& p, int* changed) {
    // dynamic shared memory (kPbSmem bytes, given only to launches with the
    // pass enabled: a static allocation would shrink every launch's L1)
    unsigned char* pb_smem = dyn_smem;
    long long* s_best = reinterpret_cast<long long*>(pb_smem);                  // [kPbVB]
    std::uint32_t* s_row = reinterpret_cast<std::uint32_t*>(s_best + kPbVB);   // [kPbVB + 1]
    std::uint32_t* s_be = s_row + kPbVB + 1;                                    // [kPbVB]
    std::uint32_t* s_seg = s_be + kPbVB;                                        // [kMaxPbBins + 1]
    std::uint32_t* s_off = s_seg + kMaxPbBins + 1;                              // [kMaxPbBins]
    ChangedMarks marks;
    const std::uint32_t nb = p.pb_nb;
    constexpr int kU = 4;
    for (std::uint32_t blk = blockIdx.x; blk < p.pb_nblk; blk += gridDim.x) {
        const std::uint32_t v0 = blk * kPbVB;
        const std::uint32_t nv = min(static_cast<std::uint32_t>(kPbVB), p.N - v0);
        const std::uint32_t* off = p.pb_off + static_cast<std::size_t>(blk) * nb;
        for (std::uint32_t j = threadIdx.x; j <= nv; j += blockDim.x)
            s_row[j] = __ldg(&p.row[v0 + j]);
        for (std::uint32_t j = threadIdx.x; j < nv; j += blockDim.x) {
            s_best[j] = 0x7fffffffffffffffll;
            s_be[j] = NONE;
        }
        for (std::uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
            const std::uint32_t o = __ldg(&off[b]);
            s_off[b] = o;
            s_seg[b + 1] = __ldg(&off[nb + b]) - o;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_seg[0] = 0;
            for (std::uint32_t b = 1; b <= nb; ++b)
                s_seg[b] += s_seg[b - 1];
        }
        __syncthreads();
        const std::uint32_t tot = s_seg[nb];
        // two sweeps over the block's candidates (kU in flight per thread):
        // the minimum per vertex, then the least edge id attaining it
        for (int sweep = 0; sweep < 2; ++sweep) {
            for (std::uint32_t f0 = threadIdx.x; f0 < tot; f0 += kU * blockDim.x) {
                std::uint32_t pos[kU], lv[kU];
                long long c[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const std::uint32_t f = min(f0 + u * blockDim.x, tot - 1);
                    std::uint32_t lo = 0, hi = nb; // s_seg[lo] <= f < s_seg[lo+1]
                    while (hi - lo > 1) {
                        const std::uint32_t mid = (lo + hi) >> 1;
                        if (s_seg[mid] <= f)
                            lo = mid;
                        else
                            hi = mid;
                    }
                    pos[u] = s_off[lo] + (f - s_seg[lo]);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    lv[u] = __ldg(&p.pb_src[pos[u]]) - v0;
                    c[u] = __ldcg(&p.pb_cand[pos[u]]);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    if (f0 + u * blockDim.x >= tot || s_row[lv[u] + 1] - s_row[lv[u]] >= p.heavy_deg)
                        continue; // past the end, or the block-cooperative path owns it
                    if (sweep == 0)
                        atomicMin(&s_best[lv[u]], c[u]);
                    else if (c[u] == s_best[lv[u]])
                        atomicMin(&s_be[lv[u]], __ldg(&p.pb_perm[pos[u]]));
                }
            }
            __syncthreads();
        }
        for (std::uint32_t j = threadIdx.x; j < nv; j += blockDim.x) {
            const std::uint32_t v = v0 + j;
            const std::uint32_t deg = s_row[j + 1] - s_row[j];
            if (deg == 0 || deg >= p.heavy_deg)
                continue;
            const std::uint32_t r = p.R == 1 ? 0u : __ldg(&p.reg[v]);
            if (!p.active[r])
                continue;
            const std::uint32_t be = s_be[j];
            const std::uint32_t cur = p.succ_e[v];
            const bool rep = cur == NONE || s_best[j] < __ldcg(&p.pb_cand[__ldg(&p.pb_inv[cur])]);
            if (rep) {
                const int2 ed = __ldg(&p.ew[be]);
                const std::uint32_t t = static_cast<std::uint32_t>(ed.x);
                p.succ_e[v] = be;
                succ_w_st<1>(p, v, t, ed.y);
                p.succ_v[v] = t;
                mark_pred(p, t);
                marks.note(p, changed, r);
            } else {
                mark_pred(p, p.succ_v[v]);
            }
        }
        __syncthreads(); // shared arrays reused by the next block
    }
    marks.flush(p, changed);
}

// ------------------------------------------- TMA-staged improvement pass
//
// For key arrays far beyond L2 (exact lane): the pass is bound by random
// key gathers from HBM, and loading the edge stream through registers
// limits how many of them a thread keeps in flight. Here one thread per CTA
// copies each chunk of kBlock/G consecutive vertices -- their row offsets
// and their edge records, contiguous in the CSR -- into shared memory with
// 1-D bulk TMA (cp.async.bulk, completion on an mbarrier), double-buffered
// so chunk i+1 lands while chunk i is processed; the threads then read
// edges from shared memory and spend their registers on key gathers. A
// chunk whose edges exceed a stage (it holds a heavy vertex, whose edges the
// block-cooperative pass handles) is processed straight from global memory.
constexpr int kStE = 2048 + 16; // edge records per stage
constexpr int kStV = kBlock + 8; // row offsets per stage
struct Staged {
    int2 edge[2][kStE];
    std::uint32_t row[2][kStV];
    unsigned long long bar[2];
    std::uint32_t ebase[2], rbase[2], v0[2], v1[2];
    int ok[2];
    unsigned par[2]; // mbarrier phase parity, kept across the launch's passes
};
constexpr std::size_t kStagedSmem = sizeof(Staged);

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void staged_init(Staged& st) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < 2; ++k) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&st.bar[k])));
            st.par[k] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

// thread 0: issue the copies of chunk [v0, v1) into stage k
__device__ __forceinline__ void staged_produce(const KP& p, Staged& st, int k, std::uint32_t v0,
                                               std::uint32_t v1) {
    const std::uint32_t e0 = __ldg(&p.row[v0]), e1 = __ldg(&p.row[v1]);
    st.v0[k] = v0;
    st.v1[k] = v1;
    const std::uint32_t ea = e0 & ~1u, eb = (e1 + 1) & ~1u; // 16-byte aligned window
    if (eb - ea > static_cast<std::uint32_t>(kStE)) {
        st.ok[k] = 0;
        return;
    }
    st.ok[k] = 1;
    const std::uint32_t rb = v0 & ~3u, rc = (v1 + 1 - rb + 3) & ~3u;
    st.ebase[k] = ea;
    st.rbase[k] = rb;
    const unsigned rbytes = rc * 4, ebytes = (eb - ea) * 8;
    const unsigned bar = smem_u32(&st.bar[k]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(rbytes + ebytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(st.row[k])), "l"(p.row + rb), "r"(rbytes), "r"(bar)
                 : "memory");
    if (ebytes)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(st.edge[k])), "l"(p.ew + ea), "r"(ebytes), "r"(bar)
                     : "memory");
}

__device__ __forceinline__ void staged_wait(Staged& st, int k, unsigned parity) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&st.bar[k])), "r"(parity)
                 : "memory");
}

template <int G, int U>
__device__ __forceinline__ void improve_staged(const KP& p, int* changed, ChangedMarks& marks) {
    Staged& st = *reinterpret_cast<Staged*>(dyn_smem);
    constexpr std::uint32_t VC = kBlock / G; // vertices per chunk
    const std::uint32_t lo = p.own_lo, hi = p.own_hi;
    const std::uint32_t nch = (hi - lo + VC - 1) / VC;
    unsigned par[2] = {st.par[0], st.par[1]};
    const long long den1 = p.lam_den[0];
    std::uint32_t c = blockIdx.x;
    int k = 0;
    if (threadIdx.x == 0 && c < nch)
        staged_produce(p, st, 0, lo + c * VC, min(hi, lo + (c + 1) * VC));
    for (; c < nch; c += gridDim.x, k ^= 1) {
        const std::uint32_t cn = c + gridDim.x;
        if (threadIdx.x == 0 && cn < nch)
            staged_produce(p, st, k ^ 1, lo + cn * VC, min(hi, lo + (cn + 1) * VC));
        __syncthreads(); // stage k's bookkeeping is visible
        const std::uint32_t v = st.v0[k] + threadIdx.x / G;
        if (st.ok[k]) {
            staged_wait(st, k, par[k]);
            par[k] ^= 1;
            if (v < st.v1[k]) {
                const std::uint32_t r0 = v - st.rbase[k];
                improve_vertex<1, G, U, false, true>(p, changed, marks, v, den1, st.edge[k], st.ebase[k],
                                                        st.row[k][r0], st.row[k][r0 + 1]);
            }
        } else if (v < st.v1[k]) {
            improve_vertex<1, G, U, false>(p, changed, marks, v, den1);
        }
        __syncthreads(); // stage k is consumed before it is refilled
    }
    if (threadIdx.x == 0) {
        st.par[0] = par[0];
        st.par[1] = par[1];
    }
}

template <int MODE, int G, int U> __device__ __forceinline__ void improve_phase(const KP& p, int* changed) {
    if (p.nheavy)
        improve_heavy<MODE>(p, changed);
    if constexpr (MODE == 1) {
        if (p.pb && !p.fused) {
            if (p.R == 1 && !p.active[0])
                return;
            pb_pass1(p);
            cg::this_grid().sync();
            pb_pass2(p, changed);
            return;
        }
    }
    ChangedMarks marks;
    if (p.R == 1 && !p.active[0])
        return; // the single region finished (block-uniform: no flush needed)
    if constexpr (MODE == 1) {
        if (p.staged) {
            improve_staged<G, U>(p, changed, marks);
            marks.flush(p, changed);
            return;
        }
    }
    bool hot = false;
    if constexpr (MODE == 1) {
        if (p.nhot) {
            const unsigned slots = 1u << (32 - p.hot_shift);
            long long* hk = hot_keys();
            std::uint32_t* hv = hot_verts(p);
            for (unsigned i = threadIdx.x; i < slots; i += kBlock)
                hv[i] = NONE;
            __syncthreads();
            for (unsigned j = threadIdx.x; j < p.nhot; j += kBlock) {
                const std::uint32_t x = __ldg(&p.hot[j]);
                const long long kx = __ldcg(&p.key_i[x]);
                unsigned i = hot_hash(x, p.hot_shift);
                for (int q = 0; q < kHotProbe; ++q) { // a hub that finds no slot is gathered
                    if (atomicCAS(&hv[i], NONE, x) == NONE) {
                        hk[i] = kx;
                        break;
                    }
                    i = (i + 1) & (slots - 1);
                }
            }
            __syncthreads();
            hot = true;
        }
    }
    const std::size_t gs = gstride() / G;
    const long long den1 = MODE != 0 ? p.lam_den[0] : 1;
    if (hot) {
        for (std::size_t vv = p.own_lo + gtid() / G; vv < p.own_hi; vv += gs)
            improve_vertex<MODE, G, U, true>(p, changed, marks, static_cast<std::uint32_t>(vv), den1);
    } else {
        for (std::size_t vv = p.own_lo + gtid() / G; vv < p.own_hi; vv += gs)
            improve_vertex<MODE, G, U, false>(p, changed, marks, static_cast<std::uint32_t>(vv), den1);
    }
    marks.flush(p, changed);
}

// The optimal cycle from its anchor (one thread: a dependent walk).
__global__ void k_cycle_out(const std::uint32_t* succ, std::uint32_t start, std::uint32_t len,
                            std::uint32_t* out) {
    if (threadIdx.x != 0)
        return;
    std::uint32_t u = start;
    for (std::uint32_t i = 0; i < len; ++i) {
        out[i] = u;
        u = succ[u];
    }
}

__global__ void k_list_heavy(std::uint32_t n, const std::uint32_t* row, std::uint32_t hdeg,
                             std::uint32_t* heavy, unsigned* count) {
    for (std::size_t v = gtid(); v < n; v += gstride())
        if (row[v + 1] - row[v] >= hdeg)
            heavy[atomicAdd(count, 1u)] = static_cast<std::uint32_t>(v);
}

// Intra-region in-degree of every vertex (the number of improvement-pass
// gathers of its key), for the choice of hub vertices.
__global__ void k_edge_indeg(std::uint64_t m, const int2* ew, unsigned* cnt) {
    for (std::uint64_t e = gtid(); e < m; e += gstride())
        atomicAdd(&cnt[static_cast<std::uint32_t>(__ldg(&ew[e]).x)], 1u);
}

__global__ void k_iota(std::uint32_t n, std::uint32_t* ids) {
    for (std::size_t v = gtid(); v < n; v += gstride())
        ids[v] = static_cast<std::uint32_t>(v);
}

// ------------------------------------------------------------ helpers

// gcd(|a|, b) for b > 0 (a cycle length): one 64-bit remainder, then the
// Euclid steps in 32 bits (64-bit division is a long software sequence, and
// this runs on the serial tail of every iteration).
__device__ __forceinline__ long long gcd_ll(long long a, long long b) {
    if (a < 0)
        a = -a;
    if (b <= 0 || b > 0xffffffffll) {
        while (b) {
            const long long t = a % b;
            a = b;
            b = t;
        }
        return a;
    }
    unsigned x = static_cast<unsigned>(b), y = static_cast<unsigned>(static_cast<unsigned long long>(a) % x);
    while (y) {
        const unsigned t = x % y;
        x = y;
        y = t;
    }
    return x;
}

template <int MODE>
__device__ __forceinline__ bool rec_less(const KP& p, std::uint32_t a, std::uint32_t b) {
    constexpr bool EXACT = MODE != 0;
    if constexpr (EXACT) {
        const __int128 l = static_cast<__int128>(ldv(p.cyc_wi[a])) * ldv(p.cyc_len[b]);
        const __int128 r = static_cast<__int128>(ldv(p.cyc_wi[b])) * ldv(p.cyc_len[a]);
        if (l != r)
            return l < r;
    } else {
        const double ma = ldv(p.cyc_wf[a]) / ldv(p.cyc_len[a]);
        const double mb = ldv(p.cyc_wf[b]) / ldv(p.cyc_len[b]);
        if (ma < mb)
            return true;
        if (mb < ma)
            return false;
    }
    return a < b;
}

__device__ __forceinline__ int ceil_log2_d(unsigned long long x) {
    return x <= 1 ? 0 : 64 - __clzll(x - 1);
}


// ------------------------------------------------------------ phases
//
// Loops containing block_append/block_flag are block-uniform.

#define OCM_BLOCK_LOOP(i, lo, hi)                                                                \
    for (std::uint64_t i##_b = (lo) + blockIdx.x * std::uint64_t(kBlock); i##_b < (hi);          \
         i##_b += gridDim.x * std::uint64_t(kBlock))

template <int MODE> __device__ __forceinline__ void ph_init(const KP& p) {
    const std::size_t tid = gtid(), nth = gstride();
    for (std::size_t v = tid; v < p.N; v += nth) {
        p.succ_e[v] = NONE;
        p.succ_v[v] = NONE;
        if (MODE == 1 && p.succ_vw)
            p.succ_vw[v] = make_int2(static_cast<int>(NONE), 0);
        key_st<MODE>(p, static_cast<std::uint32_t>(v), KeyT<MODE>(0));
        p.indeg[v] = 0;
    }
    for (std::size_t r = tid; r <= p.R; r += nth) { // slot R: trivial vertices
        p.lam_num[r] = 0;
        p.lam_den[r] = 1;
        p.lam_f[r] = 0.0;
        p.active[r] = r < p.R ? 1 : 0;
        p.changed[0][r] = 0;
        p.changed[1][r] = 0;
        p.slot[r] = EMPTY;
        p.src[r] = NONE;
        p.iters[r] = 0;
    }
}

// Region check (howard_par.hpp:189/208: a region whose pass changed nothing
// is finished) fused with the split of the still-working vertices into
// leaves of the policy graph (in-degree 0: never on a cycle, never the
// successor of anyone) and the core, whose first doubling round is done
// here. A vertex still works iff its region changed in this pass (changed is
// only ever raised for active regions).
template <int MODE>
__device__ __forceinline__ void ph_classify(const KP& p, int par, const Ring& ra, const Ring& rl,
                                            const Ring& rc) {
    constexpr bool EXACT = MODE != 0;
    const int* changed = p.changed[par];
    unsigned still = 0;
    for (std::size_t r = gtid(); r < p.R; r += gstride()) {
        if (p.active[r]) {
            if (changed[r])
                ++still;
            else
                p.active[r] = 0;
        }
        p.changed[par ^ 1][r] = 0;
    }
    block_count(still, ra);
#if OCM_CBITS
    if (p.cbits)
        for (std::size_t w = gtid(); w < (std::size_t(p.N) + 31) / 32; w += gstride())
            p.cbits[w] = 0; // set again by keep and attach
#endif
    // four consecutive vertices per thread, one reservation per ring per
    // 1024 vertices (a per-256 append made the two list counters the
    // contended words of the phase); lists stay in vertex order
    constexpr int kV = 4;
    for (std::uint64_t base = (blockIdx.x * std::uint64_t(kBlock) + threadIdx.x) * kV; ;
         base += gridDim.x * std::uint64_t(kBlock) * kV) {
        const std::uint64_t blk0 = base - threadIdx.x * kV; // block-uniform loop test
        if (blk0 >= p.N)
            break;
        unsigned lbits = 0, cbits = 0;
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            const std::uint64_t v = base + k;
            if (v < p.N && changed[__ldg(&p.reg[v])]) {
                if (!has_pred(p, static_cast<std::uint32_t>(v)))
                    lbits |= 1u << k;
                else
                    cbits |= 1u << k;
            }
        }
        std::uint64_t ls, cs;
        block_reserve2(__popc(lbits), rl, ls, __popc(cbits), rc, cs);
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            const std::uint32_t v = static_cast<std::uint32_t>(base + k);
            if (lbits >> k & 1u)
                p.plist[ls++] = v;
            if (cbits >> k & 1u) {
                // the first doubling round, straight from the policy: the
                // successor of a core vertex is a core vertex
                p.clist[cs++] = v;
                PJC x;
                if (MODE == 1 && p.succ_vw) {
                    const int2 a1 = p.succ_vw[v];
                    const int2 a2 = p.succ_vw[a1.x];
                    x.nxt = static_cast<std::uint32_t>(a2.x);
                    x.mn = min(v, static_cast<std::uint32_t>(a1.x));
                    x.w = static_cast<long long>(a1.y) + a2.y;
                } else {
                    const std::uint32_t sv = p.succ_v[v];
                    x.nxt = p.succ_v[sv];
                    x.mn = min(v, sv);
                    x.w = EXACT ? succ_w<MODE>(p, v) + succ_w<MODE>(p, sv) : 0ll;
                }
                p.pj[1][v] = x;
            }
        }
    }
}

// Synchronous pointer doubling of (segment end, least vertex, weight sum)
// over the core (closed under succ: a leaf is nobody's successor), S
// doubling steps per pass (records of 2^k steps -> 2^(k+S)): 2^S chained
// reads of the same buffer instead of S rounds and S-1 barriers -- a
// round's cost is mostly its barrier and the latency ramp, not its loads.
#ifndef OCM_ROUND_ILP
#define OCM_ROUND_ILP 1
#endif
// Doubling steps per pass S: 2^S - 1 chained gathers take records of 2^k
// steps to 2^(k+S). Fewer passes (barriers) against more gathers per step:
// S = 3 while the records are L2-resident (config 2: -2%), S = 2 beyond
// (configs 4/5: S = 3 +3-5%, S = 1 +1-3%; profiles/r02/ab_rounds_r02.log).
// A kernel per S (template SR: the exact lane has an S = 3 instantiation; a
// runtime switch inside one kernel cost configs 4/5 1-2%, the code of both
// passes living in one register allocation), chosen per session
// (OCM_ROUND_S env); -DOCM_ROUND_S=<S> fixes it at compile time.
#ifndef OCM_ROUND_S
#define OCM_ROUND_S 0
#endif
constexpr int kRoundS = OCM_ROUND_S;
template <int S> __device__ __forceinline__ void ph_round_multi(const KP& p, std::uint64_t nC, int in) {
    const PJC* __restrict__ a = p.pj[in];
    PJC* __restrict__ o = p.pj[in ^ 1];
    constexpr int kR = OCM_ROUND_ILP; // independent chains interleaved per thread
    const std::uint64_t nth = gstride();
    for (std::uint64_t i0 = gtid(); i0 < nC; i0 += kR * nth) {
        std::uint32_t v[kR];
        PJC z[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            v[r] = i0 + r * nth < nC ? p.clist[i0 + r * nth] : NONE;
            if (v[r] != NONE)
                z[r] = a[v[r]];
        }
#pragma unroll
        for (int h = 1; h < (1 << S); ++h) {
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                if (v[r] == NONE)
                    continue;
                const PJC y = a[z[r].nxt];
                z[r].nxt = y.nxt;
                z[r].mn = min(z[r].mn, y.mn);
                z[r].w += y.w;
            }
        }
#pragma unroll
        for (int r = 0; r < kR; ++r)
            if (v[r] != NONE)
                o[v[r]] = z[r];
    }
}

// Verification. M = image of succ^L. It passes iff (A)
// every vertex of M has a predecessor in M -- succ maps M into M, so this
// is |succ(M)| = |M| -- and (B) the anchor is constant along succ in M
// (every window covers its whole cycle). The mark phase records the anchors
// and counts |M|; the check phase counts |succ(M)|, tests (B), lists M (the
// cycle vertices, if it passes) and, in exact mode, already accumulates the
// per-anchor (length, weight) records (howard_par.hpp:319), cleared here.
__device__ __forceinline__ void ph_mark(const KP& p, std::uint64_t nC, int in, std::uint32_t stamp,
                                        bool exact, const Ring& rl) {
    const PJC* a = p.pj[in];
    constexpr int kR = 4;
    const std::uint64_t nth = gstride();
    for (std::uint64_t i0 = gtid(); i0 < nC; i0 += kR * nth) {
        std::uint32_t v[kR], j[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r)
            v[r] = i0 + r * nth < nC ? p.clist[i0 + r * nth] : NONE;
#pragma unroll
        for (int r = 0; r < kR; ++r)
            if (v[r] != NONE)
                j[r] = a[v[r]].nxt;
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            if (v[r] == NONE)
                continue;
            // many vertices share j: read before the exchange; the first
            // marker lists j, so M is enumerated without another full pass.
            // Only M's (length, weight) records are cleared: the anchors the
            // check phase accumulates into lie in M whenever it passes.
            if (p.cmark[j[r]] != stamp && atomicExch(&p.cmark[j[r]], stamp) != stamp) {
                p.wlist[warp_append(rl)] = j[r];
                p.cyc_len[j[r]] = 0;
                if (exact)
                    p.cyc_wi[j[r]] = 0;
            }
        }
    }
}

// The last doubling pass fused with the mark phase: each core vertex
// takes S more doubling steps (2^S chained reads of the input records) and
// marks its image j -- one phase and one barrier fewer per verification.
// Anchors are only needed on M: the check reads them from the final
// records (a cycle vertex's record of L steps covers its window), and every
// other vertex finds its anchor at its image jump(v) in M.
template <int S>
__device__ __forceinline__ void ph_round_mark(const KP& p, std::uint64_t nC, int in, std::uint32_t stamp,
                                              bool exact, const Ring& rl) {
    const PJC* __restrict__ a = p.pj[in];
    PJC* __restrict__ o = p.pj[in ^ 1];
    for (std::uint64_t i = gtid(); i < nC; i += gstride()) {
        const std::uint32_t v = p.clist[i];
        PJC z = a[v];
#pragma unroll
        for (int h = 1; h < (1 << S); ++h) {
            const PJC y = a[z.nxt];
            z.nxt = y.nxt;
            z.mn = min(z.mn, y.mn);
            z.w += y.w;
        }
        o[v] = z;
        const std::uint32_t j = z.nxt;
        if (p.cmark[j] != stamp && atomicExch(&p.cmark[j], stamp) != stamp) {
            p.wlist[warp_append(rl)] = j;
            p.cyc_len[j] = 0;
            if (exact)
                p.cyc_wi[j] = 0;
        }
    }
}

// Over the listed M only: (B) and |succ(M)|, and -- speculatively, exact
// lane -- the per-anchor (length, weight) records (howard_par.hpp:319).
template <int MODE>
__device__ __forceinline__ void ph_check(const KP& p, std::uint64_t nM, std::uint32_t stamp,
                                         unsigned* flag, const Ring& rs, const PJC* fin) {
    constexpr bool EXACT = MODE != 0;
    bool fail = false;
    unsigned fresh = 0;
    const unsigned lane = threadIdx.x & 31;
    const std::uint64_t wid = gtid() >> 5, ws = gstride() >> 5;
    for (std::uint64_t base = wid * 32; base < nM; base += ws * 32) {
        const std::uint64_t i = base + lane;
        const bool on = i < nM;
        std::uint32_t v = 0, a = 0;
        if (on) {
            v = p.wlist[i];
            const std::uint32_t s = p.succ_v[v];
            // v's anchor: the least vertex of the window of L steps from v
            a = fin[v].mn;
            fail |= fin[s].mn != a;
            p.comp[v] = a;
            if (p.cmark2[s] != stamp && atomicExch(&p.cmark2[s], stamp) != stamp)
                ++fresh;
        }
        if constexpr (EXACT) {
            // integer segmented reduction; a warp whose cycle vertices share
            // one anchor pre-reduces to one atomic pair
            const unsigned am = __ballot_sync(FULL, on);
            const int lead = __ffs(am) - 1;
            const std::uint32_t a0 = __shfl_sync(FULL, a, lead);
            const bool uni = __all_sync(FULL, !on || a == a0);
            long long w = on ? succ_w<MODE>(p, v) : 0ll;
            if (uni) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
                    w += __shfl_xor_sync(FULL, w, off);
                if (static_cast<int>(lane) == lead) {
                    atomicAdd(&p.cyc_len[a0], static_cast<unsigned>(__popc(am)));
                    atomicAdd(reinterpret_cast<unsigned long long*>(&p.cyc_wi[a0]),
                              static_cast<unsigned long long>(w));
                }
            } else if (on) {
                atomicAdd(&p.cyc_len[a], 1u);
                atomicAdd(reinterpret_cast<unsigned long long*>(&p.cyc_wi[a]),
                          static_cast<unsigned long long>(w));
            }
        }
    }
    block_flag(fail, flag, stamp);
    block_count(fresh, rs);
}

// Float lane: each anchor walks its own cycle from itself, summing in the
// reference's order (howard_par.hpp:323) -> identical means. Runs after
// the verification passed (the walk needs a true cycle).
__device__ __forceinline__ void ph_stats_float(const KP& p, std::uint64_t nM) {
    for (std::uint64_t i = gtid(); i < nM; i += gstride()) {
        const std::uint32_t v = p.wlist[i];
        if (p.comp[v] != v)
            continue;
        double s = 0.0;
        std::uint32_t len = 0, u = v;
        do {
            s += p.succ_wf[u];
            ++len;
            u = p.succ_v[u];
        } while (u != v);
        p.cyc_wf[v] = s;
        p.cyc_len[v] = len;
    }
}

// Adoption (howard_par.hpp:349-364) of region r's winning record.
template <int MODE> __device__ __forceinline__ unsigned adopt_region(const KP& p, std::uint32_t r) {
    constexpr bool EXACT = MODE != 0;
    Ctl* c = p.c;
    const unsigned long long a = p.slot[r];
    p.slot[r] = EMPTY;
    if (a == EMPTY) {
        c->error = 1;
        return 0;
    }
    p.src[r] = static_cast<std::uint32_t>(a);
    const unsigned len = p.cyc_len[a];
    if constexpr (EXACT) {
        long long num = p.cyc_wi[a], den = len;
        const long long g = gcd_ll(num, den);
        if (g > 1) {
            num /= g;
            den /= g;
        }
        if (p.iters[r] > 0 &&
            static_cast<__int128>(p.lam_num[r]) * den < static_cast<__int128>(num) * p.lam_den[r])
            c->lambda_up = 1;
        p.lam_num[r] = num;
        p.lam_den[r] = den;
        if (r == 0 && p.iters[0] < p.tr_cap) { // lambda trace of region 0
            p.tr_num[p.iters[0]] = num;
            p.tr_den[p.iters[0]] = den;
        }
        // every key |K| <= max_region * (max|w|*den + |num|) stays inside
        // the lane's bound (else: the fast lane reports it, and the session
        // re-solves in the wide lane)
        const __int128 step = static_cast<__int128>(p.max_abs_w) * den + (num < 0 ? -num : num);
        if (static_cast<__int128>(p.max_region) * step >=
            (static_cast<__int128>(1) << (MODE == 2 ? 120 : 62)))
            c->overflow = 1;
    } else {
        p.lam_f[r] = p.cyc_wf[a] / len;
        if (r == 0 && p.iters[0] < p.tr_cap)
            p.tr_f[p.iters[0]] = p.lam_f[r];
    }
    p.iters[r] += 1;
    return len;
}

// Winning-cycle values: prefix sums of w*den - num along the cycle, cut at
// the anchor (value(anchor) = 0), by pointer jumping over those vertices.
template <int MODE> struct PvOf { using T = PJV; };
template <> struct PvOf<2> { using T = PJVW; };
template <int MODE> __device__ __forceinline__ typename PvOf<MODE>::T* pv_buf(const KP& p, int j) {
    if constexpr (MODE == 2)
        return p.pvw[j];
    else
        return p.pv[j];
}

template <int MODE> __device__ __forceinline__ void wc_init_one(const KP& p, std::uint32_t v, std::uint32_t r) {
    typename PvOf<MODE>::T x;
    const std::uint32_t root = p.src[r];
    if (v == root) {
        x.acc = 0;
        x.nxt = root;
    } else {
        x.acc = static_cast<KeyT<MODE>>(succ_w<MODE>(p, v)) * p.lam_den[r] - p.lam_num[r];
        x.nxt = p.succ_v[v];
    }
    x.root = root;
    pv_buf<MODE>(p, 0)[v] = x;
}

template <int MODE>
__device__ __forceinline__ void wc_round(const KP& p, const std::uint32_t* list, std::uint64_t nW, int j,
                                         std::uint64_t from, std::uint64_t step) {
    using PV = typename PvOf<MODE>::T;
    const PV* __restrict__ a = pv_buf<MODE>(p, j & 1);
    PV* __restrict__ o = pv_buf<MODE>(p, (j & 1) ^ 1);
    for (std::uint64_t i = from; i < nW; i += step) {
        const std::uint32_t v = list[i];
        const PV x = a[v];
        const PV y = a[x.nxt];
        PV z;
        z.acc = x.acc + y.acc;
        z.nxt = y.nxt;
        z.root = x.root;
        o[v] = z;
    }
}

template <int MODE>
__device__ __forceinline__ void wc_final(const KP& p, const std::uint32_t* list, std::uint64_t nW, int wr,
                                         std::uint64_t from, std::uint64_t step) {
    const typename PvOf<MODE>::T* fin = pv_buf<MODE>(p, wr & 1);
    for (std::uint64_t i = from; i < nW; i += step) {
        const std::uint32_t v = list[i];
        key_st<MODE>(p, v, fin[v].acc);
    }
}

// Winning cycles of up to kSmemCycle vertices (listed in rem[1]) by one CTA
// entirely in shared memory: vertices get local slots through a small
// open-addressing table, then the prefix sums cut at each anchor run as
// ceil(log2(len-1)) pointer-jumping rounds over shared arrays.
constexpr unsigned kSmemCycle = 128; // 512 measured 2% slower: its 20 KB of static shared
                                     // memory per CTA came out of every launch's L1

// One instance per CTA, shared by both winning-cycle paths.
__shared__ std::uint32_t wc_key[2 * kSmemCycle], wc_val[2 * kSmemCycle];
__shared__ std::uint32_t wc_nxt[2][kSmemCycle];
__shared__ long long wc_acc[2][kSmemCycle];
__shared__ __int128 wc_acc_w[2][kSmemCycle]; // wide lane only
template <int MODE> __device__ __forceinline__ auto& wc_acc_of() {
    if constexpr (MODE == 2)
        return wc_acc_w;
    else
        return wc_acc;
}

template <int MODE> __device__ __forceinline__ void wincyc_shared(const KP& p, unsigned nW, int wr) {
    auto& s_key = wc_key;
    auto& s_val = wc_val;
    auto& s_nxt = wc_nxt;
    auto& s_acc = wc_acc_of<MODE>();
    constexpr unsigned kMask = 2 * kSmemCycle - 1;
    for (unsigned i = threadIdx.x; i < 2 * kSmemCycle; i += blockDim.x)
        s_key[i] = NONE;
    __syncthreads();
    for (unsigned i = threadIdx.x; i < nW; i += blockDim.x) {
        const std::uint32_t v = p.rem[1][i];
        unsigned h = (v * 2654435761u) & kMask;
        while (atomicCAS(&s_key[h], NONE, v) != NONE)
            h = (h + 1) & kMask;
        s_val[h] = i;
    }
    __syncthreads();
    for (unsigned i = threadIdx.x; i < nW; i += blockDim.x) {
        const std::uint32_t v = p.rem[1][i];
        const std::uint32_t r = p.R == 1 ? 0u : __ldg(&p.reg[v]);
        if (v == p.src[r]) {
            s_acc[0][i] = 0;
            s_nxt[0][i] = i;
        } else {
            s_acc[0][i] = static_cast<KeyT<MODE>>(succ_w<MODE>(p, v)) * p.lam_den[r] - p.lam_num[r];
            const std::uint32_t sv = p.succ_v[v];
            unsigned h = (sv * 2654435761u) & kMask;
            while (s_key[h] != sv)
                h = (h + 1) & kMask;
            s_nxt[0][i] = s_val[h];
        }
    }
    __syncthreads();
    for (int j = 0; j < wr; ++j) {
        const int a = j & 1, o = a ^ 1;
        for (unsigned i = threadIdx.x; i < nW; i += blockDim.x) {
            const std::uint32_t x = s_nxt[a][i];
            s_acc[o][i] = s_acc[a][i] + s_acc[a][x];
            s_nxt[o][i] = s_nxt[a][x];
        }
        __syncthreads();
    }
    for (unsigned i = threadIdx.x; i < nW; i += blockDim.x)
        key_st<MODE>(p, p.rem[1][i], s_acc[wr & 1][i]);
}

// Region-specific minimum voting (howard_par.hpp:56 vote_min; paper
// Alg. 5: a holder is replaced only by a strictly smaller (mean, anchor)),
// over the anchors among the nM cycle vertices in wlist. The last block to
// finish voting adopts every region's winner and, when the winning cycles
// are small, computes their values itself (block barriers only); otherwise
// it raises wc_big and the grid does it after the barrier.
template <int MODE>
__device__ __forceinline__ void vote_pass(const KP& p, std::uint64_t nM, std::uint64_t from, std::uint64_t step) {
    constexpr bool EXACT = MODE != 0;
    for (std::uint64_t i = from; i < nM; i += step) {
        const std::uint32_t v = p.wlist[i];
        if (p.comp[v] != v)
            continue;
        unsigned long long* cell = &p.slot[__ldg(&p.reg[v])];
        unsigned long long cur = ldv(*cell);
        for (;;) {
            if (cur != EMPTY && !rec_less<MODE>(p, v, static_cast<std::uint32_t>(cur)))
                break;
            const unsigned long long prev = atomicCAS(cell, cur, v);
            if (prev == cur)
                break;
            cur = prev;
        }
    }
}

// Adoption and the winning cycles' values by one block (s_maxlen, s_nw
// zeroed by the caller before its last barrier).
template <int MODE>
__device__ __forceinline__ void winning_cycle_tail(const KP& p, unsigned nW, unsigned maxlen,
                                                   std::uint32_t stamp);

template <int MODE>
__device__ __forceinline__ void vote_tail(const KP& p, std::uint64_t nM, std::uint32_t stamp,
                                          unsigned& s_maxlen, unsigned& s_nw) {
    constexpr bool EXACT = MODE != 0;
    for (std::uint32_t r = threadIdx.x; r < p.R; r += blockDim.x)
        if (p.active[r]) {
            const unsigned len = adopt_region<MODE>(p, r);
            atomicMax(&s_maxlen, len);
        }
    if constexpr (!EXACT)
        return;
    __syncthreads();
    // winning-cycle vertices among the cycle vertices (compacted in rem[1])
    for (std::uint64_t i = threadIdx.x; i < nM; i += blockDim.x) {
        const std::uint32_t v = p.wlist[i];
        const std::uint32_t r = p.R == 1 ? 0u : __ldg(&p.reg[v]);
        if (p.comp[v] == p.src[r])
            p.rem[1][atomicAdd(&s_nw, 1u)] = v;
    }
    __syncthreads();
    winning_cycle_tail<MODE>(p, s_nw, s_maxlen, stamp);
}

// The winning cycles' values (nW vertices listed in rem[1], longest maxlen).
template <int MODE>
__device__ __forceinline__ void winning_cycle_tail(const KP& p, unsigned nW, unsigned maxlen,
                                                   std::uint32_t stamp) {
    constexpr bool EXACT = MODE != 0;
    Ctl* c = p.c;
    const int wr = ceil_log2_d(maxlen > 1 ? maxlen - 1 : 1); // farthest: len-1 steps
    if (nW <= kSmemCycle) {
        wincyc_shared<MODE>(p, nW, wr);
        return;
    }
    for (std::uint64_t i = threadIdx.x; i < nW; i += blockDim.x) {
        const std::uint32_t v = p.rem[1][i];
        wc_init_one<MODE>(p, v, p.R == 1 ? 0u : __ldg(&p.reg[v]));
    }
    c->wc_n[stamp & 1] = (static_cast<unsigned long long>(stamp) << 32) | nW;
    c->wc_len[stamp & 1] = maxlen;
    if (nW > p.small_wc) {
        if (threadIdx.x == 0)
            c->wc_big[stamp & 1] = stamp;
        return;
    }
    __syncthreads();
    for (int j = 0; j < wr; ++j) {
        wc_round<MODE>(p, p.rem[1], nW, j, threadIdx.x, blockDim.x);
        __syncthreads();
    }
    wc_final<MODE>(p, p.rem[1], nW, wr, threadIdx.x, blockDim.x);
}


template <int MODE>
__device__ __forceinline__ void ph_vote(const KP& p, std::uint64_t nM, std::uint32_t stamp,
                                        unsigned long long done_base) {
    constexpr bool EXACT = MODE != 0;
    Ctl* c = p.c;
    vote_pass<MODE>(p, nM, gtid(), gstride());
    __shared__ int s_last;
    __shared__ unsigned s_maxlen, s_nw;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long prev = atomicAdd(&c->done, 1ull);
        s_last = prev == done_base + gridDim.x - 1;
        s_maxlen = 0;
        s_nw = 0;
        __threadfence();
    }
    __syncthreads();
    if (s_last)
        vote_tail<MODE>(p, nM, stamp, s_maxlen, s_nw);
}

// The common case in full (exact lane, one region, |M| <= one block, a
// winning cycle of <= kSmemCycle vertices): thread i keeps cycle vertex
// M[i], its anchor, successor and weight in registers from the vote to the
// values, so adoption, the winning-cycle listing and its prefix sums add no
// global round trips beyond the adoption's own.
template <int MODE>
__device__ __forceinline__ bool vote_small(const KP& p, unsigned nM, std::uint32_t stamp,
                                           const PJC* fin, unsigned* vflag = nullptr) {
    constexpr bool EXACT = MODE != 0;
    auto& s_key = wc_key;
    auto& s_val = wc_val;
    auto& s_nxt = wc_nxt;
    auto& s_acc = wc_acc_of<MODE>();
    __shared__ unsigned s_wcnt[kBlock / 32], s_nw;
    __shared__ std::uint32_t s_src;
    __shared__ unsigned s_len;
    constexpr unsigned kMask = 2 * kSmemCycle - 1;
    const unsigned i = threadIdx.x, lane = i & 31, warp = i >> 5;
    std::uint32_t v = NONE, an = NONE, sv = 0;
    long long w = 0;
    if (i < nM) {
        v = p.wlist[i];
        an = fin[v].mn; // the window of L steps from v (see ph_check)
        sv = p.succ_v[v];
        w = succ_w<MODE>(p, v);
        p.comp[v] = an;
    }
    if (vflag) {
        // the check phase's work for these few vertices (ph_check): (B)
        // anchor constant along succ, (A) |succ(M)| = |M|, and the
        // per-anchor (length, weight) records
        bool fail = false;
        int fresh = 0;
        if (i < nM) {
            fail = fin[sv].mn != an;
            fresh = p.cmark2[sv] != stamp && atomicExch(&p.cmark2[sv], stamp) != stamp;
            atomicAdd(&p.cyc_len[an], 1u);
            atomicAdd(reinterpret_cast<unsigned long long*>(&p.cyc_wi[an]),
                      static_cast<unsigned long long>(static_cast<long long>(w)));
        }
        const bool failed = __syncthreads_or(fail) || __syncthreads_count(fresh) != static_cast<int>(nM);
        if (failed) {
            if (i == 0)
                *vflag = stamp; // the grid retries with one more doubling step
            return true;
        }
        __threadfence(); // the records, before the vote reads them
        __syncthreads();
    }
    // vote (anchors only: usually one or two CASes on the one slot)
    if (i < nM && an == v) {
        unsigned long long* cell = &p.slot[0];
        unsigned long long cur = ldv(*cell);
        for (;;) {
            if (cur != EMPTY && !rec_less<MODE>(p, v, static_cast<std::uint32_t>(cur)))
                break;
            const unsigned long long prev = atomicCAS(cell, cur, v);
            if (prev == cur)
                break;
            cur = prev;
        }
    }
    for (unsigned j = i; j < 2 * kSmemCycle; j += blockDim.x)
        s_key[j] = NONE;
    __threadfence(); // the slot CASes, before adoption reads the slot
    __syncthreads();
    if (i == 0) {
        s_len = p.active[0] ? adopt_region<MODE>(p, 0) : 0u;
        s_src = p.src[0];
    }
    __syncthreads();
    // the winning cycle's vertices, numbered by a block-wide prefix count
    const bool win = i < nM && an == s_src;
    const unsigned bal = __ballot_sync(FULL, win);
    if (lane == 0)
        s_wcnt[warp] = __popc(bal);
    __syncthreads();
    if (i == 0) {
        unsigned tot = 0;
        for (unsigned j = 0; j < blockDim.x / 32; ++j) {
            const unsigned c = s_wcnt[j];
            s_wcnt[j] = tot;
            tot += c;
        }
        s_nw = tot;
    }
    __syncthreads();
    const unsigned nW = s_nw;
    if (nW > kSmemCycle)
        return false; // (block-uniform) the general path takes over
    const unsigned idx = s_wcnt[warp] + __popc(bal & ((1u << lane) - 1u));
    if (win) {
        unsigned h = (v * 2654435761u) & kMask;
        while (atomicCAS(&s_key[h], NONE, v) != NONE)
            h = (h + 1) & kMask;
        s_val[h] = idx;
    }
    __syncthreads();
    if (win) {
        if (v == s_src) {
            s_acc[0][idx] = 0;
            s_nxt[0][idx] = idx;
        } else {
            s_acc[0][idx] = static_cast<KeyT<MODE>>(w) * p.lam_den[0] - p.lam_num[0];
            unsigned h = (sv * 2654435761u) & kMask;
            while (s_key[h] != sv)
                h = (h + 1) & kMask;
            s_nxt[0][idx] = s_val[h];
        }
    }
    __syncthreads();
    const unsigned maxlen = s_len;
    const int wr = ceil_log2_d(maxlen > 1 ? maxlen - 1 : 1); // farthest: len-1 steps
    for (int j = 0; j < wr; ++j) {
        const int a = j & 1, o = a ^ 1;
        if (win) {
            const std::uint32_t x = s_nxt[a][idx];
            s_acc[o][idx] = s_acc[a][idx] + s_acc[a][x];
            s_nxt[o][idx] = s_nxt[a][x];
        }
        __syncthreads();
    }
    if (win)
        key_st<MODE>(p, v, s_acc[wr & 1][idx]);
    (void)stamp;
    return true;
}

// Few cycle vertices (the common case once the policy settles): block 0
// votes, adopts and computes the winning cycles' values alone while the
// grid waits at the phase barrier -- no grid-wide completion counter (two
// gpu-scope fences and one contended atomic per block cost more than the
// vote itself).
constexpr std::uint64_t kVoteOneBlock = 4096;

template <int MODE>
__device__ __forceinline__ void ph_vote_one_block(const KP& p, std::uint64_t nM, std::uint32_t stamp,
                                                  const PJC* fin, unsigned* vflag = nullptr) {
    constexpr bool EXACT = MODE != 0;
    __shared__ unsigned s_maxlen, s_nw;
    if (EXACT && p.R == 1 && nM <= blockDim.x) {
        if (vote_small<MODE>(p, static_cast<unsigned>(nM), stamp, fin, vflag))
            return;
        // a winning cycle too long for shared memory: list it and take the
        // general path (adoption is already done)
        __syncthreads();
        if (threadIdx.x == 0)
            s_nw = 0;
        __syncthreads();
        for (std::uint64_t i = threadIdx.x; i < nM; i += blockDim.x) {
            const std::uint32_t v = p.wlist[i];
            if (p.comp[v] == p.src[0])
                p.rem[1][atomicAdd(&s_nw, 1u)] = v;
        }
        __syncthreads();
        winning_cycle_tail<MODE>(p, s_nw, ldv(p.cyc_len[p.src[0]]), stamp);
        return;
    }
    vote_pass<MODE>(p, nM, threadIdx.x, blockDim.x);
    __threadfence(); // the block's slot CASes, before adoption reads the slots
    if (threadIdx.x == 0) {
        s_maxlen = 0;
        s_nw = 0;
    }
    __syncthreads();
    vote_tail<MODE>(p, nM, stamp, s_maxlen, s_nw);
}

// Kept component (howard_par.hpp:370/393): vertices whose policy path
// enters the winning cycle keep their edges, everyone else queues for
// re-attachment. Core and leaves in one pass over [core | leaves]. Exact
// keys: a core vertex v off the cycle gets K(v) = W_L(v)*den - L*num +
// K(jump v) from its doubling record (the winning cycle's reduced weight is
// exactly 0, so extra turns add nothing); a leaf takes K(succ) + w*den - num,
// recomputing its core successor's key the same way (never reading a key
// being written in this phase). Resets the in-degree of core vertices.
// The formula also holds ON the winning cycle (its reduced weight is 0, so
// K(u) = w(u)*den - num + K(succ u) at every cycle vertex, the anchor
// included): a leaf's successor needs no cycle-membership test (a random
// 4-byte gather at HBM-resident sizes); core vertices skip their cycle
// vertices (keys already written by the vote) with a coalesced test.
template <int MODE>
__device__ __forceinline__ KeyT<MODE> core_key(const KP& p, const PJC* a, std::uint32_t v, std::uint32_t r,
                                               unsigned long long L, bool& ovf) {
    const PJC x = a[v];
    const __int128 kk = static_cast<__int128>(x.w) * p.lam_den[r] -
                        static_cast<__int128>(L) * p.lam_num[r] + key_ld<MODE>(p, x.nxt);
    ovf |= !key_in_range<MODE>(kk);
    return static_cast<KeyT<MODE>>(kk);
}

template <int MODE>
__device__ __forceinline__ void ph_keep(const KP& p, std::uint64_t nC, std::uint64_t nL, int in,
                                        std::uint32_t stamp, unsigned long long L, const Ring& ring) {
    constexpr bool EXACT = MODE != 0;
    const PJC* a = p.pj[in];
    bool ovf = false;
    const std::uint64_t tot = nC + nL;
    // re-attachment candidates are appended per warp (no block barrier per
    // 256 items: list order does not matter to the layer discipline)
    for (std::uint64_t i = gtid(); i < tot; i += gstride()) {
        bool take = false;
        std::uint32_t v = 0;
        if (i < nC) {
            v = p.clist[i];
            const std::uint32_t r = p.R == 1 ? 0u : __ldg(&p.reg[v]);
            // v's anchor is its image's in M (jump(v) lies on v's cycle)
            const bool kept = p.comp[a[v].nxt] == p.src[r];
            p.conn[v] = kept ? 0u : NONE;
            clear_pred(p, v);
            take = !kept;
            if constexpr (EXACT)
                if (kept && p.cmark[v] != stamp)
                    key_st<MODE>(p, v, core_key<MODE>(p, a, v, r, L, ovf));
        } else {
            v = p.plist[i - nC];
            const std::uint32_t s = p.succ_v[v];
            const std::uint32_t r = p.R == 1 ? 0u : __ldg(&p.reg[v]);
            const bool kept = p.comp[a[s].nxt] == p.src[r];
            p.conn[v] = kept ? 0u : NONE;
            take = !kept;
            if constexpr (EXACT)
                if (kept) {
                    const __int128 kk = static_cast<__int128>(core_key<MODE>(p, a, s, r, L, ovf)) +
                                        static_cast<__int128>(succ_w<MODE>(p, v)) * p.lam_den[r] -
                                        p.lam_num[r];
                    ovf |= !key_in_range<MODE>(kk);
                    key_st<MODE>(p, v, static_cast<KeyT<MODE>>(kk));
                }
        }
#if OCM_CBITS
        if (p.cbits)
            cbit_set(p, v, !take);
#endif
        if (take)
            p.rem[0][warp_append(ring)] = v;
    }
    clear_pred_all(p);
    block_flag(ovf, &p.c->overflow, 1);
}

// One breadth layer of howard_par.hpp:433 connectGpi: a pending vertex
// attaches through its smallest out-edge whose head was connected in an
// earlier layer (conn < layer); the stamps make the layer discipline exact
// under any schedule. Pending vertices of degree >= kAttachHeavy are scanned
// by their whole block, 2048 edges per step with a block-wide minimum of the
// hit edge ids (one thread walking a 10^5..10^6-edge hub row 8 edges at a
// time held every other block at the layer's barrier).
#ifndef OCM_ATTACH_HEAVY
#define OCM_ATTACH_HEAVY 256
#endif
constexpr std::uint32_t kAttachHeavy = OCM_ATTACH_HEAVY;

// Is edge e's head connected in an earlier layer? (bitmap first when on)
template <int MODE>
__device__ __forceinline__ bool head_connected(const KP& p, std::uint32_t t, std::uint32_t layer) {
#if OCM_CBITS
    if (p.cbits && !(ldv(p.cbits[t >> 5]) >> (t & 31) & 1u))
        return false;
#endif
    return ldv(p.conn[t]) < layer;
}

template <int MODE>
__device__ __forceinline__ void attach_via(const KP& p, std::uint32_t x, std::uint32_t e, std::uint32_t t,
                                           std::uint32_t layer, bool& ovf) {
    constexpr bool EXACT = MODE != 0;
    p.succ_e[x] = e;
    p.succ_v[x] = t;
    if constexpr (EXACT) {
        const long long w = edge_w<MODE>(p, e, __ldg(&p.ew[e]));
        succ_w_st<MODE>(p, x, t, w);
        const std::uint32_t r = __ldg(&p.reg[x]);
        const __int128 kk = static_cast<__int128>(key_ld<MODE>(p, t)) +
                            static_cast<__int128>(w) * p.lam_den[r] - p.lam_num[r];
        ovf |= !key_in_range<MODE>(kk);
        key_st<MODE>(p, x, static_cast<KeyT<MODE>>(kk));
    } else {
        p.succ_wf[x] = p.fe[e].w;
    }
    p.conn[x] = layer;
#if OCM_CBITS
    if (p.cbits)
        atomicOr(&p.cbits[x >> 5], 1u << (x & 31));
#endif
}

template <int MODE>
__device__ __forceinline__ void ph_attach(const KP& p, int cur, std::uint64_t pending, std::uint32_t layer,
                                          const Ring& ring) {
    constexpr bool EXACT = MODE != 0;
    const std::uint32_t* list = p.rem[cur];
    bool ovf = false;
    __shared__ std::uint32_t s_hx[kBlock], s_hown[kBlock];
    __shared__ unsigned s_nh, s_min;
    // block-ordered appends: the next layer's list keeps the vertex order of
    // this one (warp-order appends measured 12% slower at config 5, where
    // layers are long and the row/edge reads profit from the order)
    OCM_BLOCK_LOOP(i0, 0, pending) {
        const std::uint64_t i = i0_b + threadIdx.x;
        bool pend = false;
        std::uint32_t x = 0;
        if (threadIdx.x == 0)
            s_nh = 0;
        __syncthreads();
        if (i < pending) {
            x = list[i];
            pend = true;
            const std::uint32_t b = __ldg(&p.row[x]), e_end = __ldg(&p.row[x + 1]);
            if (e_end - b >= kAttachHeavy) {
                const unsigned h = atomicAdd(&s_nh, 1u);
                s_hx[h] = x;
                s_hown[h] = threadIdx.x;
            } else {
            // the first out-edge (CSR order) into a vertex connected earlier;
            // 8 edges and their heads' stamps in flight at a time
            for (std::uint32_t e0 = b; pend && e0 < e_end; e0 += 8) {
                std::uint32_t tt[8], cc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const std::uint32_t e = min(e0 + u, e_end - 1); // tail masked below
                    tt[u] = EXACT ? static_cast<std::uint32_t>(__ldg(&p.ew[e]).x) : p.fe[e].t;
                }
                int hit = -1;
#if OCM_CBITS
                if (p.cbits) {
                unsigned set = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (e0 + u < e_end && (ldv(p.cbits[tt[u] >> 5]) >> (tt[u] & 31) & 1u))
                        set |= 1u << u;
                (void)cc;
                for (; set; set &= set - 1) {
                    const int u = __ffs(set) - 1;
                    if (ldv(p.conn[tt[u]]) < layer) {
                        hit = u;
                        break;
                    }
                }
                } else
#endif
                {
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    cc[u] = e0 + u < e_end ? ldv(p.conn[tt[u]]) : NONE;
#pragma unroll
                for (int u = 7; u >= 0; --u)
                    if (cc[u] < layer)
                        hit = u;
                }
                if (hit >= 0) {
                    attach_via<MODE>(p, x, e0 + hit, tt[hit], layer, ovf);
                    pend = false;
                }
            }
            }
        }
        __syncthreads();
        // the block's high-degree pending vertices, one at a time, by all
        // its threads: 8 consecutive edges per thread per step, the least
        // hit edge id wins (= the first in CSR order)
        const unsigned nh = s_nh;
        for (unsigned h = 0; h < nh; ++h) {
            const std::uint32_t hx = s_hx[h];
            const std::uint32_t b = __ldg(&p.row[hx]), e_end = __ldg(&p.row[hx + 1]);
            std::uint32_t found = NONE;
            for (std::uint32_t w0 = b; w0 < e_end; w0 += kBlock * 8) {
                if (threadIdx.x == 0)
                    s_min = NONE;
                __syncthreads();
                const std::uint32_t e0 = w0 + threadIdx.x * 8;
                for (std::uint32_t e = e0; e < min(e0 + 8, e_end); ++e) {
                    const std::uint32_t t = EXACT ? static_cast<std::uint32_t>(__ldg(&p.ew[e]).x) : p.fe[e].t;
                    if (head_connected<MODE>(p, t, layer)) {
                        atomicMin(&s_min, e);
                        break;
                    }
                }
                __syncthreads();
                found = s_min;
                __syncthreads(); // everyone read s_min before the next reset
                if (found != NONE)
                    break;
            }
            if (found != NONE && threadIdx.x == s_hown[h]) {
                const std::uint32_t t = EXACT ? static_cast<std::uint32_t>(__ldg(&p.ew[found]).x)
                                              : p.fe[found].t;
                attach_via<MODE>(p, hx, found, t, layer, ovf);
                pend = false;
            }
        }
        const std::uint64_t slot = block_append(pend, ring);
        if (pend)
            p.rem[cur ^ 1][slot] = x;
    }
    block_flag(ovf, &p.c->overflow, 1);
}

// Float lane: level-synchronous propagation from the anchor, computing
// (value(succ) + w) - lambda exactly as FloatMode::extend (policy.hpp:105).
// Working vertices are the classified core and leaves; anchors start the
// propagation, the rest are listed as pending.
__device__ __forceinline__ void ph_fprop_init(const KP& p, std::uint64_t nC, std::uint64_t nL,
                                              const Ring& ring) {
    const std::uint64_t tot = nC + nL;
    OCM_BLOCK_LOOP(i0, 0, tot) {
        const std::uint64_t i = i0_b + threadIdx.x;
        bool pend = false;
        std::uint32_t v = 0;
        if (i < tot) {
            v = i < nC ? p.clist[i] : p.plist[i - nC];
            if (v == p.src[p.R == 1 ? 0u : __ldg(&p.reg[v])]) {
                p.conn[v] = 0;
                p.key_f[v] = 0.0;
            } else {
                p.conn[v] = NONE;
                pend = true;
            }
        }
        const std::uint64_t slot = block_append(pend, ring);
        if (pend)
            p.rem[0][slot] = v;
    }
}

// One level over the still-pending vertices only: a vertex whose successor
// was valued at an earlier level takes (value(succ) + w) - lambda; the rest
// move to the next pending list.
__device__ __forceinline__ void ph_fprop_level(const KP& p, int cur, std::uint64_t pending,
                                               std::uint32_t level, const Ring& ring) {
    const std::uint32_t* list = p.rem[cur];
    OCM_BLOCK_LOOP(i0, 0, pending) {
        const std::uint64_t i = i0_b + threadIdx.x;
        bool pend = false;
        std::uint32_t v = 0;
        if (i < pending) {
            v = list[i];
            const std::uint32_t s = p.succ_v[v];
            if (ldv(p.conn[s]) < level) {
                p.key_f[v] = (ldv(p.key_f[s]) + p.succ_wf[v]) - p.lam_f[p.R == 1 ? 0u : __ldg(&p.reg[v])];
                p.conn[v] = level;
            } else {
                pend = true;
            }
        }
        const std::uint64_t slot = block_append(pend, ring);
        if (pend)
            p.rem[cur ^ 1][slot] = v;
    }
}

// The float propagation without grid barriers: each thread owns up to 32
// pending vertices (i = tid + j * threads) and keeps polling all of them,
// valuing a vertex as soon as its successor is valued (acquire on conn, then
// release). Chains resolve from the anchor; since no thread ever blocks on
// one vertex, no vertex waits on work queued behind it. A bounded number of
// empty polls turns a broken tree into the nonconv error instead of a hang.
__device__ __forceinline__ unsigned ld_acquire(const std::uint32_t* a) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(std::uint32_t* a, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

#ifndef OCM_ASYNC_PER_THREAD
#define OCM_ASYNC_PER_THREAD 16
#endif
constexpr int kAsyncPerThread = OCM_ASYNC_PER_THREAD;

__device__ __forceinline__ void ph_fprop_async(const KP& p, int cur, std::uint64_t pending,
                                               std::uint32_t level) {
    const std::uint64_t tid = gtid(), nth = gstride();
    const std::uint32_t* list = p.rem[cur];
    // the thread's vertices and their successors stay in registers (constant
    // indices after unrolling), so a poll is one acquire load per vertex
    std::uint32_t vv[kAsyncPerThread], ss[kAsyncPerThread];
    unsigned todo = 0;
#pragma unroll
    for (int j = 0; j < kAsyncPerThread; ++j) {
        vv[j] = ss[j] = 0;
        if (tid + j * nth < pending) {
            vv[j] = list[tid + j * nth];
            ss[j] = p.succ_v[vv[j]];
            todo |= 1u << j;
        }
    }
    long long idle = 0;
    while (todo) {
        bool progress = false;
#pragma unroll
        for (int j = 0; j < kAsyncPerThread; ++j) {
            if (!(todo >> j & 1u))
                continue;
            if (ld_acquire(&p.conn[ss[j]]) == NONE)
                continue;
            const std::uint32_t v = vv[j];
            const double ks = __ldcg(&p.key_f[ss[j]]);
            p.key_f[v] = (ks + p.succ_wf[v]) - p.lam_f[p.R == 1 ? 0u : __ldg(&p.reg[v])];
            st_release(&p.conn[v], level);
            todo &= ~(1u << j);
            progress = true;
        }
        if (!progress) {
            __nanosleep(100);
            if (++idle > (1ll << 25)) { // seconds without progress: not a tree
                p.c->nonconv = 1;
                return;
            }
        } else {
            idle = 0;
        }
    }
}

// ------------------------------------------------------------ the kernel
//
// Control decisions are taken by every thread from values that are
// identical grid-wide: ring counts read after a barrier, stamped flags read
// after a barrier and not written again until one barrier later (two slots,
// alternating), and thread-local loop state. A flag read right after a
// barrier is never written in the phase that follows it.

// mode: kSolveFull runs a whole solve. The sharded lane splits every
// iteration at its one exchange point: kShardBegin initialises and runs the
// first improvement pass over the rank's own vertices; the host then
// all-gathers the policy slices and max-reduces the region flags, and each
// kShardResume recounts the policy in-degrees on the full (replicated)
// policy, runs the rest of the iteration replicated, and the next owned
// improvement pass -- or finishes (Ctl::shard_done). Loop state survives in
// the control block between launches.
constexpr int kSolveFull = 0, kShardBegin = 1, kShardResume = 2;
// kShardFused: the whole sharded solve in one launch per rank -- changed
// policy entries are stored into the peers' replicas during the improvement
// pass and two cross-rank barriers per iteration (system-scope atomics on
// the peers' barrier words) replace the host exchange.
constexpr int kShardFused = 3;

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* a) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

// Cross-phase state of the kernel's loop.
struct LoopState {
    Ring ra, rl, rc; // active-region counts, lists, core list
    unsigned stamp, k_hint, k_streak, xepoch, passes, outer, rounds, verifies, layers, nsync;
    unsigned long long peeled, cored, done_base;
    long long clk0, clk_last;
    int it;
};

// One kernel per (lane mode, improvement group width G): each instantiation
// carries only its own improvement variant, so ptxas allocates registers for
// that one (a kernel holding all variants spilled inside the pass's loop).
// G in {1, 2, 4, 8}: degrees above 128*G take the block-cooperative path.
// OCM_GBAR=1 (default): the kernel's own release/acquire grid barrier;
// 0: cooperative_groups grid.sync() (2-4% slower per solve,
// profiles/r02/ab_gbar_r02.log)
#ifndef OCM_GBAR
#define OCM_GBAR 1
#endif

template <int MODE, int G, int SR = 2>
__global__ void __launch_bounds__(kBlock, kSolveMinBlocks) k_solve(KP p, int mode) {
    constexpr bool EXACT = MODE != 0;
#if !OCM_GBAR
    cg::grid_group grid = cg::this_grid();
#endif
    Ctl* const c = p.c;
    __shared__ LoopState s_park;
    LoopState st;
    st.ra.init(c->ring[0]);
    st.rl.init(c->ring[1]);
    st.rc.init(c->ring[2]);
    st.nsync = 0;
    st.clk0 = st.clk_last = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0)
        st.clk_last = st.clk0 = clock64();
    // per-phase clocks of block 0 accumulate in shared memory (a global
    // read-modify-write right after every barrier would delay block 0, and
    // with it the next barrier); written out once at the end of the launch
    __shared__ long long s_clk[PH_COUNT];
    if (threadIdx.x < PH_COUNT)
        s_clk[threadIdx.x] = 0;
    if (MODE == 1 && p.staged)
        staged_init(*reinterpret_cast<Staged*>(dyn_smem));
    auto sync = [&](int ph) {
#if OCM_GBAR
        // arrive (release) / wait (acquire) on a per-launch counter (zeroed
        // with the per-solve Ctl fields): the k-th barrier completes when
        // the counter reaches k * gridDim.x; the CTA barriers on both sides
        // extend each side to the whole block
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned target = (st.nsync + 1) * gridDim.x;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&c->gbar) : "memory");
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&c->gbar) : "memory");
            } while (static_cast<int>(v - target) < 0);
        }
        __syncthreads();
#else
        grid.sync();
#endif
        ++st.nsync;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const long long t = clock64();
            s_clk[ph] += t - st.clk_last;
            st.clk_last = t;
        }
    };
    // cross-rank barrier of the fused sharded lane, called right after a
    // grid barrier (every CTA of this rank is through the previous phase and
    // has fenced its peer stores at system scope before arriving there): the
    // leader publishes (system fence) and bumps every rank's barrier word,
    // waits for all ranks' bumps, and one more grid barrier releases the
    // rank. A bounded wait turns a missing peer into an error instead of a
    // hang. Returns false (uniformly) on timeout.
    auto xsignal = [&](int ph) -> bool {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            __threadfence_system();
            const unsigned target = (++st.xepoch) * static_cast<unsigned>(p.world);
            for (int q = 0; q < p.world; ++q)
                atomicAdd_system(p.peer_xbar[q], 1u);
            long long idle = 0;
            while (ld_acquire_sys(p.xbar) < target) {
                __nanosleep(64);
                if (++idle > (1ll << 26)) {
                    c->xfail = 1;
                    break;
                }
            }
            __threadfence_system();
        } else {
            ++st.xepoch; // every thread's copy stays in step
        }
        sync(ph);
        return ldr(c->xfail) == 0;
    };
    const int K_max = max(1, ceil_log2_d(max(p.max_region, 2u)));
    st.stamp = ldr(c->stamp);
    st.k_hint = max(1u, min(ldr(c->k_hint), static_cast<unsigned>(K_max)));
    st.k_streak = ldr(c->k_streak);
    st.xepoch = ldr(c->xepoch);
    // per-solve counters continue across the launches of a sharded solve
    st.passes = ldr(c->passes);
    st.outer = ldr(c->outer);
    st.rounds = ldr(c->rounds);
    st.verifies = ldr(c->verifies);
    st.layers = ldr(c->layers);
    st.peeled = ldr(c->peeled);
    st.cored = ldr(c->cored);
    st.done_base = ldr(c->done);
    st.it = static_cast<int>(ldr(c->it));
    bool fatal = false;  // uniform: a fixpoint failed to converge
    bool paused = false; // uniform: sharded launch ends at its exchange point

    if (mode != kShardResume) {
        ph_init<MODE>(p);
        sync(PH_INIT);
    }
    bool skip_improve = mode == kShardResume;
    if (mode == kShardResume) {
        // every block must have read the ring bases above before any block
        // appends (the first phase of a resumed launch appends at once)
        sync(PH_INIT);
    }

    for (;; ++st.it) {
        if (!skip_improve) {
            // fused lane: every rank finished the previous iteration (whose
            // replicated phases write the policy) before anyone pushes; the
            // previous phase ended with a grid barrier
            if (mode == kShardFused && !xsignal(PH_IMPROVE)) {
                fatal = true;
                break;
            }
            // park the loop state (block-uniform) in shared memory while the
            // pass runs: otherwise ptxas keeps it in registers across the
            // pass and spills the pass's own working set inside its loop
            __syncthreads();
            if (threadIdx.x == 0)
                s_park = st;
            __syncthreads();
            asm volatile("" ::: "memory");
            improve_phase<MODE, G, 4>(p, p.changed[s_park.it & 1]);
            asm volatile("" ::: "memory");
            st = s_park;
            ++st.passes;
            if (mode == kShardFused)
                __threadfence_system(); // this thread's policy/flag pushes, before arriving
            sync(PH_IMPROVE);
            if (mode == kShardBegin || mode == kShardResume) {
                paused = true;
                break;
            }
            // fused lane: wait until every rank's pushes are visible
            if (mode == kShardFused && !xsignal(PH_IMPROVE)) {
                fatal = true;
                break;
            }
        }
        skip_improve = false;
        const int par = st.it & 1;
        if (!p.indeg_in_improve) {
            // the policy of the other ranks arrived by the exchange: count
            // in-degrees over the full policy (replicated on every rank)
            for (std::size_t v = gtid(); v < p.N; v += gstride())
                if (p.changed[par][__ldg(&p.reg[v])])
                    mark_pred(p, p.succ_v[v]);
            sync(PH_CLASSIFY);
        }
        ph_classify<MODE>(p, par, st.ra, st.rl, st.rc);
        sync(PH_CLASSIFY);
        const std::uint64_t n_active = st.ra.take();
        const std::uint64_t nL = st.rl.take();
        const std::uint64_t nC = st.rc.take();
        // written only by improve/adopt/keep/attach, never by the rounds
        // that follow: every block reads the same values here
        const int4 fl = ldr4(&c->error); // error, overflow, lambda_up, nonconv
        if (n_active == 0 || fl.x || fl.y || fl.z)
            break; // quiet pass (or a failure the host reports)
        ++st.outer;
        st.peeled += nL;
        st.cored += nC;

        // ---- pointer doubling on the core, verified exactly (round 1 was
        // done by the classification)
        int in = 1, k = 1;
        ++st.rounds;
        bool first_try = true, voted = false;
        std::uint64_t nM = 0;
        for (;;) {
            // all doubling passes but the last, S steps each
            constexpr int S = kRoundS ? kRoundS : SR;
            for (; static_cast<int>(st.k_hint) - k > S; in ^= 1) {
                ph_round_multi<S>(p, nC, in);
                k += S;
                st.rounds += S;
                sync(PH_ROUND);
            }
            const unsigned stamp = ++st.stamp;
            ++st.verifies;
            unsigned* vflag = &c->vfail[stamp & 1];
            // the last pass (one or two steps) marks as it goes
            const int last = static_cast<int>(st.k_hint) - k;
            if (S >= 3 && last == 3) {
                ph_round_mark<(S >= 3 ? 3 : 2)>(p, nC, in, stamp, EXACT, st.rl);
            } else if (last == 2) {
                ph_round_mark<2>(p, nC, in, stamp, EXACT, st.rl);
            } else if (last == 1) {
                ph_round_mark<1>(p, nC, in, stamp, EXACT, st.rl);
            } else {
                ph_mark(p, nC, in, stamp, EXACT, st.rl);
            }
            if (last > 0) {
                k += last;
                st.rounds += last;
                in ^= 1;
            }
            sync(PH_VERIFY);
            nM = st.rl.take(); // |M|, listed in wlist
            if (EXACT && p.R == 1 && nM <= kBlock) {
                // few cycle vertices, one region: block 0 checks and, if the
                // check passes, votes, adopts and values the winning cycle
                // in the same phase
                if (blockIdx.x == 0)
                    ph_vote_one_block<MODE>(p, nM, stamp, p.pj[in], vflag);
                sync(PH_VOTE); // (phase clock: the one-block check+vote)
                if (ldr(*vflag) != stamp) {
                    voted = true;
                    break;
                }
            } else {
                ph_check<MODE>(p, nM, stamp, vflag, st.rc, p.pj[in]);
                sync(PH_VERIFY);
                const std::uint64_t s_size = st.rc.take();
                if (ldr(*vflag) != stamp && s_size == nM)
                    break;
            }
            if (k >= K_max) {
                fatal = true;
                break;
            }
            st.k_hint = k + 1;
            first_try = false;
        }
        if (fatal)
            break;
        // adapt the starting round count: shrink after two first-try passes
        if (first_try && ++st.k_streak >= kKShrink && k > 1) {
            st.k_hint = k - 1;
            st.k_streak = 0;
        } else {
            st.k_hint = k;
            if (!first_try)
                st.k_streak = 0;
        }
        const unsigned stamp = st.stamp;

        // ---- vote, adoption and the winning cycles' values (done with the
        // check above when the cycle vertices are few)
        if (!voted) {
            if constexpr (!EXACT) {
                ph_stats_float(p, nM);
                sync(PH_STATS);
            }
            if (nM <= kVoteOneBlock) {
                if (blockIdx.x == 0)
                    ph_vote_one_block<MODE>(p, nM, stamp, p.pj[in]);
            } else {
                ph_vote<MODE>(p, nM, stamp, st.done_base);
                st.done_base += gridDim.x;
            }
            sync(PH_VOTE);
        }
        if (EXACT && ldr(c->wc_big[stamp & 1]) == stamp) {
            const std::uint64_t nW = static_cast<std::uint32_t>(ldr(c->wc_n[stamp & 1]));
            const unsigned maxlen = ldr(c->wc_len[stamp & 1]);
            const int wr = ceil_log2_d(maxlen > 1 ? maxlen - 1 : 1);
            for (int j = 0; j < wr; ++j) {
                wc_round<MODE>(p, p.rem[1], nW, j, gtid(), gstride());
                sync(PH_WINCYC);
            }
            wc_final<MODE>(p, p.rem[1], nW, wr, gtid(), gstride());
            sync(PH_WINCYC);
        }

        // ---- kept component (core, then leaves), re-attachment
        ph_keep<MODE>(p, nC, nL, in, stamp, 1ull << k, st.rl);
        sync(PH_KEEP);
        std::uint64_t pending = st.rl.take();
        int cur = 0;
        for (std::uint32_t layer = 1; pending > 0; ++layer) {
            ph_attach<MODE>(p, cur, pending, layer, st.rl);
            sync(PH_ATTACH);
            const std::uint64_t next = st.rl.take();
            ++st.layers;
            if (next == pending) { // connect_gpi_fixpoint: not strongly connected
                fatal = true;
                break;
            }
            pending = next;
            cur ^= 1;
        }
        if (fatal)
            break;

        if constexpr (!EXACT) {
            ph_fprop_init(p, nC, nL, st.rl);
            sync(PH_FLOAT);
            std::uint64_t fpend = st.rl.take();
            int fcur = 0;
            std::uint32_t level = 1;
            // level-synchronous while the pending list is long, then
            // barrier-free (up to kAsyncPerThread pending vertices per thread)
            for (; fpend > kAsyncPerThread * gstride(); ++level) {
                ph_fprop_level(p, fcur, fpend, level, st.rl);
                sync(PH_FLOAT);
                ++st.layers;
                const std::uint64_t next = st.rl.take();
                if (next == fpend) { // no progress: not a tree into the anchor
                    fatal = true;
                    break;
                }
                fpend = next;
                fcur ^= 1;
            }
            if (fatal)
                break;
            if (fpend > 0) {
                ph_fprop_async(p, fcur, fpend, level);
                sync(PH_FLOAT);
                ++st.layers;
                if (ldr(c->nonconv))
                    fatal = true;
            }
            if (fatal)
                break;
        }
        // debug trace (sessions created with OCM_TRACE_ITERS): the policy and
        // the value plane after this iteration, as HowardTrace records them
        // (howard_par.hpp:588)
        if (p.tr_pol && st.outer - 1 < p.tr_iters) {
            const std::size_t base = std::size_t(st.outer - 1) * p.N;
            for (std::size_t v = gtid(); v < p.N; v += gstride()) {
                p.tr_pol[base + v] = p.succ_e[v];
                if constexpr (EXACT)
                    p.tr_key[base + v] = static_cast<long long>(key_ld<MODE>(p, static_cast<std::uint32_t>(v)));
                else
                    p.tr_keyf[base + v] = p.key_f[v];
            }
            sync(PH_FLOAT); // before the next pass rewrites the policy
        }
    }

    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (fatal)
            c->nonconv = 1;
        c->it = static_cast<unsigned>(st.it);
        c->shard_done = paused ? 0 : 1;
        c->stamp = st.stamp;
        c->k_hint = st.k_hint;
        c->k_streak = st.k_streak;
        c->xepoch = st.xepoch;
        c->passes = st.passes;
        c->outer = st.outer;
        c->rounds = st.rounds;
        c->verifies = st.verifies;
        c->peeled = st.peeled;
        c->cored = st.cored;
        c->layers = st.layers;
        c->syncs = st.nsync;
        c->clk_total += clock64() - st.clk0;
        for (int ph = 0; ph < PH_COUNT; ++ph)
            c->clk[ph] += s_clk[ph];
    }
}

} // namespace
} // namespace ocmb
