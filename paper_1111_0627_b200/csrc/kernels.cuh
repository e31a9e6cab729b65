// Device kernels of the policy-iteration lane (included by solver.cu only).
//
// One host iteration mirrors proj/include/ocm/howard_par.hpp:555-590 (run()):
//
//   k_improve        policy improvement over the CSR      howard_par.hpp:146 spf_pass_iter
//   k_region_check   per-region termination               howard_par.hpp:189/208
//   k_pj_*           cycle detection on the functional    howard_par.hpp:249/301
//                    policy graph by pointer doubling      (elimination + cycleIdentification)
//   k_cycle_stats    per-cycle (length, weight) segmented  howard_par.hpp:319
//                    reduction, exact integers
//   k_vote/k_adopt   per-region min (mean, anchor) vote    howard_par.hpp:56/339
//   k_wincyc_*       values on the winning cycle (prefix   howard_par.hpp:494
//                    sum by pointer jumping, cycle only)    valuePropagate
//   k_keep           kept component = policy paths into    howard_par.hpp:370/393
//                    the winning cycle, + their values      (+ valuePropagate)
//   k_attach         breadth-layered re-attachment, +      howard_par.hpp:433
//                    values of re-attached vertices         (+ valuePropagate)
//
// Results are identical to the reference's (same lambda sequence, policy,
// cycle and scalar values): every kernel computes the same function as the
// reference step it replaces, with a data-parallel schedule (DESIGN.md gives
// the argument per kernel). Exact mode keeps a vertex value as the integer
// key K = value * den (den = the region lambda's reduced denominator), so
// improvement candidates are K[t] + w*den - num and all comparisons are exact.
//
// Contention rule used throughout: no kernel lets many threads store to one
// address. Flags are OR-reduced per block (__syncthreads_or) and stored once
// per block; list appends reserve space with one atomic per block; scatters
// that may collide check the target before writing.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "devcommon.cuh"

namespace ocmb {
namespace {

__device__ __forceinline__ bool working(const KP& p, std::uint32_t v) {
    return p.active[p.reg[v]] != 0;
}

__device__ __forceinline__ std::size_t gtid() {
    return blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
}
__device__ __forceinline__ std::size_t gstride() { return std::size_t(gridDim.x) * blockDim.x; }

// Set *flag to 1 unless it already is (read first: avoids store storms).
__device__ __forceinline__ void set_flag(int* flag) {
    if (__ldcg(flag) == 0)
        *flag = 1;
}
__device__ __forceinline__ void set_flag(unsigned* flag) {
    if (__ldcg(flag) == 0u)
        *flag = 1u;
}

// Block-wide append: every thread of the block must call it (block-uniform
// loops). Returns this thread's slot (valid when take) after reserving the
// block's total with one atomic.
__device__ __forceinline__ unsigned block_append(bool take, unsigned* counter) {
    __shared__ unsigned s_cnt[kBlock / 32];
    __shared__ unsigned s_base;
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
        s_base = tot ? atomicAdd(counter, tot) : 0u;
    }
    __syncthreads();
    const unsigned slot = s_base + s_cnt[warp] + __popc(bal & ((1u << lane) - 1u));
    __syncthreads();
    return slot;
}

// ------------------------------------------------------------ init

__global__ void k_init(KP p) {
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        p.succ_e[v] = NONE;
        p.succ_v[v] = NONE;
        if (p.key_i)
            p.key_i[v] = 0;
        if (p.key_f)
            p.key_f[v] = 0.0;
        p.mark[v] = 0;
        p.mark2[v] = 0;
    }
    for (std::size_t r = gtid(); r <= p.R; r += gstride()) { // slot R: trivial vertices
        p.lam_num[r] = 0;
        p.lam_den[r] = 1;
        p.lam_f[r] = 0.0;
        p.active[r] = r < p.R ? 1 : 0;
        p.changed[r] = 0;
        p.slot[r] = EMPTY;
        p.src[r] = NONE;
        p.iters[r] = 0;
    }
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

template <int G> __device__ __forceinline__ unsigned group_mask() {
    if constexpr (G == 32)
        return FULL;
    else
        return ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
}

// Region "changed" bookkeeping with at most one store per block per region.
struct ChangedMarks {
    std::uint32_t first = NONE;
    std::uint32_t last_direct = NONE;
    __device__ __forceinline__ void note(const KP& p, std::uint32_t r) {
        if (first == NONE)
            first = r;
        else if (r != first && r != last_direct) {
            last_direct = r;
            set_flag(&p.changed[r]);
        }
    }
    __device__ __forceinline__ void flush(const KP& p) {
        __shared__ std::uint32_t s_r;
        if (threadIdx.x == 0)
            s_r = NONE;
        __syncthreads();
        if (first != NONE) {
            const std::uint32_t prev = atomicCAS(&s_r, NONE, first);
            if (prev != NONE && prev != first)
                set_flag(&p.changed[first]);
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_r != NONE)
            set_flag(&p.changed[s_r]);
    }
};

template <bool EXACT, int G, int U> __global__ void __launch_bounds__(kBlock) k_improve(KP p) {
    const unsigned lane = threadIdx.x & (G - 1);
    const unsigned gm = group_mask<G>();
    const std::size_t gid = gtid() / G;
    const std::size_t gs = gstride() / G;
    ChangedMarks marks;
    using Key = typename std::conditional<EXACT, long long, double>::type;
    for (std::size_t vv = gid; vv < p.N; vv += gs) {
        const std::uint32_t v = static_cast<std::uint32_t>(vv);
        const std::uint32_t b = p.row[v], e_end = p.row[v + 1];
        const std::uint32_t r = p.reg[v];
        const std::uint32_t cur = p.succ_e[v];
        if (!p.active[r])
            continue;
        long long num = 0, den = 1;
        double lam = 0.0;
        if constexpr (EXACT) {
            num = p.lam_num[r];
            den = p.lam_den[r];
        } else {
            lam = p.lam_f[r];
        }
        Key best = 0, curc = 0;
        std::uint32_t be = NONE, bt = 0;
        int bwi = 0;
        double bwf = 0.0;
        bool have_cur = false;
        for (std::uint32_t e0 = b + lane; e0 < e_end; e0 += G * U) {
            std::uint32_t tt[U];
            Key kk[U];
            int wi[U];
            double wf[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const std::uint32_t e = e0 + u * G;
                if (e < e_end) {
                    if constexpr (EXACT) {
                        const int2 ed = __ldg(&p.ew[e]);
                        tt[u] = static_cast<std::uint32_t>(ed.x);
                        wi[u] = ed.y;
                    } else {
                        const FEdge ed = p.fe[e];
                        tt[u] = ed.t;
                        wf[u] = ed.w;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (e0 + u * G < e_end) {
                    if constexpr (EXACT)
                        kk[u] = __ldg(&p.key_i[tt[u]]);
                    else
                        kk[u] = __ldg(&p.key_f[tt[u]]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const std::uint32_t e = e0 + u * G;
                if (e < e_end) {
                    Key c;
                    if constexpr (EXACT)
                        c = kk[u] + static_cast<long long>(wi[u]) * den - num;
                    else
                        c = (kk[u] + wf[u]) - lam; // FloatMode::extend (policy.hpp:105)
                    if (be == NONE || c < best) {
                        best = c;
                        be = e;
                        bt = tt[u];
                        if constexpr (EXACT)
                            bwi = wi[u];
                        else
                            bwf = wf[u];
                    }
                    if (e == cur) {
                        curc = c;
                        have_cur = true;
                    }
                }
            }
        }
        Key gbest = best;
        std::uint32_t gbe = be;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            const Key ob = __shfl_xor_sync(gm, gbest, off, G);
            const std::uint32_t oe = __shfl_xor_sync(gm, gbe, off, G);
            if (oe != NONE && (gbe == NONE || ob < gbest || (ob == gbest && oe < gbe))) {
                gbest = ob;
                gbe = oe;
            }
            const Key oc = __shfl_xor_sync(gm, curc, off, G);
            const bool oh = __shfl_xor_sync(gm, have_cur ? 1 : 0, off, G) != 0;
            if (oh) {
                curc = oc;
                have_cur = true;
            }
        }
        if (gbe == NONE) {
            if (lane == 0)
                p.flags->error = 1;
            continue;
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
        if (rep && gbe == be) { // owner lane of the winning edge
            p.succ_e[v] = be;
            p.succ_v[v] = bt;
            if constexpr (EXACT)
                p.succ_wi[v] = bwi;
            else
                p.succ_wf[v] = bwf;
            marks.note(p, r);
        }
    }
    marks.flush(p);
}

// Regions whose pass changed nothing are finished (howard_par.hpp:189).
__global__ void k_region_check(KP p) {
    for (std::size_t r = gtid(); r < p.R; r += gstride()) {
        if (p.active[r]) {
            if (p.changed[r])
                atomicAdd(&p.flags->active_count, 1u);
            else
                p.active[r] = 0;
        }
        p.changed[r] = 0;
    }
}

// ------------------------------------------------------------ cycles
//
// Pointer doubling on the functional policy graph. pj[v] = (jump target,
// least vertex on the jumped segment, weight sum of the segment). All
// segments have the same length L = 2^k (synchronous doubling). Once
// L >= tail + cycle length for every vertex, jump(v) lies on v's cycle and
// the least vertex of jump(v)'s segment is the least vertex of that cycle:
// the anchor of v's component (howard_par.hpp:310 cycle_anchor, minIndex),
// and the image of succ^L is exactly the set of cycle vertices (the
// survivors of the reference's elimination fixpoint, howard_par.hpp:249).
// The round count is not fixed at log2(n): k_cycle_verify checks the two
// conditions exactly and the host adds rounds until it holds.
// Regions are closed under succ, so rounds run without region checks.

template <bool EXACT> __global__ void k_pj_init(KP p) {
    if (*(volatile unsigned*)&p.flags->active_count == 0)
        return; // quiet pass: no region left
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        PJC x;
        const std::uint32_t sv = p.succ_v[v];
        x.nxt = sv == NONE ? static_cast<std::uint32_t>(v) : sv; // trivial vertices: self
        x.mn = static_cast<std::uint32_t>(v);
        x.w = EXACT ? static_cast<long long>(p.succ_wi[v]) : 0ll;
        p.pj[0][v] = x;
    }
}

__global__ void k_pj_round(KP p, int in) {
    if (*(volatile unsigned*)&p.flags->active_count == 0)
        return; // quiet pass: no region left
    const PJC* __restrict__ a = p.pj[in];
    PJC* __restrict__ o = p.pj[in ^ 1];
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        const PJC x = a[v];
        const PJC y = a[x.nxt];
        PJC z;
        z.nxt = y.nxt;
        z.mn = min(x.mn, y.mn);
        z.w = x.w + y.w;
        o[v] = z;
    }
}

__global__ void k_cycle_mark(KP p, int in, std::uint32_t stamp) {
    if (*(volatile unsigned*)&p.flags->active_count == 0)
        return; // quiet pass: no region left
    const PJC* a = p.pj[in];
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        if (!working(p, v))
            continue;
        const std::uint32_t j = a[v].nxt;
        p.comp[v] = a[j].mn;
        if (p.mark[j] != stamp) // many vertices share j: read before writing
            p.mark[j] = stamp;
        p.cyc_len[v] = 0;
        if (p.cyc_wi)
            p.cyc_wi[v] = 0;
    }
}

// Exact check of the round count. M = image of succ^L. Passes iff every
// vertex of M has a predecessor in M (so M has no tail vertex, i.e. L >=
// every tail) and comp is constant along succ inside M (so every window of
// length L covers its whole cycle, i.e. L >= every cycle length).
__global__ void k_cycle_verify1(KP p, std::uint32_t stamp) {
    if (*(volatile unsigned*)&p.flags->active_count == 0)
        return; // quiet pass: no region left
    bool fail = false;
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        if (p.mark[v] != stamp || !working(p, v))
            continue;
        const std::uint32_t s = p.succ_v[v];
        fail |= p.comp[s] != p.comp[v];
        if (p.mark2[s] != stamp)
            p.mark2[s] = stamp;
    }
    if (__syncthreads_or(fail) && threadIdx.x == 0)
        set_flag(&p.flags->verify_fail);
}

__global__ void k_cycle_verify2(KP p, std::uint32_t stamp) {
    if (*(volatile unsigned*)&p.flags->active_count == 0)
        return; // quiet pass: no region left
    bool fail = false;
    for (std::size_t v = gtid(); v < p.N; v += gstride())
        fail |= p.mark[v] == stamp && p.mark2[v] != stamp && working(p, v);
    if (__syncthreads_or(fail) && threadIdx.x == 0)
        set_flag(&p.flags->verify_fail);
}

// Segmented reduction of (length, weight) per cycle, keyed by anchor.
// Exact integers, so the atomic order is irrelevant to the result. When a
// warp's cycle vertices share one anchor (the common single-giant-cycle
// case) the warp pre-reduces and issues one atomic pair.
__global__ void k_cycle_stats(KP p, std::uint32_t stamp) {
    const unsigned lane = threadIdx.x & 31;
    const std::size_t wid = gtid() >> 5;
    const std::size_t ws = gstride() >> 5;
    for (std::size_t base = wid * 32; base < p.N; base += ws * 32) {
        const std::size_t v = base + lane;
        const bool on = v < p.N && p.mark[v] == stamp && working(p, v);
        const unsigned am = __ballot_sync(FULL, on);
        if (!am)
            continue;
        const std::uint32_t a = on ? p.comp[v] : 0u;
        const int lead = __ffs(am) - 1;
        const std::uint32_t a0 = __shfl_sync(FULL, a, lead);
        const bool uni = __all_sync(FULL, !on || a == a0);
        long long w = on ? static_cast<long long>(p.succ_wi[v]) : 0ll;
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

// Float mode: each anchor walks its own cycle from itself, summing weights
// in the reference's order (howard_par.hpp:323), so means are bit-identical.
__global__ void k_cycle_walk_float(KP p) {
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        if (p.comp[v] != v || !working(p, v))
            continue;
        double s = 0.0;
        std::uint32_t len = 0, u = static_cast<std::uint32_t>(v);
        do {
            s += p.succ_wf[u];
            ++len;
            u = p.succ_v[u];
        } while (u != v);
        p.cyc_wf[v] = s;
        p.cyc_len[v] = len;
    }
}

template <bool EXACT>
__device__ __forceinline__ bool rec_less(const KP& p, std::uint32_t a, std::uint32_t b) {
    if constexpr (EXACT) {
        const __int128 l = static_cast<__int128>(p.cyc_wi[a]) * p.cyc_len[b];
        const __int128 r = static_cast<__int128>(p.cyc_wi[b]) * p.cyc_len[a];
        if (l != r)
            return l < r;
    } else {
        const double ma = p.cyc_wf[a] / p.cyc_len[a];
        const double mb = p.cyc_wf[b] / p.cyc_len[b];
        if (ma < mb)
            return true;
        if (mb < ma)
            return false;
    }
    return a < b;
}

// Region-specific minimum voting (howard_par.hpp:56 vote_min; paper Alg. 5):
// a holder is replaced only by a strictly smaller (mean, anchor) record.
template <bool EXACT> __global__ void k_vote(KP p) {
    for (std::size_t vv = gtid(); vv < p.N; vv += gstride()) {
        const std::uint32_t v = static_cast<std::uint32_t>(vv);
        if (p.comp[v] != v || !working(p, v))
            continue;
        unsigned long long* cell = &p.slot[p.reg[v]];
        unsigned long long cur = *(volatile unsigned long long*)cell;
        for (;;) {
            if (cur != EMPTY && !rec_less<EXACT>(p, v, static_cast<std::uint32_t>(cur)))
                break;
            const unsigned long long prev = atomicCAS(cell, cur, v);
            if (prev == cur)
                break;
            cur = prev;
        }
    }
}

__device__ __forceinline__ long long gcd_ll(long long a, long long b) {
    if (a < 0)
        a = -a;
    while (b) {
        const long long t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Host-side adoption step of howard_par.hpp:349-364, per region on device.
template <bool EXACT> __global__ void k_adopt(KP p) {
    for (std::size_t r = gtid(); r < p.R; r += gstride()) {
        if (!p.active[r])
            continue;
        const unsigned long long a = p.slot[r];
        p.slot[r] = EMPTY;
        if (a == EMPTY) {
            p.flags->error = 1;
            continue;
        }
        p.src[r] = static_cast<std::uint32_t>(a);
        atomicMax(&p.flags->max_cycle, p.cyc_len[a]);
        if constexpr (EXACT) {
            long long num = p.cyc_wi[a], den = p.cyc_len[a];
            const long long g = gcd_ll(num, den);
            if (g > 1) {
                num /= g;
                den /= g;
            }
            if (p.iters[r] > 0 &&
                static_cast<__int128>(p.lam_num[r]) * den < static_cast<__int128>(num) * p.lam_den[r])
                p.flags->lambda_up = 1;
            p.lam_num[r] = num;
            p.lam_den[r] = den;
            const __int128 step =
                static_cast<__int128>(p.max_abs_w) * den + (num < 0 ? -num : num);
            if (static_cast<__int128>(p.max_region) * step >= (static_cast<__int128>(1) << 62))
                p.flags->overflow = 1;
        } else {
            p.lam_f[r] = p.cyc_wf[a] / p.cyc_len[a];
        }
        p.iters[r] += 1;
    }
}

// ------------------------------------------------------------ values
//
// Value determination (howard_par.hpp:494 valuePropagate) without a separate
// propagation fixpoint. With K = value * den, the reference computes
// K(u) = K(succ u) + w*den - num along the rebuilt policy tree rooted at the
// winning anchor. Three cases, all exact integer arithmetic:
//  * winning-cycle vertices: a pointer-jumping prefix sum over the cycle
//    vertices only, cut at the anchor (k_wincyc_*);
//  * other kept vertices (their policy path enters the winning cycle): the
//    doubling above already summed the weights of the length-L walk from v
//    to jump(v) on the cycle; since the cycle's reduced weight is exactly 0,
//    K(v) = W_L(v)*den - L*num + K(jump(v)) (k_keep);
//  * re-attached vertices: K(x) = K(t) + w*den - num at attachment, t being
//    connected in an earlier layer (k_attach).

__global__ void k_wincyc_init(KP p, std::uint32_t stamp) {
    for (std::size_t base = blockIdx.x * std::size_t(kBlock); base < p.N;
         base += gridDim.x * std::size_t(kBlock)) {
        const std::size_t v = base + threadIdx.x;
        bool take = false;
        std::uint32_t r = 0;
        if (v < p.N && p.mark[v] == stamp && working(p, v)) {
            r = p.reg[v];
            take = p.comp[v] == p.src[r];
        }
        const unsigned slot = block_append(take, &p.flags->wc_count);
        if (take) {
            p.wlist[slot] = static_cast<std::uint32_t>(v);
            PJV x;
            const std::uint32_t root = p.src[r];
            if (v == root) {
                x.acc = 0;
                x.nxt = root;
            } else {
                x.acc = static_cast<long long>(p.succ_wi[v]) * p.lam_den[r] - p.lam_num[r];
                x.nxt = p.succ_v[v];
            }
            x.root = root;
            p.pv[0][v] = x;
        }
    }
}

__global__ void k_wincyc_round(KP p, int round) {
    if (round > 0 && *(volatile unsigned*)&p.flags->notdone[round - 1] == 0)
        return;
    const int in = round & 1;
    const PJV* __restrict__ a = p.pv[in];
    PJV* __restrict__ o = p.pv[in ^ 1];
    const unsigned cnt = p.flags->wc_count;
    bool nd = false;
    for (std::size_t i = gtid(); i < cnt; i += gstride()) {
        const std::uint32_t c = p.wlist[i];
        const PJV x = a[c];
        const PJV y = a[x.nxt];
        PJV z;
        z.acc = x.acc + y.acc;
        z.nxt = y.nxt;
        z.root = x.root;
        o[c] = z;
        nd |= y.nxt != x.root;
    }
    if (__syncthreads_or(nd) && threadIdx.x == 0)
        set_flag(&p.flags->notdone[round]);
}

__global__ void k_wincyc_final(KP p, int rounds) {
    int last = rounds - 1;
    for (int j = 0; j < rounds; ++j)
        if (p.flags->notdone[j] == 0) {
            last = j;
            break;
        }
    if (p.flags->notdone[rounds - 1] != 0) {
        if (gtid() == 0)
            p.flags->wc_short = 1; // host re-runs with the exact round count
        return;
    }
    const PJV* a = p.pv[(last & 1) ^ 1];
    const unsigned cnt = p.flags->wc_count;
    for (std::size_t i = gtid(); i < cnt; i += gstride()) {
        const std::uint32_t c = p.wlist[i];
        p.key_i[c] = a[c].acc;
    }
}

__device__ __forceinline__ bool key_in_range(__int128 k) {
    const __int128 lim = static_cast<__int128>(1) << 62;
    return k < lim && k > -lim;
}

// Kept component: vertices whose policy path ends in the winning cycle keep
// their edges (howard_par.hpp:393 markMinComponent) and, in exact mode, get
// their values from the doubling sums; everyone else is queued for
// re-attachment.
template <bool EXACT>
__global__ void k_keep(KP p, int in, std::uint32_t stamp, unsigned long long L) {
    const PJC* a = p.pj[in];
    bool ovf = false;
    for (std::size_t base = blockIdx.x * std::size_t(kBlock); base < p.N;
         base += gridDim.x * std::size_t(kBlock)) {
        const std::size_t v = base + threadIdx.x;
        bool take = false;
        if (v < p.N && working(p, v)) {
            const std::uint32_t r = p.reg[v];
            const bool kept = p.comp[v] == p.src[r];
            p.conn[v] = kept ? 0u : NONE;
            take = !kept;
            if (EXACT && kept && p.mark[v] != stamp) {
                const PJC x = a[v];
                const __int128 k = static_cast<__int128>(x.w) * p.lam_den[r] -
                                   static_cast<__int128>(L) * p.lam_num[r] + p.key_i[x.nxt];
                ovf |= !key_in_range(k);
                p.key_i[v] = static_cast<long long>(k);
            }
        }
        const unsigned slot = block_append(take, &p.flags->rem_count[0]);
        if (take)
            p.rem[0][slot] = static_cast<std::uint32_t>(v);
    }
    if (__syncthreads_or(ovf) && threadIdx.x == 0)
        set_flag(&p.flags->overflow);
}

// One breadth layer of howard_par.hpp:433 connectGpi: a pending vertex
// attaches through its smallest out-edge whose head was connected in an
// earlier layer (conn < layer); connection stamps make the layer discipline
// exact regardless of schedule. Exact mode also sets the vertex's value.
template <bool EXACT> __global__ void k_attach(KP p, int in, unsigned n_in, std::uint32_t layer) {
    const std::uint32_t* list = p.rem[in];
    bool ovf = false;
    for (std::size_t base = blockIdx.x * std::size_t(kBlock); base < n_in;
         base += gridDim.x * std::size_t(kBlock)) {
        const std::size_t i = base + threadIdx.x;
        bool pending = false;
        std::uint32_t x = 0;
        if (i < n_in) {
            x = list[i];
            pending = true;
            const std::uint32_t b = p.row[x], e_end = p.row[x + 1];
            for (std::uint32_t e = b; e < e_end; ++e) {
                std::uint32_t t;
                if constexpr (EXACT)
                    t = static_cast<std::uint32_t>(p.ew[e].x);
                else
                    t = p.fe[e].t;
                if (p.conn[t] < layer) {
                    p.succ_e[x] = e;
                    p.succ_v[x] = t;
                    if constexpr (EXACT) {
                        const int w = p.ew[e].y;
                        p.succ_wi[x] = w;
                        const std::uint32_t r = p.reg[x];
                        const __int128 k = static_cast<__int128>(p.key_i[t]) +
                                           static_cast<__int128>(w) * p.lam_den[r] - p.lam_num[r];
                        ovf |= !key_in_range(k);
                        p.key_i[x] = static_cast<long long>(k);
                    } else {
                        p.succ_wf[x] = p.fe[e].w;
                    }
                    p.conn[x] = layer;
                    pending = false;
                    break;
                }
            }
        }
        const unsigned slot = block_append(pending, &p.flags->rem_count[in ^ 1]);
        if (pending)
            p.rem[in ^ 1][slot] = x;
    }
    if (__syncthreads_or(ovf) && threadIdx.x == 0)
        set_flag(&p.flags->overflow);
}

// Float mode: level-synchronous propagation from the anchor, one policy
// level per launch, each vertex computing (value(succ) + w) - lambda exactly
// as the reference does, so values are bit-identical.
__global__ void k_fprop_init(KP p) {
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        if (!working(p, v))
            continue;
        if (v == p.src[p.reg[v]]) {
            p.conn[v] = 0;
            p.key_f[v] = 0.0;
        } else {
            p.conn[v] = NONE;
        }
    }
}

__global__ void k_fprop_round(KP p, std::uint32_t level, int slot) {
    bool nd = false;
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        if (p.conn[v] != NONE || !working(p, v))
            continue;
        const std::uint32_t s = p.succ_v[v];
        if (p.conn[s] < level) {
            p.key_f[v] = (p.key_f[s] + p.succ_wf[v]) - p.lam_f[p.reg[v]];
            p.conn[v] = level;
        } else {
            nd = true;
        }
    }
    if (__syncthreads_or(nd) && threadIdx.x == 0)
        set_flag(&p.flags->notdone[slot]);
}

} // namespace
} // namespace ocmb
