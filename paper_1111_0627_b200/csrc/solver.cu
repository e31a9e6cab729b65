// B200 (sm_100a) policy-iteration solver for the optimal cycle mean.
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
//   k_keep           kept component = policy paths into    howard_par.hpp:370/393
//                    the winning cycle
//   k_attach         breadth-layered re-attachment         howard_par.hpp:433
//   k_prop_*         value determination by pointer        howard_par.hpp:494
//                    jumping along the policy tree
//
// Results are identical to the reference's (same lambda sequence, policy,
// cycle and scalar values): the kernels compute the same functions with
// different (data-parallel) schedules; see DESIGN.md for the argument per
// kernel. Exact mode keeps a vertex value as the integer key
// K = value * den (den = lambda's reduced denominator), so improvement
// candidates are K[t] + w*den - num and every comparison is exact.

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "errors.hpp"
#include "solver.hpp"

namespace ocmb {

namespace {

constexpr std::uint32_t NONE = 0xffffffffu;
constexpr unsigned long long EMPTY = ~0ull;
constexpr unsigned FULL = 0xffffffffu;
constexpr int kMaxRounds = 64;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

template <class T> struct DBuf {
    T* p = nullptr;
    std::size_t n = 0;
    void alloc(std::size_t k) {
        release();
        if (k)
            CK(cudaMalloc(&p, k * sizeof(T)));
        n = k;
    }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
};

struct __align__(16) FEdge {
    double w;
    std::uint32_t t;
    std::uint32_t pad;
};

struct Flags {
    unsigned active_count;
    unsigned rem_count[2];
    int error;          // structural (no successor / not strongly connected)
    int overflow;       // exact keys would leave int64
    int lambda_up;      // lambda increased inside a region
    unsigned notdone[kMaxRounds];
};

// Everything a kernel may touch, passed by value.
struct KP {
    std::uint32_t N, R;
    const std::uint32_t* row;
    const int2* ew;      // exact: {target, weight}
    const FEdge* fe;     // float
    const std::uint32_t* reg;
    std::uint32_t* succ_e;
    std::uint32_t* succ_v;
    int* succ_wi;
    double* succ_wf;
    long long* key_i;
    double* key_f;
    long long* lam_num;
    long long* lam_den;
    double* lam_f;
    int* active;
    int* changed;
    unsigned long long* slot;
    std::uint32_t* src;
    std::uint32_t* iters;
    unsigned long long* pj[2];
    std::uint32_t* comp;
    std::uint32_t* mark;
    std::uint32_t* cyc_len;
    long long* cyc_wi;
    double* cyc_wf;
    std::uint32_t* conn;
    std::uint32_t* rem[2];
    std::uint32_t* nxt[2];
    long long* acc[2];
    Flags* flags;
    std::uint32_t max_region;
    long long max_abs_w;
};

__device__ __forceinline__ bool working(const KP& p, std::uint32_t v) {
    return p.active[p.reg[v]] != 0;
}

// ------------------------------------------------------------ init

__global__ void k_init(KP p) {
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t v = tid; v < p.N; v += stride) {
        p.succ_e[v] = NONE;
        p.succ_v[v] = NONE;
        if (p.key_i)
            p.key_i[v] = 0;
        if (p.key_f)
            p.key_f[v] = 0.0;
        p.mark[v] = 0;
    }
    for (std::size_t r = tid; r < p.R; r += stride) {
        p.lam_num[r] = 0;
        p.lam_den[r] = 1;
        p.lam_f[r] = 0.0;
        p.active[r] = 1;
        p.changed[r] = 0;
        p.slot[r] = EMPTY;
        p.src[r] = NONE;
        p.iters[r] = 0;
    }
}

// ------------------------------------------------------------ improvement
//
// howard_par.hpp:146 spf_pass_iter / howard.hpp:63 improve_policy. G lanes
// cooperate on one vertex: lane j streams edges row[v]+j, +G, ... (coalesced
// 8-byte {target, weight} records), gathers the target's key, and the group
// reduces the lexicographic minimum (candidate, edge id), which is exactly
// the sequential "first strictly smaller" scan. Lane 0 then applies the
// replacement rule against the incumbent edge.

template <int G>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (G == 32)
        return FULL;
    else
        return ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
}

template <bool EXACT, int G> __global__ void __launch_bounds__(256) k_improve(KP p) {
    const unsigned lane = threadIdx.x & (G - 1);
    const unsigned gm = group_mask<G>();
    const std::size_t gid = (blockIdx.x * std::size_t(blockDim.x) + threadIdx.x) / G;
    const std::size_t gstride = (std::size_t(gridDim.x) * blockDim.x) / G;
    std::uint32_t last_marked = NONE;
    for (std::size_t vv = gid; vv < p.N; vv += gstride) {
        const std::uint32_t v = static_cast<std::uint32_t>(vv);
        const std::uint32_t r = p.reg[v];
        if (!p.active[r])
            continue;
        const std::uint32_t b = p.row[v], e_end = p.row[v + 1];
        std::uint32_t be = NONE;
        if constexpr (EXACT) {
            const long long num = p.lam_num[r], den = p.lam_den[r];
            long long best = 0;
            for (std::uint32_t e = b + lane; e < e_end; e += G) {
                const int2 ed = __ldg(&p.ew[e]);
                const long long c = p.key_i[ed.x] + static_cast<long long>(ed.y) * den - num;
                if (be == NONE || c < best) {
                    best = c;
                    be = e;
                }
            }
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) {
                const long long ob = __shfl_xor_sync(gm, best, off, G);
                const std::uint32_t oe = __shfl_xor_sync(gm, be, off, G);
                if (oe != NONE && (be == NONE || ob < best || (ob == best && oe < be))) {
                    best = ob;
                    be = oe;
                }
            }
            if (lane == 0) {
                if (be == NONE) {
                    p.flags->error = 1;
                } else {
                    const std::uint32_t cur = p.succ_e[v];
                    bool rep = cur == NONE;
                    if (!rep) {
                        const long long cc =
                            p.key_i[p.succ_v[v]] + static_cast<long long>(p.succ_wi[v]) * den - num;
                        rep = best < cc;
                    }
                    if (rep) {
                        const int2 ed = p.ew[be];
                        p.succ_e[v] = be;
                        p.succ_v[v] = static_cast<std::uint32_t>(ed.x);
                        p.succ_wi[v] = ed.y;
                        if (r != last_marked) {
                            last_marked = r;
                            if (*(volatile int*)&p.changed[r] == 0)
                                p.changed[r] = 1;
                        }
                    }
                }
            }
        } else {
            const double lam = p.lam_f[r];
            double best = 0.0;
            for (std::uint32_t e = b + lane; e < e_end; e += G) {
                const FEdge ed = p.fe[e];
                const double c = (p.key_f[ed.t] + ed.w) - lam;
                if (be == NONE || c < best) {
                    best = c;
                    be = e;
                }
            }
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) {
                const double ob = __shfl_xor_sync(gm, best, off, G);
                const std::uint32_t oe = __shfl_xor_sync(gm, be, off, G);
                if (oe != NONE && (be == NONE || ob < best || (ob == best && oe < be))) {
                    best = ob;
                    be = oe;
                }
            }
            if (lane == 0) {
                if (be == NONE) {
                    p.flags->error = 1;
                } else {
                    const std::uint32_t cur = p.succ_e[v];
                    bool rep = cur == NONE;
                    if (!rep) {
                        // FloatMode::strictly_better (policy.hpp:116)
                        const double cc = (p.key_f[p.succ_v[v]] + p.succ_wf[v]) - lam;
                        const double tol = 1e-9 * fmax(1.0, fmax(fabs(best), fabs(cc)));
                        rep = best < cc - tol;
                    }
                    if (rep) {
                        const FEdge ed = p.fe[be];
                        p.succ_e[v] = be;
                        p.succ_v[v] = ed.t;
                        p.succ_wf[v] = ed.w;
                        if (r != last_marked) {
                            last_marked = r;
                            if (*(volatile int*)&p.changed[r] == 0)
                                p.changed[r] = 1;
                        }
                    }
                }
            }
        }
    }
}

// Regions whose pass changed nothing are finished (howard_par.hpp:189).
__global__ void k_region_check(KP p) {
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t r = tid; r < p.R; r += stride) {
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
// Pointer doubling on the functional policy graph. pj[v] packs
// (jump target << 32 | least vertex on the jumped segment). After K rounds
// with 2^K >= region size, jump(v) lies on v's cycle and the least vertex of
// jump(v)'s segment is the least vertex of that cycle: the anchor of v's
// component (howard_par.hpp:310 cycle_anchor, minIndex). Every cycle vertex
// is the image of some vertex under succ^(2^K), so scattering a stamp to
// jump(v) marks exactly the cycle vertices (the survivors of the reference's
// elimination fixpoint, howard_par.hpp:249).

__global__ void k_pj_init(KP p) {
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t v = tid; v < p.N; v += stride)
        if (working(p, v))
            p.pj[0][v] = (static_cast<unsigned long long>(p.succ_v[v]) << 32) | v;
}

__global__ void k_pj_round(KP p, int in) {
    const unsigned long long* __restrict__ a = p.pj[in];
    unsigned long long* __restrict__ o = p.pj[in ^ 1];
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t v = tid; v < p.N; v += stride) {
        if (!working(p, v))
            continue;
        const unsigned long long x = a[v];
        const unsigned long long y = a[x >> 32];
        const unsigned long long lo = min(x & 0xffffffffull, y & 0xffffffffull);
        o[v] = (y & 0xffffffff00000000ull) | lo;
    }
}

__global__ void k_cycle_mark(KP p, int in, std::uint32_t stamp) {
    const unsigned long long* a = p.pj[in];
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t v = tid; v < p.N; v += stride) {
        if (!working(p, v))
            continue;
        const std::uint32_t j = static_cast<std::uint32_t>(a[v] >> 32);
        p.comp[v] = static_cast<std::uint32_t>(a[j] & 0xffffffffull);
        p.mark[j] = stamp;
        p.cyc_len[v] = 0;
        if (p.cyc_wi)
            p.cyc_wi[v] = 0;
    }
}

// Segmented reduction of (length, weight) per cycle, keyed by anchor.
// Exact integers, so the atomic order is irrelevant to the result. When a
// warp's cycle vertices share one anchor (the common single-giant-cycle
// case) the warp pre-reduces and issues one atomic pair.
__global__ void k_cycle_stats(KP p, std::uint32_t stamp) {
    const unsigned lane = threadIdx.x & 31;
    const std::size_t wid = (blockIdx.x * std::size_t(blockDim.x) + threadIdx.x) >> 5;
    const std::size_t wstride = (std::size_t(gridDim.x) * blockDim.x) >> 5;
    for (std::size_t base = wid * 32; base < p.N; base += wstride * 32) {
        const std::size_t v = base + lane;
        const bool on = v < p.N && working(p, v) && p.mark[v] == stamp;
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
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t v = tid; v < p.N; v += stride) {
        if (!working(p, v) || p.comp[v] != v)
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
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t vv = tid; vv < p.N; vv += stride) {
        const std::uint32_t v = static_cast<std::uint32_t>(vv);
        if (!working(p, v) || p.comp[v] != v)
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
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t r = tid; r < p.R; r += stride) {
        if (!p.active[r])
            continue;
        const unsigned long long a = p.slot[r];
        p.slot[r] = EMPTY;
        if (a == EMPTY) {
            p.flags->error = 1;
            continue;
        }
        p.src[r] = static_cast<std::uint32_t>(a);
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

// Warp-aggregated append to a compacted vertex list.
__device__ __forceinline__ void warp_append(bool take, std::uint32_t v, std::uint32_t* list,
                                            unsigned* counter) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned bal = __ballot_sync(FULL, take);
    if (!bal)
        return;
    unsigned base = 0;
    const int lead = __ffs(bal) - 1;
    if (static_cast<int>(lane) == lead)
        base = atomicAdd(counter, static_cast<unsigned>(__popc(bal)));
    base = __shfl_sync(FULL, base, lead);
    if (take)
        list[base + __popc(bal & ((1u << lane) - 1u))] = v;
}

// Kept component: vertices whose policy path ends in the winning cycle keep
// their edges (howard_par.hpp:393 markMinComponent); everyone else is queued
// for re-attachment.
__global__ void k_keep(KP p) {
    const unsigned lane = threadIdx.x & 31;
    const std::size_t wid = (blockIdx.x * std::size_t(blockDim.x) + threadIdx.x) >> 5;
    const std::size_t wstride = (std::size_t(gridDim.x) * blockDim.x) >> 5;
    for (std::size_t base = wid * 32; base < p.N; base += wstride * 32) {
        const std::size_t v = base + lane;
        bool take = false;
        if (v < p.N && working(p, v)) {
            const bool kept = p.comp[v] == p.src[p.reg[v]];
            p.conn[v] = kept ? 0u : NONE;
            take = !kept;
        }
        warp_append(take, static_cast<std::uint32_t>(v), p.rem[0], &p.flags->rem_count[0]);
    }
}

// One breadth layer of howard_par.hpp:433 connectGpi: a pending vertex
// attaches through its smallest out-edge whose head was connected in an
// earlier layer (conn < layer); connection stamps make the layer discipline
// exact regardless of schedule.
template <bool EXACT> __global__ void k_attach(KP p, int in, unsigned n_in, std::uint32_t layer) {
    const unsigned lane = threadIdx.x & 31;
    const std::size_t wid = (blockIdx.x * std::size_t(blockDim.x) + threadIdx.x) >> 5;
    const std::size_t wstride = (std::size_t(gridDim.x) * blockDim.x) >> 5;
    const std::uint32_t* list = p.rem[in];
    for (std::size_t base = wid * 32; base < n_in; base += wstride * 32) {
        const std::size_t i = base + lane;
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
                    if constexpr (EXACT)
                        p.succ_wi[x] = p.ew[e].y;
                    else
                        p.succ_wf[x] = p.fe[e].w;
                    p.conn[x] = layer;
                    pending = false;
                    break;
                }
            }
        }
        warp_append(pending, x, p.rem[in ^ 1], &p.flags->rem_count[in ^ 1]);
    }
}

// ------------------------------------------------------------ values
//
// Exact mode: value determination (howard_par.hpp:494 valuePropagate) as a
// tree prefix sum by pointer jumping. The policy is now a tree into the
// winning cycle; cutting it at the anchor (nxt = self, acc = 0) makes every
// key the sum of w*den - num along the policy path to the anchor, which is
// exactly value(u) = value(succ) + w - lambda scaled by den. Integer sums,
// so the association order is irrelevant. Rounds are gated on device: round
// j runs only if round j-1 still saw an unfinished vertex.

__global__ void k_prop_init(KP p) {
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t v = tid; v < p.N; v += stride) {
        if (!working(p, v))
            continue;
        const std::uint32_t r = p.reg[v];
        if (v == p.src[r]) {
            p.nxt[0][v] = static_cast<std::uint32_t>(v);
            p.acc[0][v] = 0;
        } else {
            p.nxt[0][v] = p.succ_v[v];
            p.acc[0][v] = static_cast<long long>(p.succ_wi[v]) * p.lam_den[r] - p.lam_num[r];
        }
    }
}

__global__ void k_prop_round(KP p, int round) {
    if (round > 0 && *(volatile unsigned*)&p.flags->notdone[round - 1] == 0)
        return;
    const int in = round & 1;
    const std::uint32_t* __restrict__ ni = p.nxt[in];
    const long long* __restrict__ ai = p.acc[in];
    std::uint32_t* __restrict__ no = p.nxt[in ^ 1];
    long long* __restrict__ ao = p.acc[in ^ 1];
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    bool flagged = false;
    for (std::size_t v = tid; v < p.N; v += stride) {
        if (!working(p, v))
            continue;
        const std::uint32_t x = ni[v];
        const std::uint32_t y = ni[x];
        ao[v] = ai[v] + ai[x];
        no[v] = y;
        if (!flagged && y != p.src[p.reg[v]]) {
            flagged = true;
            p.flags->notdone[round] = 1;
        }
    }
}

__global__ void k_prop_final(KP p, int rounds) {
    int last = rounds - 1;
    for (int j = 0; j < rounds; ++j)
        if (p.flags->notdone[j] == 0) {
            last = j;
            break;
        }
    const long long* a = p.acc[(last & 1) ^ 1];
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    if (tid == 0 && p.flags->notdone[rounds - 1] != 0)
        p.flags->error = 1; // did not converge within the round budget
    for (std::size_t v = tid; v < p.N; v += stride)
        if (working(p, v))
            p.key_i[v] = a[v];
}

// Float mode: level-synchronous propagation from the anchor, one policy
// level per launch, each vertex computing (value(succ) + w) - lambda exactly
// as the reference does, so values are bit-identical.
__global__ void k_fprop_init(KP p) {
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t v = tid; v < p.N; v += stride) {
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
    const std::size_t tid = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x;
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    bool flagged = false;
    for (std::size_t v = tid; v < p.N; v += stride) {
        if (!working(p, v) || p.conn[v] != NONE)
            continue;
        const std::uint32_t s = p.succ_v[v];
        if (p.conn[s] < level) {
            p.key_f[v] = (p.key_f[s] + p.succ_wf[v]) - p.lam_f[p.reg[v]];
            p.conn[v] = level;
        } else if (!flagged) {
            flagged = true;
            p.flags->notdone[slot] = 1;
        }
    }
}

int grid_for(std::size_t work, int sms, int per_sm = 8) {
    const std::size_t blocks = (work + 255) / 256;
    return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(blocks, std::size_t(sms) * per_sm)));
}

int ceil_log2(std::uint64_t x) {
    int k = 0;
    while ((1ull << k) < x)
        ++k;
    return k;
}

} // namespace

// ================================================================ state

struct DeviceState {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    DBuf<std::uint32_t> row, reg, succ_e, succ_v, comp, mark, cyc_len, conn, rem0, rem1, nxt0, nxt1,
        src, iters;
    DBuf<int2> ew;
    DBuf<FEdge> fe;
    DBuf<int> succ_wi, active, changed;
    DBuf<double> succ_wf, key_f, lam_f, cyc_wf;
    DBuf<long long> key_i, lam_num, lam_den, cyc_wi, acc0, acc1;
    DBuf<unsigned long long> slot, pj0, pj1;
    DBuf<Flags> flags;
    Flags* h_flags = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;
    KP kp{};

    ~DeviceState() {
        for (cudaEvent_t e : ev)
            cudaEventDestroy(e);
        if (ev_start)
            cudaEventDestroy(ev_start);
        if (ev_end)
            cudaEventDestroy(ev_end);
        if (h_flags)
            cudaFreeHost(h_flags);
        if (stream)
            cudaStreamDestroy(stream);
    }
    cudaEvent_t event(std::size_t i) {
        while (ev.size() <= i) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ev.push_back(e);
        }
        return ev[i];
    }
};

// ================================================================ host prep

Prepared prepare(const Graph& g0, const ocm_solve_options& opt) {
    Prepared pr;
    pr.n_orig = g0.n;
    pr.scc_off = opt.scc == OCM_SCC_OFF;
    const double sign = opt.objective == OCM_MAXIMIZE ? -1.0 : 1.0;
    Graph aug;
    const Graph* gp = &g0;
    if (pr.scc_off && g0.n > 0) {
        // Augment the (sign-adjusted) graph: the reference negates before
        // augmenting (solve.cpp:200-214), so big_w derives from |w| alike.
        if (sign < 0) {
            Graph neg = g0;
            for (double& w : neg.fwd_weight)
                w = -w;
            aug = augment_hamiltonian(neg, 0.0, &pr.no_cycle_above);
            for (double& w : aug.fwd_weight)
                w = -w; // undone below by sign
        } else {
            aug = augment_hamiltonian(g0, 0.0, &pr.no_cycle_above);
        }
        gp = &aug;
    }
    const Graph& g = *gp;
    pr.exact = g.integer_exact;
    const std::uint32_t n = g.n;
    std::vector<std::uint32_t> region_of;
    std::vector<char> nontrivial;
    std::uint32_t count = 0;
    if (pr.scc_off) {
        region_of.assign(n, 0);
        count = n ? 1 : 0;
        nontrivial.assign(count, 1);
    } else {
        count = tarjan_regions(g, region_of);
        std::vector<std::uint32_t> size(count, 0);
        for (std::uint32_t v = 0; v < n; ++v)
            ++size[region_of[v]];
        nontrivial.assign(count, 0);
        for (std::uint32_t v = 0; v < n; ++v) {
            const std::uint32_t r = region_of[v];
            if (size[r] > 1 || has_self_loop(g, v))
                nontrivial[r] = 1;
        }
    }
    pr.regions_total = count;
    // dense ids for non-trivial regions, in region id order
    std::vector<std::uint32_t> rid(count, NONE);
    for (std::uint32_t r = 0; r < count; ++r) {
        if (nontrivial[r])
            rid[r] = pr.R++;
        else
            ++pr.trivial;
    }
    std::vector<std::uint64_t> roff(static_cast<std::size_t>(pr.R) + 1, 0);
    for (std::uint32_t v = 0; v < n; ++v)
        if (rid[region_of[v]] != NONE)
            ++roff[rid[region_of[v]] + 1];
    for (std::uint32_t r = 0; r < pr.R; ++r) {
        pr.max_region = std::max<std::uint32_t>(pr.max_region, static_cast<std::uint32_t>(roff[r + 1]));
        roff[r + 1] += roff[r];
    }
    pr.N = static_cast<std::uint32_t>(roff[pr.R]);
    pr.orig.resize(pr.N);
    pr.reg.resize(pr.N);
    std::vector<std::uint32_t> local(n, NONE);
    {
        std::vector<std::uint64_t> fill(roff.begin(), roff.end() - 1);
        for (std::uint32_t v = 0; v < n; ++v) {
            const std::uint32_t r = rid[region_of[v]];
            if (r == NONE)
                continue;
            const std::uint64_t i = fill[r]++;
            pr.orig[i] = v;
            pr.reg[i] = r;
            local[v] = static_cast<std::uint32_t>(i);
        }
    }
    pr.row.assign(static_cast<std::size_t>(pr.N) + 1, 0);
    std::uint64_t M = 0;
    for (std::uint32_t i = 0; i < pr.N; ++i) {
        const std::uint32_t v = pr.orig[i];
        for (std::uint64_t e = g.fwd_index[v]; e < g.fwd_index[v + 1]; ++e)
            if (region_of[g.fwd_target[e]] == region_of[v])
                ++M;
        if (M >= 0xffffffffull)
            throw UnsupportedError("more than 2^32-1 intra-region edges");
        pr.row[i + 1] = static_cast<std::uint32_t>(M);
    }
    pr.M = M;
    pr.tgt.resize(M);
    pr.w.resize(M);
    double max_abs = 0.0;
    std::uint64_t k = 0;
    for (std::uint32_t i = 0; i < pr.N; ++i) {
        const std::uint32_t v = pr.orig[i];
        for (std::uint64_t e = g.fwd_index[v]; e < g.fwd_index[v + 1]; ++e) {
            const std::uint32_t t = g.fwd_target[e];
            if (region_of[t] != region_of[v])
                continue;
            pr.tgt[k] = local[t];
            const double w = sign * g.fwd_weight[e];
            pr.w[k] = w;
            max_abs = std::max(max_abs, std::fabs(w));
            ++k;
        }
    }
    if (pr.exact) {
        if (max_abs >= 2147483647.0)
            throw UnsupportedError("integer weights beyond 32 bits are not supported by the "
                                   "device lane");
        pr.max_abs_w = static_cast<std::int64_t>(max_abs);
    }
    return pr;
}

// ================================================================ session

Session::Session(const Graph& g, const ocm_solve_options& opt) : opt_(opt) {
    if (opt.algo != OCM_ALGO_HOWARD && opt.algo != OCM_ALGO_HOWARD_PAR)
        throw UnsupportedError("only the policy-iteration lanes (howard, howard-par) run on the "
                               "device");
    const auto t0 = std::chrono::steady_clock::now();
    prep_ = prepare(g, opt);
    d_ = std::make_unique<DeviceState>();
    DeviceState& d = *d_;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw CudaError("no CUDA device available (the solver has no CPU fallback)");
    d.device = opt.device;
    CK(cudaSetDevice(d.device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, d.device));
    if (prop.major < 10)
        throw CudaError(std::string("device ") + prop.name + " is not sm_100-class");
    d.sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&d.ev_start));
    CK(cudaEventCreate(&d.ev_end));
    CK(cudaMallocHost(&d.h_flags, sizeof(Flags)));

    const std::size_t N = prep_.N, R = prep_.R, M = prep_.M;
    const std::size_t N1 = std::max<std::size_t>(N, 1), R1 = std::max<std::size_t>(R, 1);
    d.row.alloc(N + 1);
    d.reg.alloc(N1);
    if (prep_.exact) {
        std::vector<int2> packed(M);
        for (std::size_t e = 0; e < M; ++e)
            packed[e] = make_int2(static_cast<int>(prep_.tgt[e]), static_cast<int>(prep_.w[e]));
        d.ew.alloc(std::max<std::size_t>(M, 1));
        CK(cudaMemcpyAsync(d.ew.p, packed.data(), M * sizeof(int2), cudaMemcpyHostToDevice, d.stream));
        h2d_bytes_ += M * sizeof(int2);
        CK(cudaStreamSynchronize(d.stream));
        d.succ_wi.alloc(N1);
        d.key_i.alloc(N1);
        d.cyc_wi.alloc(N1);
        d.acc0.alloc(N1);
        d.acc1.alloc(N1);
    } else {
        std::vector<FEdge> packed(M);
        for (std::size_t e = 0; e < M; ++e)
            packed[e] = FEdge{prep_.w[e], prep_.tgt[e], 0u};
        d.fe.alloc(std::max<std::size_t>(M, 1));
        CK(cudaMemcpyAsync(d.fe.p, packed.data(), M * sizeof(FEdge), cudaMemcpyHostToDevice, d.stream));
        h2d_bytes_ += M * sizeof(FEdge);
        CK(cudaStreamSynchronize(d.stream));
        d.succ_wf.alloc(N1);
        d.key_f.alloc(N1);
        d.cyc_wf.alloc(N1);
    }
    CK(cudaMemcpyAsync(d.row.p, prep_.row.data(), (N + 1) * sizeof(std::uint32_t),
                       cudaMemcpyHostToDevice, d.stream));
    h2d_bytes_ += (2 * N + 1) * sizeof(std::uint32_t);
    if (N)
        CK(cudaMemcpyAsync(d.reg.p, prep_.reg.data(), N * sizeof(std::uint32_t),
                           cudaMemcpyHostToDevice, d.stream));
    for (auto* b : {&d.succ_e, &d.succ_v, &d.comp, &d.mark, &d.cyc_len, &d.conn, &d.rem0, &d.rem1,
                    &d.nxt0, &d.nxt1})
        b->alloc(N1);
    d.pj0.alloc(N1);
    d.pj1.alloc(N1);
    d.src.alloc(R1);
    d.iters.alloc(R1);
    d.active.alloc(R1);
    d.changed.alloc(R1);
    d.lam_f.alloc(R1);
    d.lam_num.alloc(R1);
    d.lam_den.alloc(R1);
    d.slot.alloc(R1);
    d.flags.alloc(1);
    CK(cudaStreamSynchronize(d.stream));

    KP& p = d.kp;
    p.N = prep_.N;
    p.R = prep_.R;
    p.row = d.row.p;
    p.ew = d.ew.p;
    p.fe = d.fe.p;
    p.reg = d.reg.p;
    p.succ_e = d.succ_e.p;
    p.succ_v = d.succ_v.p;
    p.succ_wi = d.succ_wi.p;
    p.succ_wf = d.succ_wf.p;
    p.key_i = d.key_i.p;
    p.key_f = d.key_f.p;
    p.lam_num = d.lam_num.p;
    p.lam_den = d.lam_den.p;
    p.lam_f = d.lam_f.p;
    p.active = d.active.p;
    p.changed = d.changed.p;
    p.slot = d.slot.p;
    p.src = d.src.p;
    p.iters = d.iters.p;
    p.pj[0] = d.pj0.p;
    p.pj[1] = d.pj1.p;
    p.comp = d.comp.p;
    p.mark = d.mark.p;
    p.cyc_len = d.cyc_len.p;
    p.cyc_wi = d.cyc_wi.p;
    p.cyc_wf = d.cyc_wf.p;
    p.conn = d.conn.p;
    p.rem[0] = d.rem0.p;
    p.rem[1] = d.rem1.p;
    p.nxt[0] = d.nxt0.p;
    p.nxt[1] = d.nxt1.p;
    p.acc[0] = d.acc0.p;
    p.acc[1] = d.acc1.p;
    p.flags = d.flags.p;
    p.max_region = prep_.max_region;
    p.max_abs_w = prep_.max_abs_w;
    prep_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

Session::~Session() = default;

void* Session::stream() const { return d_ ? d_->stream : nullptr; }

namespace {

template <bool EXACT> void launch_improve(const KP& p, int sms, cudaStream_t s, double avg_deg) {
    int G = 1;
    while (G < 32 && G * 1.5 < avg_deg)
        G *= 2;
    const std::size_t threads = std::size_t(p.N) * G;
    const int grid = grid_for(threads, sms, 8);
    switch (G) {
    case 1: k_improve<EXACT, 1><<<grid, 256, 0, s>>>(p); break;
    case 2: k_improve<EXACT, 2><<<grid, 256, 0, s>>>(p); break;
    case 4: k_improve<EXACT, 4><<<grid, 256, 0, s>>>(p); break;
    case 8: k_improve<EXACT, 8><<<grid, 256, 0, s>>>(p); break;
    case 16: k_improve<EXACT, 16><<<grid, 256, 0, s>>>(p); break;
    default: k_improve<EXACT, 32><<<grid, 256, 0, s>>>(p); break;
    }
}

} // namespace

template <class M> void Session::run(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap) {
    constexpr bool EXACT = M::value;
    DeviceState& d = *d_;
    KP& p = d.kp;
    cudaStream_t s = d.stream;
    const int gv = grid_for(p.N, d.sms);
    const int gr = grid_for(std::max<std::uint32_t>(p.R, 1), d.sms);
    const double avg_deg = p.N ? double(prep_.M) / p.N : 1.0;
    std::uint64_t launches = 0, fix_iters = 0;
    std::uint32_t passes = 0, outer = 0;
    Flags& hf = *d.h_flags;

    std::uint64_t d2h = 0;
    auto read_flags = [&] {
        d2h += sizeof(Flags);
        CK(cudaMemcpyAsync(&hf, p.flags, sizeof(Flags), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hf.error)
            throw std::logic_error("howard_par: structural error (a vertex has no successor "
                                   "inside its region, or a region is not strongly connected)");
        if (hf.lambda_up)
            throw std::logic_error("vote_and_adopt: lambda increased");
        if (hf.overflow)
            throw RangeError("exact value keys would exceed 62 bits for this graph");
    };

    CK(cudaEventRecord(d.ev_start, s));
    CK(cudaMemsetAsync(p.flags, 0, sizeof(Flags), s));
    if (p.N) {
        k_init<<<gv, 256, 0, s>>>(p);
        ++launches;
    }
    const int K = std::max(1, ceil_log2(std::max<std::uint32_t>(prep_.max_region, 2)));
    const int prop_rounds = std::min(kMaxRounds, K + 1);
    while (p.N) {
        CK(cudaMemsetAsync(&p.flags->active_count, 0, sizeof(unsigned), s));
        CK(cudaEventRecord(d.event(2 * passes), s));
        launch_improve<EXACT>(p, d.sms, s, avg_deg);
        CK(cudaEventRecord(d.event(2 * passes + 1), s));
        ++passes;
        k_region_check<<<gr, 256, 0, s>>>(p);
        launches += 2;
        read_flags();
        if (hf.active_count == 0)
            break;
        ++outer;
        const std::uint32_t stamp = outer;

        // cycles of the policy graph
        k_pj_init<<<gv, 256, 0, s>>>(p);
        ++launches;
        int in = 0;
        for (int k = 0; k < K; ++k, in ^= 1) {
            k_pj_round<<<gv, 256, 0, s>>>(p, in);
            ++launches;
        }
        fix_iters += K;
        k_cycle_mark<<<gv, 256, 0, s>>>(p, in, stamp);
        if constexpr (EXACT)
            k_cycle_stats<<<gv, 256, 0, s>>>(p, stamp);
        else
            k_cycle_walk_float<<<gv, 256, 0, s>>>(p);
        k_vote<EXACT><<<gv, 256, 0, s>>>(p);
        k_adopt<EXACT><<<gr, 256, 0, s>>>(p);
        CK(cudaMemsetAsync(&p.flags->rem_count[0], 0, sizeof(unsigned), s));
        k_keep<<<gv, 256, 0, s>>>(p);
        launches += 5;
        read_flags();

        // breadth-layered re-attachment
        unsigned pending = hf.rem_count[0];
        int cur = 0;
        for (std::uint32_t layer = 1; pending > 0; ++layer) {
            CK(cudaMemsetAsync(&p.flags->rem_count[cur ^ 1], 0, sizeof(unsigned), s));
            k_attach<EXACT><<<grid_for(pending, d.sms), 256, 0, s>>>(p, cur, pending, layer);
            ++launches;
            ++fix_iters;
            read_flags();
            const unsigned next = hf.rem_count[cur ^ 1];
            if (next == pending)
                throw std::logic_error("connect_gpi_fixpoint: region is not strongly connected");
            pending = next;
            cur ^= 1;
        }

        // value determination
        if constexpr (EXACT) {
            CK(cudaMemsetAsync(p.flags->notdone, 0, sizeof(hf.notdone), s));
            k_prop_init<<<gv, 256, 0, s>>>(p);
            for (int j = 0; j < prop_rounds; ++j)
                k_prop_round<<<gv, 256, 0, s>>>(p, j);
            k_prop_final<<<gv, 256, 0, s>>>(p, prop_rounds);
            launches += 2 + prop_rounds;
            fix_iters += prop_rounds;
        } else {
            k_fprop_init<<<gv, 256, 0, s>>>(p);
            ++launches;
            for (std::uint32_t level = 1;; ++level) {
                CK(cudaMemsetAsync(&p.flags->notdone[0], 0, sizeof(unsigned), s));
                k_fprop_round<<<gv, 256, 0, s>>>(p, level, 0);
                ++launches;
                ++fix_iters;
                read_flags();
                if (hf.notdone[0] == 0)
                    break;
                if (level > prep_.max_region + 1)
                    throw std::logic_error("value propagation did not converge");
            }
        }
    }
    CK(cudaEventRecord(d.ev_end, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    read_flags();

    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, d.ev_start, d.ev_end));
    double imp = 0.0;
    for (std::uint32_t i = 0; i < passes; ++i) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, d.event(2 * i), d.event(2 * i + 1)));
        imp += t;
    }

    std::memset(out, 0, sizeof *out);
    out->mu_den = 1;
    out->outer_iters = outer;
    out->spf_passes = passes;
    out->regions = prep_.regions_total;
    out->trivial_regions = prep_.trivial;
    out->n_solved = prep_.N;
    out->m_solved = prep_.M;
    out->launches = launches;
    out->fixpoint_iters = fix_iters;
    out->device_ms = ms;
    out->improve_ms = imp;
    out->host_prep_ms = prep_ms_;
    out->h2d_bytes = h2d_bytes_;
    out->d2h_bytes = d2h;
    if (prep_.R == 0)
        return;

    const std::size_t R = prep_.R;
    std::vector<long long> ln(R), ld(R);
    std::vector<double> lf(R);
    std::vector<std::uint32_t> src(R), its(R);
    CK(cudaMemcpy(src.data(), p.src, R * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(its.data(), p.iters, R * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ln.data(), p.lam_num, R * sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ld.data(), p.lam_den, R * sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lf.data(), p.lam_f, R * sizeof(double), cudaMemcpyDeviceToHost));
    out->d2h_bytes += R * (3 * sizeof(long long) + 2 * sizeof(std::uint32_t));
    // least (mean, original anchor) over regions (solve.cpp:73 / howard_par.hpp:592)
    std::size_t best = R;
    auto less = [&](std::size_t a, std::size_t b) {
        if (EXACT) {
            const __int128 l = static_cast<__int128>(ln[a]) * ld[b];
            const __int128 r = static_cast<__int128>(ln[b]) * ld[a];
            if (l != r)
                return l < r;
        } else {
            if (lf[a] != lf[b])
                return lf[a] < lf[b];
        }
        return prep_.orig[src[a]] < prep_.orig[src[b]];
    };
    for (std::size_t r = 0; r < R; ++r) {
        if (its[r] == 0 || src[r] == NONE)
            throw std::logic_error("howard_par: first improvement pass made no change");
        if (best == R || less(r, best))
            best = r;
    }
    long long num = ln[best], den = ld[best];
    double mu = EXACT ? double(num) / double(den) : lf[best];
    if (prep_.scc_off) {
        const bool acyclic = EXACT ? static_cast<__int128>(static_cast<long long>(prep_.no_cycle_above)) * den <
                                         static_cast<__int128>(num)
                                   : prep_.no_cycle_above < mu;
        if (acyclic)
            return;
    }
    out->has_cycle = 1;
    out->exact = EXACT;
    if (opt_.objective == OCM_MAXIMIZE) {
        num = -num;
        mu = -mu;
    }
    if (EXACT) {
        out->mu_num = num;
        out->mu_den = den;
    }
    out->mu = mu;
    std::vector<std::uint32_t> succ(prep_.N);
    CK(cudaMemcpy(succ.data(), p.succ_v, prep_.N * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    out->d2h_bytes += prep_.N * sizeof(std::uint32_t);
    std::uint32_t u = src[best], len = 0;
    do {
        if (cycle_buf && len < cap)
            cycle_buf[len] = prep_.orig[u];
        ++len;
        u = succ[u];
    } while (u != src[best] && len <= prep_.N);
    out->cycle_len = len;
}

struct ExactTag {
    static constexpr bool value = true;
};
struct FloatTag {
    static constexpr bool value = false;
};

void Session::solve(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap) {
    CK(cudaSetDevice(d_->device));
    if (prep_.exact)
        run<ExactTag>(out, cycle_buf, cap);
    else
        run<FloatTag>(out, cycle_buf, cap);
    solved_ = true;
}

void Session::values(std::int64_t* key_num, std::int64_t* lam_num, std::int64_t* lam_den,
                     double* fval, std::uint32_t* succ_vertex) {
    if (!solved_)
        throw std::logic_error("session has not been solved yet");
    DeviceState& d = *d_;
    const std::size_t N = prep_.N, R = prep_.R, n = prep_.n_orig;
    std::vector<long long> key(N), ln(R), ld(R);
    std::vector<double> kf(N);
    std::vector<std::uint32_t> sv(N);
    if (N) {
        if (prep_.exact)
            CK(cudaMemcpy(key.data(), d.kp.key_i, N * sizeof(long long), cudaMemcpyDeviceToHost));
        else
            CK(cudaMemcpy(kf.data(), d.kp.key_f, N * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sv.data(), d.kp.succ_v, N * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    }
    if (R) {
        CK(cudaMemcpy(ln.data(), d.kp.lam_num, R * sizeof(long long), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ld.data(), d.kp.lam_den, R * sizeof(long long), cudaMemcpyDeviceToHost));
    }
    for (std::size_t v = 0; v < n; ++v) {
        if (key_num) key_num[v] = 0;
        if (lam_num) lam_num[v] = 0;
        if (lam_den) lam_den[v] = 1;
        if (fval) fval[v] = 0.0;
        if (succ_vertex) succ_vertex[v] = NONE;
    }
    for (std::size_t i = 0; i < N; ++i) {
        const std::uint32_t v = prep_.orig[i];
        if (key_num) key_num[v] = prep_.exact ? key[i] : 0;
        if (lam_num) lam_num[v] = ln[prep_.reg[i]];
        if (lam_den) lam_den[v] = ld[prep_.reg[i]];
        if (fval) fval[v] = prep_.exact ? 0.0 : kf[i];
        if (succ_vertex) succ_vertex[v] = prep_.orig[sv[i]];
    }
}

} // namespace ocmb
