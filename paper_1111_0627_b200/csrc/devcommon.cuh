// Types and helpers shared by the device translation units (solver.cu,
// prep.cu). Kernels themselves stay TU-local.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "errors.hpp"
#include "prepinfo.hpp"

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            throw ::ocmb::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));          \
    } while (0)

namespace ocmb {

constexpr std::uint32_t NONE = 0xffffffffu;
constexpr unsigned long long EMPTY = ~0ull;
constexpr unsigned FULL = 0xffffffffu;
#ifndef OCM_BLOCK
#define OCM_BLOCK 256
#endif
constexpr int kBlock = OCM_BLOCK;
constexpr int kMaxShards = 8; // ranks of the fused sharded lane (one per GPU of a box)
constexpr int kMaxPbBins = 512; // target bins of the propagation-blocked improvement pass

struct __align__(16) FEdge {
    double w;
    std::uint32_t t;
    std::uint32_t pad;
};

// Pointer-jumping record for value determination: accumulated key along the
// jumped segment, the segment end, and the root (anchor) of the vertex.
struct __align__(16) PJV {
    long long acc;
    std::uint32_t nxt;
    std::uint32_t root;
};

// The same for the wide exact lane (128-bit accumulated keys).
struct __align__(16) PJVW {
    __int128 acc;
    std::uint32_t nxt;
    std::uint32_t root;
    std::uint64_t pad;
};

// Pointer-doubling record for cycle detection: segment end, least vertex on
// the segment, weight sum of the segment.
struct __align__(16) PJC {
    std::uint32_t nxt;
    std::uint32_t mn;
    long long w;
};

// Device-resident control block of the persistent solver kernel (k_solve).
// Nothing in it is reset between iterations: list appends and counts go
// through cumulative 64-bit counters used in ping-pong pairs (see Ring in
// solve_kernel.cuh), and one-shot flags carry the unique stamp of the check
// that raised them, so no phase has to clear state another block may still
// be reading.
enum Phase {
    PH_INIT, PH_IMPROVE, PH_CLASSIFY, PH_ROUND, PH_VERIFY, PH_STATS, PH_VOTE, PH_WINCYC, PH_KEEP,
    PH_LEAVES, PH_ATTACH, PH_FLOAT, PH_COUNT
};

struct Ctl {
    // ---- persistent across the session's solves (zeroed once at creation)
    unsigned long long ring[3][2]; // cumulative append counters (ring, slot)
    unsigned long long done;       // blocks through the vote phase (cumulative)
    unsigned long long wc_n[2];    // (stamp << 32) | winning-cycle vertices listed
    unsigned wc_len[2];            // longest winning cycle (slot stamp & 1)
    unsigned wc_big[2];            // = stamp when the grid must do the winning cycles
    unsigned stamp;                // last verification stamp used
    unsigned k_hint;               // doubling rounds that sufficed last iteration
    unsigned k_streak;             // consecutive first-try verifications
    unsigned xepoch;               // cross-rank barriers passed (fused sharded lane)
    unsigned vfail[2];             // = stamp of a failed verification (slot stamp & 1)
    // ---- per solve (host clears from here on before every launch)
    int error;     // structural (no successor / not strongly connected)
    int overflow;  // exact keys would leave +-2^62
    int lambda_up; // lambda increased inside a region
    int nonconv;   // a fixpoint did not converge within its bound
    int xfail;     // fused sharded lane: a peer never reached the barrier
    unsigned it;         // iteration index (sharded launches resume it)
    unsigned shard_done; // sharded lane: the last launch finished the solve
    unsigned passes;
    unsigned outer;
    unsigned rounds;               // pointer-doubling rounds (all iterations)
    unsigned verifies;             // cycle verifications
    unsigned long long peeled;     // leaves split off (all iterations)
    unsigned long long cored;      // vertices doubled (all iterations)
    unsigned layers;               // attach layers + float levels
    unsigned syncs;                // grid barriers
    long long clk_total;           // block-0 SM clock over the launch
    long long clk[PH_COUNT];       // ... per phase (time up to the phase's barrier)
    unsigned gbar;                 // grid-barrier arrivals (OCM_GBAR)
};
constexpr std::size_t kCtlSolveOffset = offsetof(Ctl, error);
// error, overflow, lambda_up, nonconv are read together after every
// classification barrier (one 16-byte load)
static_assert(offsetof(Ctl, error) % 16 == 0 && offsetof(Ctl, overflow) == offsetof(Ctl, error) + 4 &&
                  offsetof(Ctl, lambda_up) == offsetof(Ctl, error) + 8,
              "Ctl failure flags must form one aligned 16-byte group");

// Everything a kernel may touch, passed by value.
struct KP {
    std::uint32_t N, R;
    const std::uint32_t* row;
    const int2* ew;  // exact: {target, weight}
    const FEdge* fe; // float
    const std::uint32_t* reg;
    std::uint32_t* succ_e;
    std::uint32_t* succ_v;
    int* succ_wi;
    double* succ_wf;
    long long* key_i;
    double* key_f;
    __int128* key_w;           // wide exact lane: 128-bit keys
    const int* ew_hi;          // wide exact lane: high 32 bits of each edge weight
    int* succ_whi;             // wide exact lane: high 32 bits of the policy weight
    int2* succ_vw;             // fast exact lane, one rank: packed {head, weight} shadow of the policy
    // lambda of region 0 after each adoption (the reference's HowardTrace,
    // howard_par.hpp:588), up to tr_cap iterations
    long long* tr_num;
    long long* tr_den;
    double* tr_f;
    unsigned tr_cap;
    std::uint32_t* tr_pol; // debug: policy per iteration (tr_iters x N), or null
    long long* tr_key;     // debug: value keys per iteration (exact lanes, low 64 bits)
    double* tr_keyf;       // debug: values per iteration (float lane)
    unsigned tr_iters;
    long long* lam_num;
    long long* lam_den;
    double* lam_f;
    int* active;
    int* changed[2];
    unsigned long long* slot;
    std::uint32_t* src;
    std::uint32_t* iters;
    // cycle phase
    std::uint32_t* indeg; // policy in-degree (leaf split)
    std::uint32_t* plist; // leaves of the policy graph this iteration
    std::uint32_t* clist; // the other working vertices (the core)
    std::uint32_t* cmark; // verification stamps: image of succ^L
    std::uint32_t* cmark2;
    PJC* pj[2];           // doubling records (vertex-indexed)
    std::uint32_t* comp;  // anchor: least vertex of the reached cycle
    std::uint32_t* wlist; // cycle vertices (image of succ^L) this iteration
    std::uint32_t* cyc_len;
    long long* cyc_wi;
    double* cyc_wf;
    std::uint32_t* conn;
    std::uint32_t* cbits; // connected-vertex bitmap (attach's head test), N/8 bytes
    int round_s;          // doubling steps per pass (2 or 3; selects the k_solve instantiation)
    std::uint32_t* rem[2];
    PJV* pv[2];
    PJVW* pvw[2];
    Ctl* c;
    std::uint32_t max_region;
    long long max_abs_w;
    const std::uint32_t* heavy; // vertices of intra-region degree >= heavy_deg
    std::uint32_t nheavy;
    std::uint32_t heavy_deg;
    // hub vertices (highest intra-region in-degree) whose keys every CTA
    // stages in a shared-memory hash table at the start of each improvement
    // pass (exact lane); 0 = off
    const std::uint32_t* hot;
    std::uint32_t nhot;
    std::uint32_t hot_shift; // table slots = 2^(32 - hot_shift)
    int staged;              // TMA-staged improvement pass (exact lane, HBM-resident keys)
    std::uint32_t own_lo, own_hi; // improvement range (all vertices unless sharded)
    // fused sharded lane (kShardFused): the rank's peers' policy replicas and
    // flags (peer memory: NVLink-mapped IPC pointers between GPUs, plain
    // pointers between shards sharing a GPU) and the cross-rank barrier words
    int rank, world, fused;
    std::uint32_t* peer_succ_e[kMaxShards];
    std::uint32_t* peer_succ_v[kMaxShards];
    void* peer_succ_w[kMaxShards];
    int* peer_changed[2][kMaxShards];
    unsigned* peer_xbar[kMaxShards];
    unsigned* xbar;
    int indeg_in_improve;         // 1: the improvement pass counts policy in-degrees
    // propagation-blocked improvement pass (exact lane, HBM-resident keys)
    int pb;
    const int2* pb_tw;            // bin-ordered {target, weight}
    const std::uint32_t* pb_perm; // bin position -> edge id
    const std::uint32_t* pb_inv;  // edge id -> bin position
    const std::uint32_t* pb_src;  // bin position -> source vertex
    const std::uint32_t* pb_off;  // [blk * pb_nb + b]: first position of vertex block blk in bin b
    long long* pb_cand;           // candidate per bin position
    std::uint64_t pb_m;
    std::uint32_t pb_nb, pb_nblk;
    // tuning (launch arguments)
    int G;                 // improvement lanes per vertex
    int U;                 // edges in flight per lane (4)
    std::uint32_t small_wc; // winning cycles up to this many vertices: one block
};

// The library's own stream-ordered memory pool for the current device
// (created once, release threshold = keep everything cached, so re-creating
// sessions does not pay cudaMalloc/cudaFree synchronisation). A private pool:
// the default pool's threshold is left alone for everything else in the
// process. Defined in solver.cu.
cudaMemPool_t session_pool();

template <class T> struct DBuf {
    T* p = nullptr;
    std::size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    // Stream-ordered allocation from the library's private pool.
    cudaStream_t st = nullptr;
    bool plain = false; // cudaMalloc'ed (IPC-exportable), not pool memory
    void alloc(std::size_t k, cudaStream_t s = nullptr) {
        release();
        st = s;
        if (k)
            CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), k * sizeof(T),
                                       session_pool(), st));
        n = k;
    }
    // Memory other processes can map (cudaIpcGetMemHandle does not accept
    // stream-ordered pool allocations): the fused sharded lane's exchange
    // buffers.
    void alloc_shared(std::size_t k) {
        release();
        if (k)
            CK(cudaMalloc(reinterpret_cast<void**>(&p), k * sizeof(T)));
        plain = true;
        n = k;
    }
    void release() {
        if (p) {
            if (plain)
                cudaFree(p);
            else
                cudaFreeAsync(p, st);
        }
        p = nullptr;
        n = 0;
        plain = false;
    }
    ~DBuf() { release(); }
};

inline int grid_for(std::size_t work, int sms, int per_sm = 8) {
    const std::size_t blocks = (work + kBlock - 1) / kBlock;
    const std::size_t cap = std::size_t(sms) * per_sm;
    return static_cast<int>(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

inline int ceil_log2(std::uint64_t x) {
    int k = 0;
    while ((1ull << k) < x)
        ++k;
    return k;
}

// Device state of a session: the prepared graph plus solver scratch.
struct DeviceState {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    DBuf<std::uint32_t> row, reg, succ_e, succ_v, comp, wlist, cyc_len, conn, rem0, rem1, src,
        iters, indeg, plist, clist, cmark, cmark2, heavy, xbar, hot, cbits;
    DBuf<PJV> pv0, pv1;
    DBuf<PJVW> pvw0, pvw1;
    DBuf<__int128> key_w;
    DBuf<int> ew_hi, succ_whi;
    DBuf<int2> succ_vw;
    DBuf<long long> tr_num, tr_den;
    DBuf<double> tr_f;
    DBuf<std::uint32_t> tr_pol;
    DBuf<long long> tr_key;
    DBuf<double> tr_keyf;
    DBuf<PJC> pj0, pj1;
    DBuf<int2> ew;
    DBuf<FEdge> fe;
    DBuf<int> succ_wi, active, changed0, changed1;
    DBuf<double> succ_wf, key_f, lam_f, cyc_wf;
    DBuf<long long> key_i, lam_num, lam_den, cyc_wi;
    DBuf<unsigned long long> slot;
    DBuf<Ctl> ctl;
    DBuf<int2> pb_tw;
    DBuf<std::uint32_t> pb_perm, pb_inv, pb_off, pb_src;
    DBuf<long long> pb_cand;
    Ctl* h_ctl = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;
    cudaStream_t side = nullptr;      // weight upload overlapping the region split
    cudaEvent_t side_done = nullptr;
    cudaEvent_t alloc_done = nullptr; // orders side-stream use after allocations on `stream`
    std::vector<void*> ipc_opened;    // peer buffers mapped with cudaIpcOpenMemHandle
    KP kp{};
    cudaEvent_t ev_alloc_done(cudaStream_t s) {
        if (!alloc_done)
            CK(cudaEventCreateWithFlags(&alloc_done, cudaEventDisableTiming));
        CK(cudaEventRecord(alloc_done, s));
        return alloc_done;
    }

    ~DeviceState() {
        if (stream)
            cudaStreamSynchronize(stream);
        for (auto* b : {&row, &reg, &succ_e, &succ_v, &comp, &wlist, &cyc_len, &conn, &rem0, &rem1,
                        &src, &iters, &indeg, &plist, &clist, &cmark, &cmark2, &heavy, &xbar, &hot,
                        &cbits})
            b->release();
        pv0.release();
        pv1.release();
        pvw0.release();
        pvw1.release();
        key_w.release();
        ew_hi.release();
        succ_whi.release();
        succ_vw.release();
        tr_num.release();
        tr_den.release();
        tr_f.release();
        tr_pol.release();
        tr_key.release();
        tr_keyf.release();
        pj0.release();
        pj1.release();
        ew.release();
        fe.release();
        succ_wi.release();
        active.release();
        changed0.release();
        changed1.release();
        succ_wf.release();
        key_f.release();
        lam_f.release();
        cyc_wf.release();
        key_i.release();
        lam_num.release();
        lam_den.release();
        cyc_wi.release();
        slot.release();
        ctl.release();
        pb_tw.release();
        pb_perm.release();
        pb_inv.release();
        pb_off.release();
        pb_src.release();
        pb_cand.release();
        if (stream)
            cudaStreamSynchronize(stream);
        for (cudaEvent_t e : ev)
            cudaEventDestroy(e);
        for (void* q : ipc_opened)
            cudaIpcCloseMemHandle(q);
        if (side) {
            cudaStreamSynchronize(side);
            cudaStreamDestroy(side);
        }
        if (side_done)
            cudaEventDestroy(side_done);
        if (alloc_done)
            cudaEventDestroy(alloc_done);
        if (ev_start)
            cudaEventDestroy(ev_start);
        if (ev_end)
            cudaEventDestroy(ev_end);
        delete h_ctl;
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

} // namespace ocmb
