// Host orchestration of the B200 policy-iteration lane: region split and
// upload (prepare / Session), the per-iteration launch sequence (run), and
// result read-back. The kernels live in kernels.cuh.

#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "errors.hpp"
#include "solve_kernel.cuh"
#include "gen.hpp"
#include "solver.hpp"

namespace ocmb {

void device_prepare(const HostCsr& g, const ocm_solve_options& opt, DeviceState& d, PrepInfo& info);
void device_generate_prepare(const GenSpec& spec, const ocm_solve_options& opt, DeviceState& d,
                             PrepInfo& info);

// ================================================================ session

namespace {

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// Per-device facts looked up once per process (device properties and the
// cooperative occupancy of k_solve cost milliseconds per query).
constexpr int kGs[4] = {1, 2, 4, 8};

// k_solve instantiation for (mode: 0 float, 1 exact, 2 wide exact; group
// width index 0..3)
// row 3: the exact lane with three doubling steps per pass (small graphs)
const void* solve_fn(int mode, int gi) {
    static const void* fns[4][4] = {
        {reinterpret_cast<const void*>(&k_solve<0, 1>), reinterpret_cast<const void*>(&k_solve<0, 2>),
         reinterpret_cast<const void*>(&k_solve<0, 4>), reinterpret_cast<const void*>(&k_solve<0, 8>)},
        {reinterpret_cast<const void*>(&k_solve<1, 1>), reinterpret_cast<const void*>(&k_solve<1, 2>),
         reinterpret_cast<const void*>(&k_solve<1, 4>), reinterpret_cast<const void*>(&k_solve<1, 8>)},
        {reinterpret_cast<const void*>(&k_solve<2, 1>), reinterpret_cast<const void*>(&k_solve<2, 2>),
         reinterpret_cast<const void*>(&k_solve<2, 4>), reinterpret_cast<const void*>(&k_solve<2, 8>)},
        {reinterpret_cast<const void*>(&k_solve<1, 1, 3>), reinterpret_cast<const void*>(&k_solve<1, 2, 3>),
         reinterpret_cast<const void*>(&k_solve<1, 4, 3>), reinterpret_cast<const void*>(&k_solve<1, 8, 3>)}};
    return fns[mode][gi];
}

struct DeviceFacts {
    int sms = 0, major = 0;
    int per_sm[4][4] = {}; // cooperative CTAs per SM of solve_fn(row, G)
    std::string name;
};

const DeviceFacts& device_facts(int dev) {
    static std::mutex mu;
    static std::map<int, DeviceFacts> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(dev);
    if (it != cache.end())
        return it->second;
    DeviceFacts f;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    f.sms = prop.multiProcessorCount;
    f.major = prop.major;
    f.name = prop.name;
    if (f.major >= 10) {
        for (int e = 0; e < 4; ++e)
            for (int gi = 0; gi < 4; ++gi) {
                int per_sm = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_fn(e, gi), kBlock, 0));
                f.per_sm[e][gi] = std::max(1, std::min(per_sm, kSolveMinBlocks));
            }
    }
    return cache.emplace(dev, f).first->second;
}

} // namespace

cudaMemPool_t session_pool() {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto it = pools.find(dev);
    if (it != pools.end())
        return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    CK(cudaMemPoolCreate(&pool, &props));
    std::uint64_t keep = ~0ull;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    return pools.emplace(dev, pool).first->second;
}


Session::Session(const Graph& g, const ocm_solve_options& opt, std::uint32_t rank, std::uint32_t world)
    : Session(csr_view(g), opt, rank, world) {}

Session::Session(const HostCsr& g, const ocm_solve_options& opt, std::uint32_t rank,
                 std::uint32_t world)
    : opt_(opt), rank_(rank), world_(world) {
    init([&](DeviceState& d) { device_prepare(g, opt, d, prep_); });
}

Session::Session(const GenSpec& spec, const ocm_solve_options& opt, std::uint32_t rank,
                 std::uint32_t world)
    : opt_(opt), rank_(rank), world_(world) {
    init([&](DeviceState& d) { device_generate_prepare(spec, opt, d, prep_); });
}

void Session::init(const std::function<void(DeviceState&)>& prepare) {
    const ocm_solve_options& opt = opt_;
    if (world_ == 0 || rank_ >= world_)
        throw std::invalid_argument("shard rank must be below the world size");
    if (opt.algo != OCM_ALGO_HOWARD && opt.algo != OCM_ALGO_HOWARD_PAR)
        throw UnsupportedError("only the policy-iteration lanes (howard, howard-par) run on the "
                               "device");
    const auto t0 = std::chrono::steady_clock::now();
    d_ = std::make_unique<DeviceState>();
    DeviceState& d = *d_;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw CudaError("no CUDA device available (the solver has no CPU fallback)");
    d.device = opt.device;
    if (d.device < 0 || d.device >= ndev)
        throw std::invalid_argument("device ordinal out of range");
    CK(cudaSetDevice(d.device));
    const DeviceFacts& facts = device_facts(d.device);
    if (facts.major < 10)
        throw CudaError("device " + facts.name + " is not sm_100-class");
    d.sms = facts.sms;
    CK(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&d.ev_start));
    CK(cudaEventCreate(&d.ev_end));
    d.h_ctl = new Ctl{}; // 300 B read back per launch: pageable is fine
    const auto t_prep = std::chrono::steady_clock::now();
    prepare(d);
    const auto t_alloc = std::chrono::steady_clock::now();

    const std::size_t N = prep_.n, R1 = std::size_t(prep_.R) + 1;
    const std::size_t N1 = std::max<std::size_t>(N, 1);
    // policy arrays are padded to world equal chunks for the all-gather
    chunk_ = static_cast<std::uint32_t>((N + world_ - 1) / world_);
    const std::size_t NP = std::max<std::size_t>(N1, std::size_t(chunk_) * world_);
    // exchange buffers of a sharded session can be mapped by peer processes
    const bool shared = world_ > 1;
    auto xalloc = [&](auto& buf, std::size_t k) {
        if (shared)
            buf.alloc_shared(k);
        else
            buf.alloc(k, d.stream);
    };
    if (prep_.exact) {
        xalloc(d.succ_wi, NP);
        d.key_i.alloc(N1, d.stream);
        d.cyc_wi.alloc(N1, d.stream);
        d.pv0.alloc(N1, d.stream);
        d.pv1.alloc(N1, d.stream);
        if (!prep_.wide && world_ == 1) {
            // packed {head, weight} shadow of the policy for the leaf split's
            // random reads (kept in step by every policy write of the fast
            // exact lane; the sharded lanes exchange the plain arrays)
            d.succ_vw.alloc(N1, d.stream);
        }
        if (prep_.wide) {
            if (world_ > 1)
                throw UnsupportedError("the sharded lanes run the 64-bit exact lane only (weights "
                                       "below 2^31)");
            alloc_wide();
        }
    } else {
        xalloc(d.succ_wf, NP);
        d.key_f.alloc(N1, d.stream);
        d.cyc_wf.alloc(N1, d.stream);
    }
    xalloc(d.succ_e, NP);
    xalloc(d.succ_v, NP);
    xalloc(d.xbar, 1);
    for (auto* b : {&d.comp, &d.wlist, &d.cyc_len, &d.conn, &d.rem0, &d.rem1,
                    &d.indeg, &d.plist, &d.clist, &d.cmark, &d.cmark2})
        b->alloc(N1, d.stream);
    d.cbits.alloc((N1 + 31) / 32, d.stream);
    d.pj0.alloc(N1, d.stream);
    d.pj1.alloc(N1, d.stream);
    d.src.alloc(R1, d.stream);
    d.iters.alloc(R1, d.stream);
    d.active.alloc(R1, d.stream);
    xalloc(d.changed0, R1);
    xalloc(d.changed1, R1);
    d.lam_f.alloc(R1, d.stream);
    d.lam_num.alloc(R1, d.stream);
    d.lam_den.alloc(R1, d.stream);
    d.slot.alloc(R1, d.stream);
    d.ctl.alloc(1, d.stream);
    // verification stamps start at 1: the stamp arrays and the control block
    // start from zero once per session
    CK(cudaMemsetAsync(d.cmark.p, 0, N1 * sizeof(std::uint32_t), d.stream));
    CK(cudaMemsetAsync(d.cmark2.p, 0, N1 * sizeof(std::uint32_t), d.stream));
    CK(cudaMemsetAsync(d.ctl.p, 0, sizeof(Ctl), d.stream));
    CK(cudaMemsetAsync(d.xbar.p, 0, sizeof(unsigned), d.stream));
    {
        Ctl init{};
        init.k_hint = 4;
        CK(cudaMemcpyAsync(d.ctl.p, &init, sizeof(Ctl), cudaMemcpyHostToDevice, d.stream));
    }
    CK(cudaStreamSynchronize(d.stream));

    // G lanes per improvement vertex (U = 4 edges in flight per lane): one
    // lane up to degree 8 (measured best at 8), then G*8 ~ average degree;
    // vertices of degree >= 32*G*4 go to the block-cooperative path.
    // OCM_IMPROVE_G / OCM_HEAVY_DEG override.
    {
        const double avg_deg =
            prep_.R ? double(prep_.M) / std::max<double>(1.0, double(prep_.n - prep_.trivial)) : 1.0;
        int G = 1;
        while (G < 8 && G * 8 < avg_deg)
            G *= 2;
        G = env_int("OCM_IMPROVE_G", G);
        gi_ = G >= 8 ? 3 : G >= 4 ? 2 : G >= 2 ? 1 : 0;
        G = kGs[gi_];
        d.kp.G = G;
        d.kp.U = 4;
        d.kp.heavy_deg = static_cast<std::uint32_t>(env_int("OCM_HEAVY_DEG", 32 * 4 * G));
        DBuf<unsigned> cnt;
        cnt.alloc(1, d.stream);
        CK(cudaMemsetAsync(cnt.p, 0, 4, d.stream));
        const std::uint32_t cap = static_cast<std::uint32_t>(
            std::min<std::uint64_t>(N, prep_.M / std::max<std::uint32_t>(d.kp.heavy_deg, 1) + 1));
        d.heavy.alloc(std::max<std::uint32_t>(cap, 1), d.stream);
        if (N)
            k_list_heavy<<<grid_for(N, d.sms), kBlock, 0, d.stream>>>(
                static_cast<std::uint32_t>(N), d.row.p, d.kp.heavy_deg, d.heavy.p, cnt.p);
        unsigned nh = 0;
        CK(cudaMemcpyAsync(&nh, cnt.p, 4, cudaMemcpyDeviceToHost, d.stream));
        CK(cudaStreamSynchronize(d.stream));
        d.kp.nheavy = nh;
        d.kp.heavy = d.heavy.p;
    }
    choose_hubs();

    // one CTA per SM slot the register budget allows (<= kSolveMinBlocks);
    // small graphs take one CTA per kBlock vertices: fewer arrivals make every
    // grid barrier cheaper and there is no work for more threads anyway
    mode_ = prep_.exact ? (prep_.wide ? 2 : 1) : 0;
    // two 16-byte doubling records per vertex: 3 steps per pass while they
    // stay within ~64 MB of L2, 2 beyond (exact lane)
    d.kp.round_s = std::max(2, std::min(3, env_int("OCM_ROUND_S", N <= (std::size_t(1) << 21) ? 3 : 2)));
    grid_ = facts.per_sm[krow()][gi_] * d.sms;
    // TMA-staged improvement for key arrays beyond the ~64 MB that random
    // gathers keep at L2 speed (OCM_STAGED=0/1 forces it off/on)
    {
        const int st = env_int("OCM_STAGED", -1);
        d.kp.staged = mode_ == 1 && d.kp.nhot == 0 && st != 0 &&
                      (st == 1 || std::size_t(prep_.n) * 8 > (std::size_t(64) << 20));
    }
    if (dyn_smem_bytes()) { // the staged pass / hub table use dynamic shared memory
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_fn(krow(), gi_), kBlock,
                                                         dyn_smem_bytes()));
        grid_ = std::min(grid_, std::max(1, per_sm) * d.sms);
    }
    if (const int env_grid = env_int("OCM_GRID", 0))
        grid_ = std::max(1, std::min(grid_, env_grid));
    else
        grid_ = static_cast<int>(std::max<std::size_t>(
            1, std::min<std::size_t>(grid_, (N + kBlock - 1) / kBlock)));

    KP& p = d.kp;
    p.N = prep_.n;
    p.R = prep_.R;
    p.row = d.row.p;
    p.ew = d.ew.p;
    p.fe = d.fe.p;
    p.reg = d.reg.p;
    p.succ_e = d.succ_e.p;
    p.succ_v = d.succ_v.p;
    p.succ_wi = d.succ_wi.p;
    p.succ_wf = d.succ_wf.p;
    p.succ_vw = d.succ_vw.p;
    d.tr_num.alloc(kTraceCap, d.stream);
    d.tr_den.alloc(kTraceCap, d.stream);
    d.tr_f.alloc(kTraceCap, d.stream);
    p.tr_num = d.tr_num.p;
    p.tr_den = d.tr_den.p;
    p.tr_f = d.tr_f.p;
    p.tr_cap = kTraceCap;
    if (const int ti = env_int("OCM_TRACE_ITERS", 0); ti > 0 && world_ == 1) {
        // debug: keep the policy and values of the first ti iterations
        const std::size_t cells = std::size_t(ti) * std::max<std::size_t>(N, 1);
        d.tr_pol.alloc(cells, d.stream);
        if (prep_.exact)
            d.tr_key.alloc(cells, d.stream);
        else
            d.tr_keyf.alloc(cells, d.stream);
        p.tr_pol = d.tr_pol.p;
        p.tr_key = d.tr_key.p;
        p.tr_keyf = d.tr_keyf.p;
        p.tr_iters = static_cast<unsigned>(ti);
    }
    p.key_i = d.key_i.p;
    p.key_f = d.key_f.p;
    p.lam_num = d.lam_num.p;
    p.lam_den = d.lam_den.p;
    p.lam_f = d.lam_f.p;
    p.active = d.active.p;
    p.changed[0] = d.changed0.p;
    p.changed[1] = d.changed1.p;
    p.slot = d.slot.p;
    p.src = d.src.p;
    p.iters = d.iters.p;
    p.pj[0] = d.pj0.p;
    p.pj[1] = d.pj1.p;
    p.comp = d.comp.p;
    p.indeg = d.indeg.p;
    p.plist = d.plist.p;
    p.clist = d.clist.p;
    p.cmark = d.cmark.p;
    p.cmark2 = d.cmark2.p;
    p.wlist = d.wlist.p;
    p.cyc_len = d.cyc_len.p;
    p.cyc_wi = d.cyc_wi.p;
    p.cyc_wf = d.cyc_wf.p;
    p.conn = d.conn.p;
    p.cbits = N >= static_cast<std::size_t>(env_int("OCM_CBITS_MIN_N", 1 << 24)) ? d.cbits.p : nullptr;
    p.rem[0] = d.rem0.p;
    p.rem[1] = d.rem1.p;
    p.pv[0] = d.pv0.p;
    p.pv[1] = d.pv1.p;
    p.c = d.ctl.p;
    p.max_region = prep_.max_region;
    p.max_abs_w = prep_.max_abs_w;
    p.own_lo = static_cast<std::uint32_t>(std::min<std::size_t>(N, std::size_t(rank_) * chunk_));
    p.own_hi = static_cast<std::uint32_t>(std::min<std::size_t>(N, std::size_t(rank_ + 1) * chunk_));
    p.indeg_in_improve = world_ == 1 ? 1 : 0;
    p.rank = static_cast<int>(rank_);
    p.world = static_cast<int>(world_);
    p.fused = 0;
    p.xbar = d.xbar.p;
    for (int q = 0; q < kMaxShards; ++q)
        p.peer_xbar[q] = nullptr;
    p.peer_xbar[rank_ < static_cast<std::uint32_t>(kMaxShards) ? rank_ : 0] = d.xbar.p;
    build_blocked_edges();
    h2d_bytes_ = prep_.h2d_bytes;
    const auto t_end = std::chrono::steady_clock::now();
    prep_ms_ = std::chrono::duration<double, std::milli>(t_end - t0).count();
    if (std::getenv("OCM_PREP_TIMING")) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "{\"init_setup_ms\": %.3f, \"prepare_ms\": %.3f, \"session_alloc_ms\": %.3f}\n",
                     ms(t0, t_prep), ms(t_prep, t_alloc), ms(t_alloc, t_end));
    }
}

// Bin-ordered copy of the intra-region edges for the propagation-blocked
// improvement pass (solve_kernel.cuh pb_pass1/pb_pass2), built once per
// session with OCM_PB=1 (exact lane, one rank). Opt-in: measured on B200 it
// gains 6% on BASELINE config 4 and loses 5% on config 5, the
// two passes streaming at only ~1.5 TB/s inside the persistent kernel.
// A stable radix sort of the edge ids by target bin keeps CSR order inside
// every bin; pb_off holds, per block of kPbVB vertices and bin, the first
// position whose source is in the block or later.
namespace {
__global__ void kb_keys(std::uint32_t m, const int2* ew, std::uint32_t bin, std::uint32_t* key,
                        std::uint32_t* id) {
    for (std::size_t e = gtid(); e < m; e += gstride()) {
        key[e] = static_cast<std::uint32_t>(ew[e].x) / bin;
        id[e] = static_cast<std::uint32_t>(e);
    }
}
__global__ void kb_bin_start(std::uint32_t m, const std::uint32_t* key, std::uint32_t nb, std::uint32_t* start) {
    for (std::size_t b = gtid(); b <= nb; b += gstride()) {
        std::uint32_t lo = 0, hi = m; // first position with key >= b
        while (lo < hi) {
            const std::uint32_t mid = lo + (hi - lo) / 2;
            if (key[mid] < b)
                lo = mid + 1;
            else
                hi = mid;
        }
        start[b] = lo;
    }
}
__global__ void kb_sources(std::uint32_t n, const std::uint32_t* row, std::uint32_t* src) {
    for (std::size_t v = gtid(); v < n; v += gstride())
        for (std::uint32_t e = row[v]; e < row[v + 1]; ++e)
            src[e] = static_cast<std::uint32_t>(v);
}
__global__ void kb_gather(std::uint32_t m, const std::uint32_t* perm, const int2* ew, const std::uint32_t* src_csr,
                          int2* tw, std::uint32_t* inv, std::uint32_t* src) {
    for (std::size_t i = gtid(); i < m; i += gstride()) {
        const std::uint32_t e = perm[i];
        tw[i] = ew[e];
        src[i] = src_csr[e];
        inv[e] = static_cast<std::uint32_t>(i);
    }
}
__global__ void kb_offsets(std::uint32_t n, std::uint32_t nblk, std::uint32_t nb, const std::uint32_t* row,
                           const std::uint32_t* perm, const std::uint32_t* start, std::uint32_t* off) {
    const std::size_t tot = std::size_t(nblk + 1) * nb;
    for (std::size_t i = gtid(); i < tot; i += gstride()) {
        const std::uint32_t blk = static_cast<std::uint32_t>(i / nb), b = static_cast<std::uint32_t>(i % nb);
        const std::uint32_t first = row[min(static_cast<std::size_t>(n), std::size_t(blk) * kPbVB)];
        std::uint32_t lo = start[b], hi = start[b + 1]; // first position with edge id >= first
        while (lo < hi) {
            const std::uint32_t mid = lo + (hi - lo) / 2;
            if (perm[mid] < first)
                lo = mid + 1;
            else
                hi = mid;
        }
        off[i] = lo;
    }
}
} // namespace

// Hub vertices for the staged key table (exact lane): the highest
// intra-region in-degrees. Opt-in: measured on B200 the table is slower than
// plain gathers even where 1024 hubs receive 25% of the edges (web-like
// graph, 6.4*10^7 vertices: 531 vs 492 ms of improvement per min solve,
// profiles/r02/hot_staging_r02.log) -- L2 serves the few hub sectors at full
// rate and the per-edge probe costs more than the gathers it saves.
// OCM_HOT=-1 chooses automatically (>= 2% of the edges into at most 1024
// vertices of >= 64x the average in-degree), OCM_HOT=1 forces it on for any
// graph with edges (tests), OCM_HOT_SLOTS sets the table size (power of two,
// 2 slots per hub).
void Session::choose_hubs() {
    DeviceState& d = *d_;
    KP& p = d.kp;
    p.nhot = 0;
    p.hot = nullptr;
    p.hot_shift = 32;
    hot_bytes_ = 0;
    const int mode = env_int("OCM_HOT", 0);
    const std::size_t N = prep_.n;
    if (mode == 0 || !prep_.exact || prep_.wide || prep_.M == 0 || N == 0 || d.kp.pb)
        return;
    unsigned slots = static_cast<unsigned>(env_int("OCM_HOT_SLOTS", 2048));
    slots = std::max(64u, std::min(slots, 8192u));
    while (slots & (slots - 1))
        slots &= slots - 1;
    const unsigned cap = slots / 2;
    cudaStream_t s = d.stream;
    DBuf<unsigned> cnt, ids, cnt_sorted, ids_sorted;
    cnt.alloc(N, s);
    ids.alloc(N, s);
    cnt_sorted.alloc(N, s);
    ids_sorted.alloc(N, s);
    CK(cudaMemsetAsync(cnt.p, 0, N * 4, s));
    k_edge_indeg<<<grid_for(prep_.M, d.sms, 16), kBlock, 0, s>>>(prep_.M, d.ew.p, cnt.p);
    k_iota<<<grid_for(N, d.sms), kBlock, 0, s>>>(static_cast<std::uint32_t>(N), ids.p);
    std::size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, cnt.p, cnt_sorted.p, ids.p,
                                                 ids_sorted.p, static_cast<int>(N), 0, 32, s));
    DBuf<unsigned char> tmp;
    tmp.alloc(std::max<std::size_t>(bytes, 1), s);
    CK(cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, cnt.p, cnt_sorted.p, ids.p,
                                                 ids_sorted.p, static_cast<int>(N), 0, 32, s));
    const unsigned take = static_cast<unsigned>(std::min<std::size_t>(cap, N));
    std::vector<unsigned> top(take);
    CK(cudaMemcpyAsync(top.data(), cnt_sorted.p, take * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double avg = double(prep_.M) / double(std::max<std::size_t>(1, N - prep_.trivial));
    unsigned n_hot = 0;
    std::uint64_t covered = 0;
    for (unsigned i = 0; i < take; ++i) {
        if (top[i] == 0 || (mode != 1 && double(top[i]) < 64.0 * avg))
            break;
        ++n_hot;
        covered += top[i];
    }
    hot_coverage_ = double(covered) / double(prep_.M);
    if (n_hot == 0 || (mode != 1 && hot_coverage_ < 0.02))
        return;
    d.hot.alloc(n_hot, s);
    CK(cudaMemcpyAsync(d.hot.p, ids_sorted.p, n_hot * 4ull, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    unsigned lg = 0;
    while ((1u << lg) < slots)
        ++lg;
    p.hot = d.hot.p;
    p.nhot = n_hot;
    p.hot_shift = 32 - lg;
    hot_bytes_ = std::size_t(slots) * 12;
}

namespace {
// sign extension of the 32-bit weights into the wide lane's high halves
__global__ void k_widen(std::uint64_t m, const int2* ew, int* ew_hi, std::uint32_t n,
                        const int* succ_wi, int* succ_whi) {
    for (std::uint64_t e = gtid(); e < m; e += gstride())
        ew_hi[e] = ew[e].y < 0 ? -1 : 0;
    for (std::uint64_t v = gtid(); v < n; v += gstride())
        succ_whi[v] = succ_wi[v] < 0 ? -1 : 0;
}
} // namespace

// Buffers of the wide exact lane (128-bit keys, winning-cycle records, the
// high halves of the policy weights; prep writes ew_hi for wide graphs).
void Session::alloc_wide() {
    DeviceState& d = *d_;
    const std::size_t N1 = std::max<std::size_t>(prep_.n, 1);
    d.key_w.alloc(N1, d.stream);
    d.pvw0.alloc(N1, d.stream);
    d.pvw1.alloc(N1, d.stream);
    d.succ_whi.alloc(N1, d.stream);
    d.kp.key_w = d.key_w.p;
    d.kp.pvw[0] = d.pvw0.p;
    d.kp.pvw[1] = d.pvw1.p;
    d.kp.succ_whi = d.succ_whi.p;
    d.kp.ew_hi = d.ew_hi.p;
}

// The fast lane's adoption check found that a key could leave +-2^62 (long
// cycles with large weights): switch the session to the wide lane for good.
// Its 32-bit weights widen by sign extension; everything else is re-run.
void Session::promote_wide() {
    DeviceState& d = *d_;
    if (world_ > 1)
        throw RangeError("exact value keys would exceed 62 bits for this graph (the sharded lanes "
                         "run 64-bit keys only)");
    if (!d.ew_hi.p) {
        d.ew_hi.alloc(std::max<std::uint64_t>(prep_.M, 1) + 2, d.stream);
        CK(cudaMemsetAsync(d.ew_hi.p, 0, (std::max<std::uint64_t>(prep_.M, 1) + 2) * 4, d.stream));
    }
    prep_.wide = true;
    alloc_wide();
    k_widen<<<grid_for(std::max<std::uint64_t>(prep_.M, prep_.n), d.sms, 8), kBlock, 0, d.stream>>>(
        prep_.M, d.ew.p, d.ew_hi.p, prep_.n, d.succ_wi.p, d.succ_whi.p);
    CK(cudaGetLastError());
    d.kp.staged = 0;
    d.kp.nhot = 0;
    d.kp.pb = 0;
    mode_ = 2;
    const DeviceFacts& facts = device_facts(d.device);
    const int before = grid_;
    grid_ = std::min(before, facts.per_sm[2][gi_] * d.sms);
    CK(cudaStreamSynchronize(d.stream));
}

int Session::krow() const { return mode_ == 1 && d_->kp.round_s == 3 ? 3 : mode_; }

std::size_t Session::dyn_smem_bytes() const {
    const KP& p = d_->kp;
    if (p.pb)
        return kPbSmem;
    if (p.staged)
        return kStagedSmem;
    return p.nhot ? hot_bytes_ : 0;
}

void Session::build_blocked_edges() {
    DeviceState& d = *d_;
    KP& p = d.kp;
    p.pb = 0;
    const std::uint64_t N = prep_.n, M = prep_.M;
    if (env_int("OCM_PB", 0) != 1 || !prep_.exact || prep_.wide || world_ != 1 || prep_.R == 0 ||
        M == 0)
        return;
    // bins of ~2M vertices (16 MB of keys); OCM_PB_BIN overrides (tests)
    std::uint64_t bin = std::max<std::uint64_t>(std::uint64_t(env_int("OCM_PB_BIN", 1 << 21)),
                                                (N + kMaxPbBins - 1) / kMaxPbBins);
    bin = std::max<std::uint64_t>(bin, 1);
    const std::uint32_t nb = static_cast<std::uint32_t>((N + bin - 1) / bin);
    const std::uint32_t nblk = static_cast<std::uint32_t>((N + kPbVB - 1) / kPbVB);
    const std::uint32_t m = static_cast<std::uint32_t>(M);
    cudaStream_t s = d.stream;
    const int g = grid_for(M, d.sms, 8);
    {
        DBuf<std::uint32_t> key_in, key_out, id_in, start;
        key_in.alloc(M, s);
        key_out.alloc(M, s);
        id_in.alloc(M, s);
        d.pb_perm.alloc(M, s);
        kb_keys<<<g, kBlock, 0, s>>>(m, d.ew.p, static_cast<std::uint32_t>(bin), key_in.p, id_in.p);
        const int end_bit = std::max(1, ceil_log2(std::uint64_t(nb) + 1));
        std::size_t bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key_in.p, key_out.p, id_in.p, d.pb_perm.p,
                                           static_cast<long long>(M), 0, end_bit, s));
        DBuf<unsigned char> tmp;
        tmp.alloc(std::max<std::size_t>(bytes, 1), s);
        CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key_in.p, key_out.p, id_in.p, d.pb_perm.p,
                                           static_cast<long long>(M), 0, end_bit, s));
        tmp.release();
        key_in.release();
        id_in.release();
        start.alloc(std::size_t(nb) + 1, s);
        kb_bin_start<<<grid_for(nb + 1, d.sms), kBlock, 0, s>>>(m, key_out.p, nb, start.p);
        key_out.release();
        d.pb_tw.alloc(M, s);
        d.pb_inv.alloc(M, s);
        d.pb_src.alloc(M, s);
        {
            DBuf<std::uint32_t> src_csr;
            src_csr.alloc(M, s);
            kb_sources<<<grid_for(N, d.sms, 8), kBlock, 0, s>>>(static_cast<std::uint32_t>(N), d.row.p, src_csr.p);
            kb_gather<<<g, kBlock, 0, s>>>(m, d.pb_perm.p, d.ew.p, src_csr.p, d.pb_tw.p, d.pb_inv.p, d.pb_src.p);
        }
        d.pb_off.alloc((std::size_t(nblk) + 1) * nb, s);
        kb_offsets<<<grid_for((std::size_t(nblk) + 1) * nb, d.sms, 8), kBlock, 0, s>>>(
            static_cast<std::uint32_t>(N), nblk, nb, d.row.p, d.pb_perm.p, start.p, d.pb_off.p);
        d.pb_cand.alloc(M, s);
        CK(cudaStreamSynchronize(s));
    }
    p.pb = 1;
    p.staged = 0; // the blocked pass replaces the staged one (and its shared memory)
    p.pb_tw = d.pb_tw.p;
    p.pb_perm = d.pb_perm.p;
    p.pb_inv = d.pb_inv.p;
    p.pb_src = d.pb_src.p;
    p.pb_off = d.pb_off.p;
    p.pb_cand = d.pb_cand.p;
    p.pb_m = M;
    p.pb_nb = nb;
    p.pb_nblk = nblk;
}

Session::~Session() = default;

void* Session::stream() const { return d_ ? d_->stream : nullptr; }

// One cooperative launch of k_solve in the given mode; returns its event time.
// One cooperative launch of k_solve in the given mode: enqueue, then (unless
// the caller overlaps it with peers' launches) wait and check the outcome.
template <class M> void Session::launch_async(int mode) {
    constexpr bool EXACT = M::value;
    DeviceState& d = *d_;
    KP& p = d.kp;
    cudaStream_t s = d.stream;
    p.small_wc = 4096;
    p.fused = mode == kShardFused ? 1 : 0;
    if (mode != kShardResume) {
        CK(cudaMemsetAsync(reinterpret_cast<char*>(p.c) + kCtlSolveOffset, 0,
                           sizeof(Ctl) - kCtlSolveOffset, s));
        d2h_ = 0;
        solve_ms_ = 0.0;
        launches_ = 0;
    } else {
        // a resumed launch keeps the solve's counters but counts its grid
        // barriers from zero
        CK(cudaMemsetAsync(&p.c->gbar, 0, sizeof(unsigned), s));
    }
    CK(cudaEventRecord(d.ev_start, s));
    if (prep_.R > 0) {
        void* args[] = {&p, &mode};
        CK(cudaLaunchCooperativeKernel(solve_fn(krow(), gi_), dim3(grid_), dim3(kBlock), args,
                                       dyn_smem_bytes(), s));
        ++launches_;
    }
    CK(cudaEventRecord(d.ev_end, s));
}

float Session::launch_wait() {
    DeviceState& d = *d_;
    Ctl& hc = *d.h_ctl;
    // (a copy into pageable memory blocks the host until the kernel is done:
    // issued here, not in launch_async, so peers' launches are not held up)
    CK(cudaMemcpyAsync(d.h_ctl, d.kp.c, sizeof(Ctl), cudaMemcpyDeviceToHost, d.stream));
    d2h_ += sizeof(Ctl);
    CK(cudaStreamSynchronize(d.stream));
    CK(cudaGetLastError());
    if (prep_.R == 0)
        hc.shard_done = 1;
    if (hc.xfail) {
        // the cross-rank barrier words are now out of step with the peers':
        // no later fused launch may run on this session
        fused_broken_ = true;
        throw std::runtime_error("fused sharded lane: a peer rank never reached the cross-rank "
                                 "barrier (are all ranks launched and connected?)");
    }
    if (hc.error)
        throw std::logic_error("howard_par: structural error (a vertex has no successor "
                               "inside its region, or a region is not strongly connected)");
    if (hc.lambda_up)
        throw std::logic_error("vote_and_adopt: lambda increased");
    if (hc.overflow)
        throw RangeError("exact value keys would exceed 62 bits for this graph");
    if (hc.nonconv)
        throw std::logic_error("a device fixpoint did not converge within its bound");
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, d.ev_start, d.ev_end));
    solve_ms_ += ms;
    return ms;
}

template <class M> float Session::launch(int mode) {
    launch_async<M>(mode);
    return launch_wait();
}

// Result of the solve that just finished: counters, the optimal region's
// lambda and its cycle (read back from the device).
template <class M> void Session::collect(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap) {
    constexpr bool EXACT = M::value;
    DeviceState& d = *d_;
    KP& p = d.kp;
    Ctl& hc = *d.h_ctl;
    const double ms = solve_ms_;
    std::uint64_t d2h = d2h_;
    static const bool phases_on = std::getenv("OCM_PHASES") != nullptr;
    if (phases_on && prep_.R > 0 && hc.clk_total > 0) {
        static const char* names[PH_COUNT] = {"init",  "improve", "classify", "round",
                                              "verify", "stats",  "vote",     "wincyc",
                                              "keep",  "leaves",  "attach",   "float"};
        std::string ph;
        for (int i = 0; i < PH_COUNT; ++i) {
            char buf[64];
            std::snprintf(buf, sizeof buf, "%s\"%s\": %.3f", i ? ", " : "", names[i],
                          ms * double(hc.clk[i]) / double(hc.clk_total));
            ph += buf;
        }
        std::fprintf(stderr,
                     "{\"device_ms\": %.3f, \"phases_ms\": {%s}, \"passes\": %u, \"outer\": %u, "
                     "\"rounds\": %u, \"verifies\": %u, \"peeled\": %llu, \"cored\": %llu, "
                     "\"layers\": %u, \"syncs\": %u, \"k_hint\": %u, \"launches\": %u, \"N\": %u, "
                     "\"M\": %llu, \"nhot\": %u, \"hot_coverage\": %.4f}\n",
                     ms, ph.c_str(), hc.passes, hc.outer, hc.rounds, hc.verifies,
                     (unsigned long long)hc.peeled, (unsigned long long)hc.cored, hc.layers, hc.syncs,
                     hc.k_hint, launches_, p.N, (unsigned long long)prep_.M, p.nhot, hot_coverage_);
    }

    std::memset(out, 0, sizeof *out);
    out->mu_den = 1;
    out->outer_iters = hc.outer;
    out->spf_passes = hc.passes;
    out->regions = prep_.regions_total;
    out->trivial_regions = prep_.trivial;
    out->n_solved = prep_.n;
    out->m_solved = prep_.M;
    out->launches = launches_;
    out->fixpoint_iters = std::uint64_t(hc.rounds) + hc.layers;
    out->device_ms = ms;
    // share of the launch spent in improvement phases (SM clock spans of
    // block 0, measured between the same grid barriers) times the event time
    out->improve_ms = hc.clk_total ? ms * double(hc.clk[PH_IMPROVE]) / double(hc.clk_total) : 0.0;
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
        return src[a] < src[b];
    };
    std::uint64_t outer_sum = 0;
    for (std::size_t r = 0; r < R; ++r) {
        if (its[r] == 0 || src[r] == NONE)
            throw std::logic_error("howard_par: first improvement pass made no change");
        outer_sum += its[r];
        if (best == R || less(r, best))
            best = r;
    }
    if (opt_.algo == OCM_ALGO_HOWARD) {
        // run_howard_seq (src/solve.cpp:71-72) sums every region's outer
        // iterations and improvement passes (a region's passes = its
        // adoptions + the final quiet pass); howard-par reports the maximum
        // over the concurrently iterating regions (hc.outer / hc.passes)
        out->outer_iters = static_cast<std::uint32_t>(outer_sum);
        out->spf_passes = static_cast<std::uint32_t>(outer_sum + R);
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
    // the optimal cycle, walked on the device from its anchor (its length is
    // the adopted record's); very long cycles fall back to the host walk
    const std::uint32_t start = src[best];
    std::uint32_t clen = 0;
    CK(cudaMemcpy(&clen, p.cyc_len + start, sizeof clen, cudaMemcpyDeviceToHost));
    out->d2h_bytes += sizeof clen;
    std::uint32_t len = 0;
    if (clen > 0 && clen <= (1u << 16)) {
        DBuf<std::uint32_t> cyc;
        cyc.alloc(clen, d.stream);
        k_cycle_out<<<1, 32, 0, d.stream>>>(p.succ_v, start, clen, cyc.p);
        std::vector<std::uint32_t> h(clen);
        CK(cudaMemcpyAsync(h.data(), cyc.p, clen * sizeof(std::uint32_t), cudaMemcpyDeviceToHost,
                           d.stream));
        CK(cudaStreamSynchronize(d.stream));
        out->d2h_bytes += clen * sizeof(std::uint32_t);
        for (; len < clen; ++len)
            if (cycle_buf && len < cap)
                cycle_buf[len] = h[len];
    } else {
        std::vector<std::uint32_t> succ(prep_.n);
        CK(cudaMemcpy(succ.data(), p.succ_v, prep_.n * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
        out->d2h_bytes += prep_.n * sizeof(std::uint32_t);
        std::uint32_t u = start;
        do {
            if (cycle_buf && len < cap)
                cycle_buf[len] = u;
            ++len;
            u = succ[u];
        } while (u != start && len <= prep_.n);
    }
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
    if (world_ > 1)
        throw std::invalid_argument("sharded session: drive it with shard_step / shard_finish");
    if (prep_.exact) {
        try {
            launch<ExactTag>(kSolveFull);
        } catch (const RangeError&) {
            // a key could leave the fast lane's +-2^62: redo the solve with
            // 128-bit keys (the same policy iteration, so the same result)
            if (mode_ != 1)
                throw;
            promote_wide();
            launch<ExactTag>(kSolveFull);
        }
        collect<ExactTag>(out, cycle_buf, cap);
    } else {
        launch<FloatTag>(kSolveFull);
        collect<FloatTag>(out, cycle_buf, cap);
    }
    solved_ = true;
}

bool Session::shard_step() {
    CK(cudaSetDevice(d_->device));
    const int mode = shard_started_ ? kShardResume : kShardBegin;
    if (prep_.exact)
        launch<ExactTag>(mode);
    else
        launch<FloatTag>(mode);
    shard_started_ = true;
    const bool done = d_->h_ctl->shard_done != 0;
    if (done)
        shard_started_ = false;
    return done;
}

void Session::shard_finish(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap) {
    CK(cudaSetDevice(d_->device));
    if (prep_.exact)
        collect<ExactTag>(out, cycle_buf, cap);
    else
        collect<FloatTag>(out, cycle_buf, cap);
    solved_ = true;
}

void Session::shard_peer_info(ocm_shard_peer* out) const {
    const DeviceState& d = *d_;
    std::memset(out, 0, sizeof *out);
    out->device = d.device;
    out->rank = rank_;
    const void* bufs[6] = {d.succ_e.p, d.succ_v.p,
                           prep_.exact ? static_cast<const void*>(d.succ_wi.p)
                                       : static_cast<const void*>(d.succ_wf.p),
                           d.changed0.p, d.changed1.p, d.xbar.p};
    for (int i = 0; i < 6; ++i) {
        out->ptr[i] = reinterpret_cast<std::uint64_t>(bufs[i]);
        if (world_ > 1) {
            cudaIpcMemHandle_t h;
            CK(cudaIpcGetMemHandle(&h, const_cast<void*>(bufs[i])));
            static_assert(sizeof h == sizeof out->ipc[0], "IPC handle size");
            std::memcpy(out->ipc[i], &h, sizeof h);
        }
    }
}

void Session::shard_connect(const ocm_shard_peer* peers, std::uint32_t world, bool ipc) {
    DeviceState& d = *d_;
    if (world != world_)
        throw std::invalid_argument("peer list does not match the session's world size");
    if (world_ > static_cast<std::uint32_t>(kMaxShards))
        throw std::invalid_argument("the fused sharded lane supports at most 8 ranks");
    CK(cudaSetDevice(d.device));
    KP& p = d.kp;
    for (std::uint32_t q = 0; q < world; ++q) {
        if (peers[q].rank != q)
            throw std::invalid_argument("peer list must be ordered by rank");
        void* b[6];
        for (int i = 0; i < 6; ++i) {
            if (q == rank_) {
                b[i] = reinterpret_cast<void*>(peers[q].ptr[i]);
            } else if (ipc) {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, peers[q].ipc[i], sizeof h);
                CK(cudaIpcOpenMemHandle(&b[i], h, cudaIpcMemLazyEnablePeerAccess));
                d.ipc_opened.push_back(b[i]);
            } else {
                b[i] = reinterpret_cast<void*>(peers[q].ptr[i]);
                if (peers[q].device != d.device) {
                    const cudaError_t e = cudaDeviceEnablePeerAccess(peers[q].device, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                        CK(e);
                    cudaGetLastError();
                }
            }
        }
        p.peer_succ_e[q] = static_cast<std::uint32_t*>(b[0]);
        p.peer_succ_v[q] = static_cast<std::uint32_t*>(b[1]);
        p.peer_succ_w[q] = b[2];
        p.peer_changed[0][q] = static_cast<int*>(b[3]);
        p.peer_changed[1][q] = static_cast<int*>(b[4]);
        p.peer_xbar[q] = static_cast<unsigned*>(b[5]);
    }
    connected_ = true;
}

void Session::fused_launch() {
    if (!connected_)
        throw std::logic_error("fused sharded lane: connect the peers first");
    if (fused_broken_)
        throw std::logic_error("fused sharded lane: a previous solve timed out at a cross-rank "
                               "barrier; the barrier epochs are out of step, recreate the "
                               "sessions");
    CK(cudaSetDevice(d_->device));
    if (prep_.exact)
        launch_async<ExactTag>(kShardFused);
    else
        launch_async<FloatTag>(kShardFused);
}

void Session::fused_finish(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap) {
    CK(cudaSetDevice(d_->device));
    launch_wait();
    if (prep_.exact)
        collect<ExactTag>(out, cycle_buf, cap);
    else
        collect<FloatTag>(out, cycle_buf, cap);
    solved_ = true;
}

void Session::shard_buffers(ocm_shard_buffers* b) const {
    const DeviceState& d = *d_;
    std::memset(b, 0, sizeof *b);
    b->rank = rank_;
    b->world = world_;
    b->chunk = chunk_;
    b->own_lo = d.kp.own_lo;
    b->own_hi = d.kp.own_hi;
    b->n = prep_.n;
    b->succ_e = d.succ_e.p;
    b->succ_v = d.succ_v.p;
    b->succ_w = prep_.exact ? static_cast<void*>(d.succ_wi.p) : static_cast<void*>(d.succ_wf.p);
    b->succ_w_bytes = prep_.exact ? 4 : 8;
    b->changed0 = d.changed0.p;
    b->changed1 = d.changed1.p;
    b->regions = prep_.R + 1;
    b->stream = d.stream;
}

namespace {
__device__ __forceinline__ void cert_add(unsigned long long* dst, unsigned long long v) {
    v = __reduce_add_sync(FULL, static_cast<unsigned>(v)); // per-thread counts stay < 2^32
    if ((threadIdx.x & 31) == 0 && v)
        atomicAdd(dst, v);
}

// Bellman optimality of the keys and the policy edge, one thread per vertex.
__global__ void k_certify_vertices(KP p, unsigned long long* cnt) {
    unsigned long long verts = 0, edges = 0, kv = 0, pv = 0;
    for (std::size_t v = gtid(); v < p.N; v += gstride()) {
        const std::uint32_t r = p.reg[v];
        const std::uint32_t b = p.row[v], e_end = p.row[v + 1];
        if (r >= p.R || b == e_end)
            continue;
        ++verts;
        // keys and weights of either exact lane (wide: 128-bit keys, the
        // weights' high halves in ew_hi / succ_whi)
        auto key = [&](std::uint32_t x) -> __int128 { return p.key_w ? p.key_w[x] : p.key_i[x]; };
        auto wgt = [&](std::uint32_t e, int2 ed) -> long long {
            return p.key_w ? (static_cast<long long>(p.ew_hi[e]) << 32) | static_cast<unsigned>(ed.y)
                           : ed.y;
        };
        const __int128 K = key(static_cast<std::uint32_t>(v));
        const long long num = p.lam_num[r], den = p.lam_den[r];
        for (std::uint32_t e = b; e < e_end; ++e) {
            const int2 ed = p.ew[e];
            const __int128 c = key(static_cast<std::uint32_t>(ed.x)) +
                               static_cast<__int128>(wgt(e, ed)) * den - num;
            kv += c < K;
            ++edges;
        }
        const std::uint32_t se = p.succ_e[v];
        if (se < b || se >= e_end) {
            ++pv;
        } else {
            const int2 ed = p.ew[se];
            const long long we = wgt(se, ed);
            const __int128 c = key(static_cast<std::uint32_t>(ed.x)) + static_cast<__int128>(we) * den - num;
            const long long ws = p.key_w ? (static_cast<long long>(p.succ_whi[v]) << 32) |
                                               static_cast<unsigned>(p.succ_wi[v])
                                         : p.succ_wi[v];
            pv += c != K || p.succ_v[v] != static_cast<std::uint32_t>(ed.x) || ws != we;
        }
    }
    cert_add(&cnt[0], verts);
    cert_add(&cnt[1], edges);
    cert_add(&cnt[3], kv);
    cert_add(&cnt[4], pv);
}

// Every region's anchor cycle, one thread per region (a dependent walk).
__global__ void k_certify_cycles(KP p, unsigned long long* cnt) {
    unsigned long long regs = 0, cv = 0;
    for (std::size_t r = gtid(); r < p.R; r += gstride()) {
        ++regs;
        const std::uint32_t a = p.src[r];
        if (a >= p.N) {
            ++cv;
            continue;
        }
        std::uint32_t u = a, mn = a;
        unsigned long long len = 0;
        long long sum = 0;
        do {
            sum += p.key_w ? (static_cast<long long>(p.succ_whi[u]) << 32) | static_cast<unsigned>(p.succ_wi[u])
                           : p.succ_wi[u];
            u = p.succ_v[u];
            mn = min(mn, u);
            ++len;
        } while (u != a && u < p.N && len <= p.N);
        cv += u != a || mn != a ||
              static_cast<__int128>(sum) * p.lam_den[r] != static_cast<__int128>(len) * p.lam_num[r];
    }
    cert_add(&cnt[2], regs);
    cert_add(&cnt[5], cv);
}
} // namespace

void Session::certify(ocm_certificate* out) {
    if (!solved_)
        throw std::logic_error("session has not been solved yet");
    if (!prep_.exact)
        throw UnsupportedError("the optimality certificate covers the exact (integer-weight) lane");
    DeviceState& d = *d_;
    std::memset(out, 0, sizeof *out);
    if (prep_.R == 0 || prep_.n == 0)
        return;
    DBuf<unsigned long long> cnt;
    cnt.alloc(6, d.stream);
    CK(cudaMemsetAsync(cnt.p, 0, 6 * sizeof(unsigned long long), d.stream));
    k_certify_vertices<<<grid_for(prep_.n, d.sms, 8), kBlock, 0, d.stream>>>(d.kp, cnt.p);
    k_certify_cycles<<<grid_for(prep_.R, d.sms, 1), kBlock, 0, d.stream>>>(d.kp, cnt.p);
    unsigned long long h[6];
    CK(cudaMemcpyAsync(h, cnt.p, sizeof h, cudaMemcpyDeviceToHost, d.stream));
    CK(cudaStreamSynchronize(d.stream));
    out->vertices = h[0];
    out->edges = h[1];
    out->regions = h[2];
    out->key_violations = h[3];
    out->policy_violations = h[4];
    out->cycle_violations = h[5];
}

void Session::values(std::int64_t* key_num, std::int64_t* lam_num, std::int64_t* lam_den,
                     double* fval, std::uint32_t* succ_vertex) {
    if (!solved_)
        throw std::logic_error("session has not been solved yet");
    DeviceState& d = *d_;
    const std::size_t n = prep_.n, R1 = std::size_t(prep_.R) + 1;
    std::vector<long long> key(n), ln(R1), ld(R1);
    std::vector<double> kf(n);
    std::vector<std::uint32_t> sv(n), reg(n);
    if (n) {
        if (prep_.exact && mode_ == 2) {
            std::vector<__int128> kw(n);
            CK(cudaMemcpy(kw.data(), d.kp.key_w, n * sizeof(__int128), cudaMemcpyDeviceToHost));
            for (std::size_t v = 0; v < n; ++v) {
                if (kw[v] != static_cast<__int128>(static_cast<long long>(kw[v])) && key_num)
                    throw RangeError("a value key exceeds 64 bits: read it with ocm_session_keys_wide");
                key[v] = static_cast<long long>(kw[v]);
            }
        } else if (prep_.exact)
            CK(cudaMemcpy(key.data(), d.kp.key_i, n * sizeof(long long), cudaMemcpyDeviceToHost));
        else
            CK(cudaMemcpy(kf.data(), d.kp.key_f, n * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sv.data(), d.kp.succ_v, n * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(reg.data(), d.kp.reg, n * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    }
    CK(cudaMemcpy(ln.data(), d.kp.lam_num, R1 * sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ld.data(), d.kp.lam_den, R1 * sizeof(long long), cudaMemcpyDeviceToHost));
    for (std::size_t v = 0; v < n; ++v) {
        const bool solved = reg[v] != prep_.R;
        if (key_num) key_num[v] = solved && prep_.exact ? key[v] : 0;
        if (lam_num) lam_num[v] = solved ? ln[reg[v]] : 0;
        if (lam_den) lam_den[v] = solved ? ld[reg[v]] : 1;
        if (fval) fval[v] = solved && !prep_.exact ? kf[v] : 0.0;
        if (succ_vertex) succ_vertex[v] = solved ? sv[v] : NONE;
    }
}

} // namespace ocmb

namespace ocmb {

// Exact value keys at full width: hi:lo = the 128-bit key (narrow lane:
// sign-extended 64-bit keys); vertices outside every region get 0.
void Session::keys_wide(std::int64_t* hi, std::uint64_t* lo) {
    if (!solved_)
        throw std::logic_error("session has not been solved yet");
    if (!prep_.exact)
        throw UnsupportedError("value keys exist in the exact lane only");
    DeviceState& d = *d_;
    const std::size_t n = prep_.n;
    std::vector<std::uint32_t> reg(n);
    std::vector<__int128> k(n);
    if (n) {
        CK(cudaMemcpy(reg.data(), d.kp.reg, n * 4, cudaMemcpyDeviceToHost));
        if (mode_ == 2) {
            CK(cudaMemcpy(k.data(), d.kp.key_w, n * sizeof(__int128), cudaMemcpyDeviceToHost));
        } else {
            std::vector<long long> k64(n);
            CK(cudaMemcpy(k64.data(), d.kp.key_i, n * 8, cudaMemcpyDeviceToHost));
            for (std::size_t v = 0; v < n; ++v)
                k[v] = k64[v];
        }
    }
    for (std::size_t v = 0; v < n; ++v) {
        const __int128 x = reg[v] != prep_.R ? k[v] : 0;
        hi[v] = static_cast<std::int64_t>(x >> 64);
        lo[v] = static_cast<std::uint64_t>(x);
    }
}

} // namespace ocmb

namespace ocmb {

// lambda of region 0 after each adoption of the last solve
void Session::lambda_trace(std::int64_t* num, std::int64_t* den, double* f, std::uint32_t cap,
                           std::uint32_t* len) {
    if (!solved_)
        throw std::logic_error("session has not been solved yet");
    DeviceState& d = *d_;
    std::uint32_t it = 0;
    if (prep_.R > 0)
        CK(cudaMemcpy(&it, d.kp.iters, 4, cudaMemcpyDeviceToHost));
    const std::uint32_t k = std::min({it, cap, kTraceCap});
    *len = it;
    if (k == 0)
        return;
    if (prep_.exact) {
        if (num)
            CK(cudaMemcpy(num, d.kp.tr_num, k * 8ull, cudaMemcpyDeviceToHost));
        if (den)
            CK(cudaMemcpy(den, d.kp.tr_den, k * 8ull, cudaMemcpyDeviceToHost));
    } else if (f) {
        CK(cudaMemcpy(f, d.kp.tr_f, k * 8ull, cudaMemcpyDeviceToHost));
    }
}

} // namespace ocmb

namespace ocmb {

// debug trace (OCM_TRACE_ITERS sessions): policy edge ids and value keys
// (exact, low 64 bits) or values (float) after iteration `it` of the last solve
void Session::iter_trace(std::uint32_t it, std::uint32_t* succ_e, std::int64_t* key, double* fval) {
    DeviceState& d = *d_;
    if (!d.kp.tr_pol)
        throw std::logic_error("session created without OCM_TRACE_ITERS");
    if (it >= d.kp.tr_iters)
        throw std::invalid_argument("iteration beyond the traced ones");
    const std::size_t n = prep_.n, base = std::size_t(it) * n;
    if (succ_e)
        CK(cudaMemcpy(succ_e, d.kp.tr_pol + base, n * 4, cudaMemcpyDeviceToHost));
    if (key && d.kp.tr_key)
        CK(cudaMemcpy(key, d.kp.tr_key + base, n * 8, cudaMemcpyDeviceToHost));
    if (fval && d.kp.tr_keyf)
        CK(cudaMemcpy(fval, d.kp.tr_keyf + base, n * 8, cudaMemcpyDeviceToHost));
}

} // namespace ocmb
