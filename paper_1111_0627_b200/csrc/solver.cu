// Host orchestration of the B200 policy-iteration lane: region split and
// upload (prepare / Session), the per-iteration launch sequence (run), and
// result read-back. The kernels live in kernels.cuh.

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "errors.hpp"
#include "kernels.cuh"
#include "solver.hpp"

namespace ocmb {

void device_prepare(const Graph& g, const ocm_solve_options& opt, DeviceState& d, PrepInfo& info);

// ================================================================ session

Session::Session(const Graph& g, const ocm_solve_options& opt) : opt_(opt) {
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
    CK(cudaSetDevice(d.device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, d.device));
    if (prop.major < 10)
        throw CudaError(std::string("device ") + prop.name + " is not sm_100-class");
    d.sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    {
        // keep freed blocks cached in the default pool across sessions
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, d.device));
        std::uint64_t keep = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    CK(cudaEventCreate(&d.ev_start));
    CK(cudaEventCreate(&d.ev_end));
    CK(cudaMallocHost(&d.h_flags, sizeof(Flags)));

    device_prepare(g, opt, d, prep_);

    const std::size_t N = prep_.n, R1 = std::size_t(prep_.R) + 1;
    const std::size_t N1 = std::max<std::size_t>(N, 1);
    if (prep_.exact) {
        d.succ_wi.alloc(N1, d.stream);
        d.key_i.alloc(N1, d.stream);
        d.cyc_wi.alloc(N1, d.stream);
        d.pv0.alloc(N1, d.stream);
        d.pv1.alloc(N1, d.stream);
    } else {
        d.succ_wf.alloc(N1, d.stream);
        d.key_f.alloc(N1, d.stream);
        d.cyc_wf.alloc(N1, d.stream);
    }
    for (auto* b : {&d.succ_e, &d.succ_v, &d.comp, &d.mark, &d.mark2, &d.wlist, &d.cyc_len, &d.conn,
                    &d.rem0, &d.rem1})
        b->alloc(N1, d.stream);
    d.pj0.alloc(N1, d.stream);
    d.pj1.alloc(N1, d.stream);
    d.src.alloc(R1, d.stream);
    d.iters.alloc(R1, d.stream);
    d.active.alloc(R1, d.stream);
    d.changed.alloc(R1, d.stream);
    d.lam_f.alloc(R1, d.stream);
    d.lam_num.alloc(R1, d.stream);
    d.lam_den.alloc(R1, d.stream);
    d.slot.alloc(R1, d.stream);
    d.flags.alloc(1, d.stream);
    CK(cudaStreamSynchronize(d.stream));

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
    p.mark2 = d.mark2.p;
    p.wlist = d.wlist.p;
    p.cyc_len = d.cyc_len.p;
    p.cyc_wi = d.cyc_wi.p;
    p.cyc_wf = d.cyc_wf.p;
    p.conn = d.conn.p;
    p.rem[0] = d.rem0.p;
    p.rem[1] = d.rem1.p;
    p.pv[0] = d.pv0.p;
    p.pv[1] = d.pv1.p;
    p.flags = d.flags.p;
    p.max_region = prep_.max_region;
    p.max_abs_w = prep_.max_abs_w;
    h2d_bytes_ = prep_.h2d_bytes;
    prep_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

Session::~Session() = default;

void* Session::stream() const { return d_ ? d_->stream : nullptr; }

namespace {

template <bool EXACT, int U> void launch_improve_u(const KP& p, int grid_sms, cudaStream_t s, int G) {
    const std::size_t threads = std::size_t(p.N) * G;
    const int grid = grid_for(threads, grid_sms, 8);
    switch (G) {
    case 1: k_improve<EXACT, 1, U><<<grid, kBlock, 0, s>>>(p); break;
    case 2: k_improve<EXACT, 2, U><<<grid, kBlock, 0, s>>>(p); break;
    case 4: k_improve<EXACT, 4, U><<<grid, kBlock, 0, s>>>(p); break;
    case 8: k_improve<EXACT, 8, U><<<grid, kBlock, 0, s>>>(p); break;
    case 16: k_improve<EXACT, 16, U><<<grid, kBlock, 0, s>>>(p); break;
    default: k_improve<EXACT, 32, U><<<grid, kBlock, 0, s>>>(p); break;
    }
}

// G lanes per vertex with U edges in flight per lane, G*U ~ average degree.
// OCM_IMPROVE_G / OCM_IMPROVE_U override the choice (tuning sweeps).
template <bool EXACT> void launch_improve(const KP& p, int sms, cudaStream_t s, double avg_deg) {
    static const int env_g = std::getenv("OCM_IMPROVE_G") ? std::atoi(std::getenv("OCM_IMPROVE_G")) : 0;
    static const int env_u = std::getenv("OCM_IMPROVE_U") ? std::atoi(std::getenv("OCM_IMPROVE_U")) : 0;
    const int U = env_u ? env_u : 4;
    int G = 1;
    while (G < 32 && G * U < avg_deg)
        G *= 2;
    if (env_g)
        G = env_g;
    switch (U) {
    case 1: launch_improve_u<EXACT, 1>(p, sms, s, G); break;
    case 2: launch_improve_u<EXACT, 2>(p, sms, s, G); break;
    case 8: launch_improve_u<EXACT, 8>(p, sms, s, G); break;
    default: launch_improve_u<EXACT, 4>(p, sms, s, G); break;
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
    const double avg_deg = prep_.R ? double(prep_.M) / std::max<double>(1.0, double(prep_.n - prep_.trivial)) : 1.0;
    std::uint64_t launches = 0, fix_iters = 0;
    std::uint32_t passes = 0, outer = 0;
    Flags& hf = *d.h_flags;

    // Optional per-phase CUDA-event breakdown (OCM_PHASES=1 -> one JSON line
    // on stderr per solve). Events are recorded on the launching stream.
    static const bool phases_on = std::getenv("OCM_PHASES") != nullptr;
    std::vector<std::pair<int, cudaEvent_t>> marks;
    std::vector<cudaEvent_t> pool;
    auto mark = [&](int phase) {
        if (!phases_on)
            return;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, s));
        marks.push_back({phase, e});
    };
    std::uint64_t layers_total = 0;
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
        k_init<<<gv, kBlock, 0, s>>>(p);
        ++launches;
    }
    // Upper bound on doubling rounds (2^K_max >= region size) and the
    // session's running estimates of the rounds actually needed.
    const int K_max = std::max(1, ceil_log2(std::max<std::uint32_t>(prep_.max_region, 2)));
    int k_need = std::min(K_max, k_hint_);
    std::uint32_t stamp = stamp_base_;
    // Two host synchronisations per iteration: (1) after the improvement pass
    // and the cycle-detection check (termination + round-count verdict), (2)
    // after the kept-component pass (re-attachment workload). Kernels between
    // them are gated on device flags, so the quiet final pass costs no work.
    while (prep_.R > 0) {
        mark(0);
        CK(cudaMemsetAsync(&p.flags->active_count, 0, sizeof(unsigned), s));
        CK(cudaEventRecord(d.event(2 * passes), s));
        launch_improve<EXACT>(p, d.sms, s, avg_deg);
        CK(cudaEventRecord(d.event(2 * passes + 1), s));
        ++passes;
        k_region_check<<<gr, kBlock, 0, s>>>(p);
        launches += 2;

        // cycles of the policy graph: double until the exact check passes
        mark(1);
        k_pj_init<EXACT><<<gv, kBlock, 0, s>>>(p);
        ++launches;
        int in = 0, k = 0;
        bool quiet = false;
        for (;;) {
            for (; k < k_need; ++k, in ^= 1) {
                k_pj_round<<<gv, kBlock, 0, s>>>(p, in);
                ++launches;
                ++fix_iters;
            }
            ++stamp;
            CK(cudaMemsetAsync(&p.flags->verify_fail, 0, sizeof(int), s));
            k_cycle_mark<<<gv, kBlock, 0, s>>>(p, in, stamp);
            k_cycle_verify1<<<gv, kBlock, 0, s>>>(p, stamp);
            k_cycle_verify2<<<gv, kBlock, 0, s>>>(p, stamp);
            launches += 3;
            read_flags();
            if (hf.active_count == 0) {
                quiet = true;
                break;
            }
            if (!hf.verify_fail)
                break;
            if (k >= K_max)
                throw std::logic_error("cycle detection did not converge within log2(n) rounds");
            k_need = k + 1;
        }
        if (quiet)
            break;
        ++outer;
        k_hint_ = k;

        mark(2);
        CK(cudaMemsetAsync(&p.flags->max_cycle, 0, 3 * sizeof(unsigned), s)); // + wc_count, wc_short
        if constexpr (EXACT)
            k_cycle_stats<<<gv, kBlock, 0, s>>>(p, stamp);
        else
            k_cycle_walk_float<<<gv, kBlock, 0, s>>>(p);
        k_vote<EXACT><<<gv, kBlock, 0, s>>>(p);
        k_adopt<EXACT><<<gr, kBlock, 0, s>>>(p);
        launches += 3;
        // values of the winning cycle(s): prefix sums cut at the anchor, with
        // the round count of the previous iteration (+1); re-run exactly if short
        auto wincyc = [&](int rounds) {
            CK(cudaMemsetAsync(p.flags->notdone, 0, rounds * sizeof(unsigned), s));
            const int gw = grid_for(std::max<std::uint32_t>(prep_.max_region, 1), d.sms);
            for (int j = 0; j < rounds; ++j)
                k_wincyc_round<<<gw, kBlock, 0, s>>>(p, j);
            k_wincyc_final<<<gw, kBlock, 0, s>>>(p, rounds);
            launches += 1 + rounds;
            fix_iters += rounds;
        };
        auto keep = [&] {
            CK(cudaMemsetAsync(&p.flags->rem_count[0], 0, sizeof(unsigned), s));
            k_keep<EXACT><<<gv, kBlock, 0, s>>>(p, in, stamp, 1ull << k);
            ++launches;
        };
        if constexpr (EXACT) {
            k_wincyc_init<<<gv, kBlock, 0, s>>>(p, stamp);
            ++launches;
            wincyc(std::min(kMaxRounds, wc_hint_));
        }
        keep();
        read_flags();
        if (EXACT && hf.wc_short) {
            const int rounds = std::min(kMaxRounds, ceil_log2(std::max(hf.max_cycle, 2u)) + 1);
            CK(cudaMemsetAsync(&p.flags->wc_short, 0, sizeof(int), s));
            wincyc(rounds);
            keep();
            read_flags();
            if (hf.wc_short)
                throw std::logic_error("winning-cycle prefix sums did not converge");
        }
        if (EXACT)
            wc_hint_ = std::max(2, ceil_log2(std::max(hf.max_cycle, 2u)) + 1);

        // breadth-layered re-attachment (+ values of re-attached vertices)
        mark(3);
        unsigned pending = hf.rem_count[0];
        int cur = 0;
        for (std::uint32_t layer = 1; pending > 0; ++layer) {
            CK(cudaMemsetAsync(&p.flags->rem_count[cur ^ 1], 0, sizeof(unsigned), s));
            k_attach<EXACT><<<grid_for(pending, d.sms), kBlock, 0, s>>>(p, cur, pending, layer);
            ++launches;
            ++fix_iters;
            read_flags();
            const unsigned next = hf.rem_count[cur ^ 1];
            if (next == pending)
                throw std::logic_error("connect_gpi_fixpoint: region is not strongly connected");
            pending = next;
            cur ^= 1;
            ++layers_total;
        }

        // float mode: level-synchronous value propagation (bit-exact order)
        mark(4);
        if constexpr (!EXACT) {
            k_fprop_init<<<gv, kBlock, 0, s>>>(p);
            ++launches;
            for (std::uint32_t level = 1;; ++level) {
                CK(cudaMemsetAsync(&p.flags->notdone[0], 0, sizeof(unsigned), s));
                k_fprop_round<<<gv, kBlock, 0, s>>>(p, level, 0);
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
    stamp_base_ = stamp;
    mark(5);
    CK(cudaEventRecord(d.ev_end, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    read_flags();
    if (phases_on && !marks.empty()) {
        double acc[6] = {0, 0, 0, 0, 0, 0};
        for (std::size_t i = 0; i + 1 < marks.size(); ++i) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, marks[i].second, marks[i + 1].second));
            acc[marks[i].first] += t;
        }
        for (auto& m : marks)
            cudaEventDestroy(m.second);
        std::fprintf(stderr,
                     "{\"phases_ms\": {\"improve+check\": %.3f, \"pointer_jump\": %.3f, "
                     "\"stats_vote_keep\": %.3f, \"attach\": %.3f, \"values\": %.3f}, "
                     "\"passes\": %u, \"attach_layers\": %llu, \"N\": %u, \"M\": %llu}\n",
                     acc[0], acc[1], acc[2], acc[3], acc[4], passes,
                     (unsigned long long)layers_total, p.N, (unsigned long long)prep_.M);
    }

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
    out->n_solved = prep_.n;
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
        return src[a] < src[b];
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
    std::vector<std::uint32_t> succ(prep_.n);
    CK(cudaMemcpy(succ.data(), p.succ_v, prep_.n * sizeof(std::uint32_t), cudaMemcpyDeviceToHost));
    out->d2h_bytes += prep_.n * sizeof(std::uint32_t);
    std::uint32_t u = src[best], len = 0;
    do {
        if (cycle_buf && len < cap)
            cycle_buf[len] = u;
        ++len;
        u = succ[u];
    } while (u != src[best] && len <= prep_.n);
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
    const std::size_t n = prep_.n, R1 = std::size_t(prep_.R) + 1;
    std::vector<long long> key(n), ln(R1), ld(R1);
    std::vector<double> kf(n);
    std::vector<std::uint32_t> sv(n), reg(n);
    if (n) {
        if (prep_.exact)
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
