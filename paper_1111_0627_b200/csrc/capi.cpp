// extern "C" boundary of libocm_b200.so (declared in include/ocm_b200.h).
// Translates the reference's exception contract into return codes and keeps
// the last message per thread.

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>
#include <string>

#include "../../include/ocm_b200.h"
#include "errors.hpp"
#include "gen.hpp"
#include "graph.hpp"
#include "solver.hpp"

struct ocm_graph {
    ocmb::Graph g;
    // Host arrays are page-locked on first device use (one registration per
    // graph, released with the graph) so every later upload is a pinned copy.
    // The handle is read-only to callers and may be shared by threads: the
    // registration runs once under a lock, and only the ranges this graph
    // registered itself are ever unregistered.
    std::mutex pin_mu;
    std::vector<const void*> registered;
    bool pin_tried = false;
    void pin() {
        std::lock_guard<std::mutex> lock(pin_mu);
        if (pin_tried)
            return;
        pin_tried = true;
        const std::pair<const void*, std::size_t> ranges[] = {
            {g.fwd_index.data(), g.fwd_index.size() * sizeof(std::uint64_t)},
            {g.fwd_target.data(), g.fwd_target.size() * sizeof(std::uint32_t)},
            {g.fwd_weight.data(), g.fwd_weight.size() * sizeof(double)}};
        for (const auto& [p, bytes] : ranges) {
            if (bytes == 0)
                continue;
            if (cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterPortable) !=
                cudaSuccess) {
                cudaGetLastError(); // pageable copies still work, only slower
                unpin_locked();
                return;
            }
            registered.push_back(p);
        }
    }
    void unpin_locked() {
        for (const void* p : registered)
            cudaHostUnregister(const_cast<void*>(p));
        registered.clear();
        cudaGetLastError();
    }
    ~ocm_graph() { unpin_locked(); }
};
struct ocm_session {
    std::unique_ptr<ocmb::Session> s;
};

namespace {

thread_local std::string g_err;
thread_local int g_err_line = 0;

template <class F> int guard(F&& f) {
    g_err.clear();
    g_err_line = 0;
    try {
        f();
        return OCM_OK;
    } catch (const ocmb::ParseError& e) {
        g_err = e.what();
        g_err_line = e.line();
        return OCM_E_PARSE;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return OCM_E_INVALID;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return OCM_E_LOGIC;
    } catch (const ocmb::CudaError& e) {
        g_err = e.what();
        return OCM_E_CUDA;
    } catch (const ocmb::RangeError& e) {
        g_err = e.what();
        return OCM_E_RANGE;
    } catch (const ocmb::UnsupportedError& e) {
        g_err = e.what();
        return OCM_E_UNSUPPORTED;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return OCM_E_RANGE;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return OCM_E_RANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OCM_E_IO;
    }
}

ocm_solve_options defaults(const ocm_solve_options* o) {
    ocm_solve_options d{};
    d.algo = OCM_ALGO_HOWARD_PAR;
    d.objective = OCM_MINIMIZE;
    d.scc = OCM_SCC_TARJAN;
    d.device = 0;
    d.epsilon = 1e-9;
    return o ? *o : d;
}

} // namespace

extern "C" {

const char* ocm_last_error(void) { return g_err.c_str(); }
int ocm_last_error_line(void) { return g_err_line; }
const char* ocm_version(void) { return "ocm_b200 0.1 (sm_100a)"; }

int ocm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess)
        return 0;
    return n;
}

int ocm_build_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                    const double* w, ocm_graph** out) {
    return guard([&] {
        if (m && (!src || !dst || !w))
            throw std::invalid_argument("null edge arrays");
        auto g = std::make_unique<ocm_graph>();
        g->g = ocmb::build_graph(n, m, src, dst, w);
        *out = g.release();
    });
}

int ocm_parse_graph_text(const char* text, size_t len, const char* source, ocm_graph** out) {
    return guard([&] {
        auto g = std::make_unique<ocm_graph>();
        g->g = ocmb::parse_graph_text(text ? text : "", text ? len : 0, source ? source : "<text>");
        *out = g.release();
    });
}

int ocm_read_graph_file(const char* path, ocm_graph** out) {
    return guard([&] {
        auto g = std::make_unique<ocm_graph>();
        g->g = ocmb::read_graph_file(path ? path : "");
        *out = g.release();
    });
}

int ocm_generate_uniform(uint32_t n, uint32_t deg, int32_t wlo, int32_t whi, uint64_t seed,
                         ocm_graph** out) {
    return guard([&] {
        auto g = std::make_unique<ocm_graph>();
        g->g = ocmb::generate_uniform(n, deg, wlo, whi, seed);
        *out = g.release();
    });
}

namespace {
ocmb::GenSpec spec_of(const ocm_generator* g) {
    if (!g)
        throw std::invalid_argument("null generator");
    ocmb::GenSpec s;
    s.kind = g->kind;
    s.n = g->n;
    s.deg = g->deg;
    s.dmax = g->dmax;
    s.wlo = g->wlo;
    s.whi = g->whi;
    s.seed = g->seed;
    return s;
}
} // namespace

int ocm_generate(const ocm_generator* spec, ocm_graph** out) {
    return guard([&] {
        auto g = std::make_unique<ocm_graph>();
        g->g = ocmb::generate(spec_of(spec));
        *out = g.release();
    });
}

int ocm_session_create_generated(const ocm_generator* spec, const ocm_solve_options* opt,
                                 ocm_session** out) {
    return guard([&] {
        auto s = std::make_unique<ocm_session>();
        s->s = std::make_unique<ocmb::Session>(spec_of(spec), defaults(opt));
        *out = s.release();
    });
}

uint32_t ocm_session_n(const ocm_session* s) { return s ? s->s->n() : 0; }

int ocm_session_create_shard(const ocm_graph* g, const ocm_generator* spec,
                             const ocm_solve_options* opt, uint32_t rank, uint32_t world,
                             ocm_session** out) {
    return guard([&] {
        if ((g == nullptr) == (spec == nullptr))
            throw std::invalid_argument("pass exactly one of a graph and a generator");
        auto s = std::make_unique<ocm_session>();
        if (g) {
            const_cast<ocm_graph*>(g)->pin();
            s->s = std::make_unique<ocmb::Session>(g->g, defaults(opt), rank, world);
        } else {
            s->s = std::make_unique<ocmb::Session>(spec_of(spec), defaults(opt), rank, world);
        }
        *out = s.release();
    });
}

int ocm_session_shard_buffers(ocm_session* s, ocm_shard_buffers* out) {
    return guard([&] { s->s->shard_buffers(out); });
}

int ocm_session_shard_step(ocm_session* s, int32_t* done) {
    return guard([&] { *done = s->s->shard_step() ? 1 : 0; });
}

int ocm_session_shard_finish(ocm_session* s, ocm_solution* out, uint32_t* cycle_buf,
                             uint32_t cycle_cap) {
    return guard([&] { s->s->shard_finish(out, cycle_buf, cycle_cap); });
}

int ocm_session_shard_peer_info(ocm_session* s, ocm_shard_peer* out) {
    return guard([&] { s->s->shard_peer_info(out); });
}

int ocm_session_shard_connect(ocm_session* s, const ocm_shard_peer* peers, uint32_t world,
                              int32_t use_ipc) {
    return guard([&] {
        if (!peers)
            throw std::invalid_argument("null peer list");
        s->s->shard_connect(peers, world, use_ipc != 0);
    });
}

int ocm_session_shard_fused_launch(ocm_session* s) {
    return guard([&] { s->s->fused_launch(); });
}

int ocm_session_shard_fused_finish(ocm_session* s, ocm_solution* out, uint32_t* cycle_buf,
                                   uint32_t cycle_cap) {
    return guard([&] { s->s->fused_finish(out, cycle_buf, cycle_cap); });
}

int ocm_generate_model(uint32_t states, const ocm_transition* transitions, uint32_t n_transitions,
                       int32_t uses_server, uint32_t clients, uint64_t max_states,
                       ocm_graph** out) {
    return guard([&] {
        if (n_transitions && !transitions)
            throw std::invalid_argument("null transition array");
        ocmb::Scenario sc;
        sc.states = states;
        sc.uses_server = uses_server != 0;
        for (uint32_t i = 0; i < n_transitions; ++i)
            sc.transitions.push_back({transitions[i].from, transitions[i].to, transitions[i].cost,
                                      transitions[i].acquires != 0, transitions[i].releases != 0});
        auto g = std::make_unique<ocm_graph>();
        g->g = ocmb::generate_model(sc, clients, max_states ? max_states : 5000000ull);
        *out = g.release();
    });
}

void ocm_graph_free(ocm_graph* g) { delete g; }
uint32_t ocm_graph_n(const ocm_graph* g) { return g ? g->g.n : 0; }
uint64_t ocm_graph_m(const ocm_graph* g) { return g ? g->g.m : 0; }
int ocm_graph_integer_exact(const ocm_graph* g) { return g && g->g.integer_exact ? 1 : 0; }

int ocm_graph_csr(const ocm_graph* g, const uint64_t** fwd_index, const uint32_t** fwd_target,
                  const double** fwd_weight) {
    return guard([&] {
        if (!g || !fwd_index || !fwd_target || !fwd_weight)
            throw std::invalid_argument("null graph or output");
        *fwd_index = g->g.fwd_index.data();
        *fwd_target = g->g.fwd_target.data();
        *fwd_weight = g->g.fwd_weight.data();
    });
}

int ocm_graph_edges(const ocm_graph* g, uint32_t* src, uint32_t* dst, double* w) {
    return guard([&] { ocmb::graph_edges(g->g, src, dst, w); });
}

int ocm_session_create(const ocm_graph* g, const ocm_solve_options* opt, ocm_session** out) {
    return guard([&] {
        if (!g)
            throw std::invalid_argument("null graph");
        const_cast<ocm_graph*>(g)->pin();
        auto s = std::make_unique<ocm_session>();
        s->s = std::make_unique<ocmb::Session>(g->g, defaults(opt));
        *out = s.release();
    });
}

int ocm_session_solve(ocm_session* s, ocm_solution* out, uint32_t* cycle_buf, uint32_t cycle_cap) {
    return guard([&] { s->s->solve(out, cycle_buf, cycle_cap); });
}

int ocm_session_values(ocm_session* s, int64_t* key_num, int64_t* lam_num, int64_t* lam_den,
                       double* fval, uint32_t* succ_vertex) {
    return guard([&] { s->s->values(key_num, lam_num, lam_den, fval, succ_vertex); });
}

int ocm_session_certify(ocm_session* s, ocm_certificate* out) {
    return guard([&] {
        if (!s || !out)
            throw std::invalid_argument("null session or output");
        s->s->certify(out);
    });
}

int ocm_session_keys_wide(ocm_session* s, int64_t* key_hi, uint64_t* key_lo) {
    return guard([&] {
        if (!s || !key_hi || !key_lo)
            throw std::invalid_argument("null session or output");
        s->s->keys_wide(key_hi, key_lo);
    });
}

int ocm_session_lambda_trace(ocm_session* s, int64_t* num, int64_t* den, double* f, uint32_t cap,
                             uint32_t* len) {
    return guard([&] {
        if (!s || !len)
            throw std::invalid_argument("null session or output");
        s->s->lambda_trace(num, den, f, cap, len);
    });
}

int ocm_session_iter_trace(ocm_session* s, uint32_t iter, uint32_t* succ_edge, int64_t* key,
                           double* fval) {
    return guard([&] {
        if (!s)
            throw std::invalid_argument("null session");
        s->s->iter_trace(iter, succ_edge, key, fval);
    });
}

int ocm_session_is_wide(const ocm_session* s) { return s && s->s->wide() ? 1 : 0; }

void* ocm_session_stream(ocm_session* s) { return s ? s->s->stream() : nullptr; }

void ocm_session_free(ocm_session* s) { delete s; }

int ocm_solve(const ocm_graph* g, const ocm_solve_options* opt, ocm_solution* out,
              uint32_t* cycle_buf, uint32_t cycle_cap) {
    return guard([&] {
        if (!g)
            throw std::invalid_argument("null graph");
        std::memset(out, 0, sizeof *out);
        out->mu_den = 1;
        if (g->g.n == 0)
            return; // solve.cpp:199: an empty graph has no cycle
        const_cast<ocm_graph*>(g)->pin();
        ocmb::Session sess(g->g, defaults(opt));
        sess.solve(out, cycle_buf, cycle_cap);
    });
}

int ocm_solve_csr(uint32_t n, uint32_t m, const uint32_t* fwd_index, const uint32_t* fwd_target,
                  const double* fwd_weight, const ocm_solve_options* opt, ocm_solution* out,
                  uint32_t* cycle_buf, uint32_t cycle_cap) {
    return guard([&] {
        if (!out || (n && !fwd_index) || (m && (!fwd_target || !fwd_weight)))
            throw std::invalid_argument("null CSR array or output");
        std::memset(out, 0, sizeof *out);
        out->mu_den = 1;
        if (n == 0) {
            if (m)
                throw std::invalid_argument("edge 0 endpoint out of range");
            return; // solve.cpp:199: an empty graph has no cycle
        }
        ocmb::HostCsr h;
        h.n = n;
        h.m = m;
        h.index32 = fwd_index;
        h.target = fwd_target;
        h.weight = fwd_weight;
        h.validated = false;
        ocmb::Session sess(h, defaults(opt));
        sess.solve(out, cycle_buf, cycle_cap);
    });
}

int ocm_session_create_csr(uint32_t n, uint32_t m, const uint32_t* fwd_index,
                           const uint32_t* fwd_target, const double* fwd_weight,
                           const ocm_solve_options* opt, ocm_session** out) {
    return guard([&] {
        if (!out || !fwd_index || (m && (!fwd_target || !fwd_weight)))
            throw std::invalid_argument("null CSR array or output");
        ocmb::HostCsr h;
        h.n = n;
        h.m = m;
        h.index32 = fwd_index;
        h.target = fwd_target;
        h.weight = fwd_weight;
        h.validated = false;
        auto s = std::make_unique<ocm_session>();
        s->s = std::make_unique<ocmb::Session>(h, defaults(opt));
        *out = s.release();
    });
}

} // extern "C"
