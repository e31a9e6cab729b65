// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (compiled from the
// reference's own sources in place by oracle/Makefile into oracle/_ref/).
// It exists so tests/, bench.py's reference arm and the golden-vector script
// can drive the reference's public entry points from Python via ctypes:
//
//   ocm::build_graph           proj/include/ocm/graph.hpp:76
//   ocm::solve                 proj/include/ocm/solve.hpp:64  (src/solve.cpp:198)
//   ocm::HowardPar<M>::run     proj/include/ocm/howard_par.hpp:544
//   ocm::tarjan_scc            proj/include/ocm/scc.hpp:34
//   ocm::generate_model        proj/include/ocm/model_gen.hpp:67
//   ocm::parse_graph_text      proj/include/ocm/graph_io.hpp:41
//
// Nothing here re-implements the algorithm; it only marshals arrays.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ocm/graph.hpp"
#include "ocm/graph_io.hpp"
#include "ocm/howard_par.hpp"
#include "ocm/model_gen.hpp"
#include "ocm/scc.hpp"
#include "ocm/solve.hpp"

namespace {

thread_local std::string g_err;

ocm::Graph make_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                      const double* w) {
    std::vector<ocm::EdgeInput> es(m);
    for (uint64_t i = 0; i < m; ++i)
        es[i] = {src[i], dst[i], w[i]};
    return ocm::build_graph(n, es);
}

} // namespace

extern "C" {

struct ref_result {
    int32_t has_cycle;
    int32_t exact;
    int64_t mu_num;
    int64_t mu_den;
    double mu;
    uint32_t cycle_len;     // full length of the optimal cycle
    uint32_t outer_iters;
    uint32_t spf_passes;
    uint32_t regions;
    uint32_t trivial_regions;
    uint64_t launches;
    uint64_t fixpoint_iters;
    double solve_ms;        // wall time of ocm::solve only (graph already built)
    double build_ms;        // wall time of ocm::build_graph
};

const char* ref_last_error(void) { return g_err.c_str(); }

// algo: 0 howard, 1 howard-par, 2 lawler, 3 tree, 4 oracle-enum, 5 oracle-dp
// objective: 0 min, 1 max; scc: 0 tarjan, 1 parallel, 2 off
// schedule: 0 seq, 1 par, 2 shuffle
int ref_solve(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst, const double* w,
              int algo, int objective, int scc, int schedule, unsigned workers, uint64_t seed,
              double epsilon, ref_result* out, uint32_t* cycle_buf, uint32_t cycle_cap) {
    try {
        auto t0 = std::chrono::steady_clock::now();
        const ocm::Graph g = make_graph(n, m, src, dst, w);
        auto t1 = std::chrono::steady_clock::now();
        ocm::SolveOptions opt;
        opt.algo = static_cast<ocm::Algo>(algo);
        opt.objective = objective ? ocm::Objective::Maximize : ocm::Objective::Minimize;
        opt.scc = static_cast<ocm::SccStrategy>(scc);
        opt.epsilon = epsilon;
        opt.engine.schedule = static_cast<ocm::Schedule>(schedule);
        opt.engine.workers = workers;
        opt.engine.seed = seed;
        const ocm::Solution s = ocm::solve(g, opt);
        auto t2 = std::chrono::steady_clock::now();
        std::memset(out, 0, sizeof *out);
        out->has_cycle = s.has_cycle;
        out->exact = s.exact;
        out->mu_num = s.mu_exact.num;
        out->mu_den = s.mu_exact.den;
        out->mu = s.mu;
        out->cycle_len = static_cast<uint32_t>(s.cycle_vertices.size());
        for (uint32_t i = 0; i < out->cycle_len && i < cycle_cap; ++i)
            cycle_buf[i] = s.cycle_vertices[i];
        out->outer_iters = s.stats.outer_iters;
        out->spf_passes = s.stats.spf_passes;
        out->regions = s.stats.regions;
        out->trivial_regions = s.stats.trivial_regions;
        out->launches = s.stats.launches;
        out->fixpoint_iters = s.stats.fixpoint_iters;
        out->build_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        out->solve_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Runs the reference's region-concurrent data-parallel lane (HowardPar over
// the Tarjan partition, exactly what solve() does for --algo howard-par
// --scc tarjan) and exports the final per-vertex value plane: the plane the
// last value propagation wrote (howard_par.hpp:589 pushes the same plane into
// the trace). Exact graphs fill wsum/steps, float graphs fill fval.
// region_lambda_* receive, per vertex, the lambda of the vertex's region
// (0/1 for trivial regions) so values can be compared as exact rationals.
int ref_howard_values(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                      const double* w, int objective, int64_t* wsum, int64_t* steps,
                      double* fval, int64_t* lam_num, int64_t* lam_den, double* lam_f,
                      uint32_t* succ_vertex) {
    try {
        ocm::Graph g = make_graph(n, m, src, dst, w);
        if (objective)
            g = ocm::negate_weights(g);
        const ocm::RegionMap rm = ocm::tarjan_scc(g);
        ocm::Engine eng({ocm::Schedule::Seq, 1, 1});
        if (g.integer_exact) {
            ocm::HowardPar<ocm::ExactMode> hp(eng, g, rm);
            hp.run();
            const auto& plane = hp.vals.plane[hp.parity];
            for (uint32_t v = 0; v < n; ++v) {
                wsum[v] = plane[v].wsum;
                steps[v] = plane[v].steps;
                const ocm::Rational l = hp.lambda[rm.region_of[v]];
                lam_num[v] = l.num;
                lam_den[v] = l.den;
                const ocm::EdgeId e = hp.pg.succ_edge[v];
                succ_vertex[v] = e == ocm::kNoEdge ? ocm::kNoVertex : g.fwd_target[e];
            }
        } else {
            ocm::HowardPar<ocm::FloatMode> hp(eng, g, rm);
            hp.run();
            const auto& plane = hp.vals.plane[hp.parity];
            for (uint32_t v = 0; v < n; ++v) {
                fval[v] = plane[v];
                lam_f[v] = hp.lambda[rm.region_of[v]];
                const ocm::EdgeId e = hp.pg.succ_edge[v];
                succ_vertex[v] = e == ocm::kNoEdge ? ocm::kNoVertex : g.fwd_target[e];
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// kind: 0 worker_scenario, 1 server_scenario, 2 loop_scenario(costs).
// Writes the generated graph's edges in edge-id order when the capacity
// suffices; always reports n and m. Returns 1 on a reference exception.
int ref_generate_model(int kind, const int64_t* costs, uint32_t n_costs, uint32_t clients,
                       uint32_t* n_out, uint64_t* m_out, uint64_t cap, uint32_t* src,
                       uint32_t* dst, double* w) {
    try {
        ocm::Scenario sc = kind == 0 ? ocm::worker_scenario()
                           : kind == 1 ? ocm::server_scenario()
                                       : ocm::loop_scenario(std::vector<std::int64_t>(costs, costs + n_costs));
        const ocm::GeneratedModel m = ocm::generate_model(sc, clients);
        *n_out = m.graph.n;
        *m_out = m.graph.m;
        if (cap >= m.graph.m) {
            for (uint32_t u = 0; u < m.graph.n; ++u)
                for (uint64_t e = m.graph.fwd_index[u]; e < m.graph.fwd_index[u + 1]; ++e) {
                    src[e] = u;
                    dst[e] = m.graph.fwd_target[e];
                    w[e] = m.graph.fwd_weight[e];
                }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// ocm::parse_graph_text on `text`: returns 0 and n/m (+ the edges in edge-id
// order when cap >= m), 1 with the message in ref_last_error() and the line in
// *line_out on a ParseError, 2 on any other exception (message likewise).
int ref_parse_graph_text(const char* text, uint64_t len, const char* source, uint32_t* n_out,
                         uint64_t* m_out, int32_t* exact_out, uint64_t cap, uint32_t* src,
                         uint32_t* dst, double* w, int32_t* line_out) {
    try {
        const ocm::Graph g = ocm::parse_graph_text(std::string_view(text, len), source);
        *n_out = g.n;
        *m_out = g.m;
        *exact_out = g.integer_exact;
        if (cap >= g.m)
            for (uint64_t e = 0; e < g.m; ++e) {
                src[e] = g.fwd_source[e];
                dst[e] = g.fwd_target[e];
                w[e] = g.fwd_weight[e];
            }
        return 0;
    } catch (const ocm::ParseError& e) {
        g_err = e.what();
        *line_out = e.line();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// A reference Graph built once and solved many times (possibly from several
// threads at once: ocm::solve only reads the const Graph), so timing loops
// measure ocm::solve alone.
void* ref_graph_create(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                       const double* w) {
    try {
        return new ocm::Graph(make_graph(n, m, src, dst, w));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_graph_free(void* g) { delete static_cast<ocm::Graph*>(g); }

int ref_graph_solve(const void* gp, int algo, int objective, int scc, ref_result* out,
                    uint32_t* cycle_buf, uint32_t cycle_cap) {
    try {
        const ocm::Graph& g = *static_cast<const ocm::Graph*>(gp);
        ocm::SolveOptions opt;
        opt.algo = static_cast<ocm::Algo>(algo);
        opt.objective = objective ? ocm::Objective::Maximize : ocm::Objective::Minimize;
        opt.scc = static_cast<ocm::SccStrategy>(scc);
        auto t0 = std::chrono::steady_clock::now();
        const ocm::Solution s = ocm::solve(g, opt);
        auto t1 = std::chrono::steady_clock::now();
        std::memset(out, 0, sizeof *out);
        out->has_cycle = s.has_cycle;
        out->exact = s.exact;
        out->mu_num = s.mu_exact.num;
        out->mu_den = s.mu_exact.den;
        out->mu = s.mu;
        out->cycle_len = static_cast<uint32_t>(s.cycle_vertices.size());
        for (uint32_t i = 0; i < out->cycle_len && i < cycle_cap; ++i)
            cycle_buf[i] = s.cycle_vertices[i];
        out->outer_iters = s.stats.outer_iters;
        out->spf_passes = s.stats.spf_passes;
        out->regions = s.stats.regions;
        out->trivial_regions = s.stats.trivial_regions;
        out->launches = s.stats.launches;
        out->fixpoint_iters = s.stats.fixpoint_iters;
        out->solve_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_lambda_trace2(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                      const double* w, int objective, int scc_off, int64_t* num, int64_t* den,
                      double* f, uint32_t cap, uint32_t* len);

// The reference's per-iteration lambda trace (HowardPar::run(trace),
// howard_par.hpp:588, recorded when the graph is a single region): exact
// graphs fill num/den, float graphs f; returns the iteration count in *len
// (at most cap entries written). Returns 1 on an exception, 2 when the graph
// is not one region.
int ref_lambda_trace(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const double* w, int objective, int64_t* num, int64_t* den, double* f,
                     uint32_t cap, uint32_t* len) {
    return ref_lambda_trace2(n, m, src, dst, w, objective, 0, num, den, f, cap, len);
}

// scc_off: the trace of the Hamiltonian-augmented graph solve() runs for
// --scc off (solve.cpp:48, graph.cpp:105) -- one region by construction
int ref_lambda_trace2(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                      const double* w, int objective, int scc_off, int64_t* num, int64_t* den,
                      double* f, uint32_t cap, uint32_t* len) {
    try {
        ocm::Graph g = make_graph(n, m, src, dst, w);
        if (objective)
            g = ocm::negate_weights(g);
        if (scc_off)
            g = ocm::augment_hamiltonian(g).graph;
        const ocm::RegionMap rm = ocm::tarjan_scc(g);
        if (rm.count != 1)
            return 2;
        ocm::Engine eng({ocm::Schedule::Seq, 1, 1});
        if (g.integer_exact) {
            ocm::HowardPar<ocm::ExactMode> hp(eng, g, rm);
            ocm::HowardTrace<ocm::ExactMode> tr;
            hp.run(&tr);
            *len = static_cast<uint32_t>(tr.size());
            for (uint32_t i = 0; i < tr.size() && i < cap; ++i) {
                num[i] = tr[i].lambda.num;
                den[i] = tr[i].lambda.den;
            }
        } else {
            ocm::HowardPar<ocm::FloatMode> hp(eng, g, rm);
            ocm::HowardTrace<ocm::FloatMode> tr;
            hp.run(&tr);
            *len = static_cast<uint32_t>(tr.size());
            for (uint32_t i = 0; i < tr.size() && i < cap; ++i)
                f[i] = tr[i].lambda;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// The reference's full per-iteration trace on a single-region graph: for
// iteration i < cap_iters, succ_edge[i*n + v], and the value plane (exact:
// wsum/steps, float: fval). *len = iterations. Returns 2 when not one region.
int ref_iter_trace(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                   const double* w, int objective, uint32_t cap_iters, uint32_t* succ_edge,
                   int64_t* wsum, int64_t* steps, double* fval, uint32_t* len) {
    try {
        ocm::Graph g = make_graph(n, m, src, dst, w);
        if (objective)
            g = ocm::negate_weights(g);
        const ocm::RegionMap rm = ocm::tarjan_scc(g);
        if (rm.count != 1)
            return 2;
        ocm::Engine eng({ocm::Schedule::Seq, 1, 1});
        auto dump = [&](const auto& tr, auto&& put) {
            *len = static_cast<uint32_t>(tr.size());
            for (uint32_t i = 0; i < tr.size() && i < cap_iters; ++i)
                for (uint32_t v = 0; v < n; ++v) {
                    succ_edge[std::size_t(i) * n + v] = tr[i].succ_edge[v];
                    put(std::size_t(i) * n + v, tr[i].values[v]);
                }
        };
        if (g.integer_exact) {
            ocm::HowardPar<ocm::ExactMode> hp(eng, g, rm);
            ocm::HowardTrace<ocm::ExactMode> tr;
            hp.run(&tr);
            dump(tr, [&](std::size_t k, const auto& val) {
                wsum[k] = val.wsum;
                steps[k] = val.steps;
            });
        } else {
            ocm::HowardPar<ocm::FloatMode> hp(eng, g, rm);
            ocm::HowardTrace<ocm::FloatMode> tr;
            hp.run(&tr);
            dump(tr, [&](std::size_t k, const auto& val) { fval[k] = val; });
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

} // extern "C"
