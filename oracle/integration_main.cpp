// TEST INFRASTRUCTURE ONLY — the drop-in boundary proven in C++.
//
// Compiled by oracle/Makefile (target `integration`) against the reference's
// own headers and sources (unmodified, in place) plus integration/
// howard_b200_lane.hpp, linked to the product library libocm_b200.so.
// For every graph file on the command line it reads the graph with the
// reference's read_graph_file (graph_io.hpp:45), then for each objective and
// SCC strategy (tarjan, parallel, off) solves it twice:
//   * the reference's ocm::solve (solve.cpp:198) with lane howard and with
//     lane howard-par;
//   * the same solve() front end (negation for Maximize, solve.cpp:203-215)
//     dispatching to run_howard_b200 -- exactly what the patched solve.cpp of
//     INTEGRATION.md §1 runs -- with the matching statistics convention;
// and prints one line per comparison:
//   OK|FAIL <file> <objective> <scc> <lane> [detail]
// Exit status 0 iff every comparison matched (mean as an exact rational or
// the same double, cycle vertices, outer iterations, improvement passes,
// region counts).

#include <cstdio>
#include <exception>
#include <string>

#include "howard_b200_lane.hpp"
#include "ocm/graph_io.hpp"

namespace {

ocm::Solution solve_b200(const ocm::Graph& input, const ocm::SolveOptions& opt, ocm::Algo like) {
    if (input.n == 0)
        return {};
    ocm::Graph negated;
    const bool maximize = opt.objective == ocm::Objective::Maximize;
    if (maximize)
        negated = ocm::negate_weights(input);
    const ocm::Graph& g = maximize ? negated : input;
    ocm::Solution s = ocm::run_howard_b200(g, opt, like);
    if (maximize && s.has_cycle) {
        s.mu = -s.mu;
        if (s.exact)
            s.mu_exact = -s.mu_exact;
    }
    return s;
}

std::string diff(const ocm::Solution& a, const ocm::Solution& b) {
    if (a.has_cycle != b.has_cycle)
        return "has_cycle";
    if (a.has_cycle) {
        if (a.exact != b.exact)
            return "exact";
        if (a.exact && !(a.mu_exact == b.mu_exact))
            return "mu " + std::to_string(a.mu_exact.num) + "/" + std::to_string(a.mu_exact.den) +
                   " vs " + std::to_string(b.mu_exact.num) + "/" + std::to_string(b.mu_exact.den);
        if (a.mu != b.mu)
            return "mu(double)";
        if (a.cycle_vertices != b.cycle_vertices)
            return "cycle";
    }
    if (a.stats.outer_iters != b.stats.outer_iters || a.stats.spf_passes != b.stats.spf_passes)
        return "stats " + std::to_string(a.stats.outer_iters) + "/" +
               std::to_string(a.stats.spf_passes) + " vs " + std::to_string(b.stats.outer_iters) +
               "/" + std::to_string(b.stats.spf_passes);
    if (a.stats.regions != b.stats.regions || a.stats.trivial_regions != b.stats.trivial_regions)
        return "regions";
    return "";
}

} // namespace

int main(int argc, char** argv) {
    int bad = 0;
    for (int i = 1; i < argc; ++i) {
        const std::string path = argv[i];
        ocm::Graph g;
        try {
            g = ocm::read_graph_file(path);
        } catch (const std::exception& e) {
            std::printf("FAIL %s read %s\n", path.c_str(), e.what());
            ++bad;
            continue;
        }
        for (const auto obj : {ocm::Objective::Minimize, ocm::Objective::Maximize})
            for (const auto scc : {ocm::SccStrategy::Tarjan, ocm::SccStrategy::Parallel,
                                   ocm::SccStrategy::Off})
                for (const auto lane : {ocm::Algo::HowardSeq, ocm::Algo::HowardPar}) {
                    ocm::SolveOptions opt;
                    opt.algo = lane;
                    opt.objective = obj;
                    opt.scc = scc;
                    const char* on = obj == ocm::Objective::Minimize ? "min" : "max";
                    const char* sn = scc == ocm::SccStrategy::Off        ? "off"
                                     : scc == ocm::SccStrategy::Parallel ? "parallel"
                                                                         : "tarjan";
                    const char* ln = lane == ocm::Algo::HowardSeq ? "howard" : "howard-par";
                    try {
                        const ocm::Solution ref = ocm::solve(g, opt);
                        const ocm::Solution dev = solve_b200(g, opt, lane);
                        const std::string d = diff(ref, dev);
                        std::printf("%s %s %s %s %s %s\n", d.empty() ? "OK" : "FAIL", path.c_str(),
                                    on, sn, ln, d.c_str());
                        bad += !d.empty();
                    } catch (const std::exception& e) {
                        std::printf("FAIL %s %s %s %s exception %s\n", path.c_str(), on, sn, ln,
                                    e.what());
                        ++bad;
                    }
                }
    }
    return bad ? 1 : 0;
}
