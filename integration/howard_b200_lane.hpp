// The B200 lane as a maintainer adds it to the reference.
//
// Drop-in for proj/src/solve.cpp: include this file there (after the
// reference's own headers), add `HowardB200` to `enum class Algo`
// (proj/include/ocm/solve.hpp:21) and route it in `run_min`
// (solve.cpp:183):
//
//     case Algo::HowardB200:
//         return run_howard_b200(g, opt);
//
// Link libocm_b200.so (include/ocm_b200.h). solve() (solve.cpp:198) has
// already negated the weights for Objective::Maximize when run_min is called,
// so the lane always minimises. The graph goes to the device as the
// reference's own CSR arrays (graph.hpp:38-41), read in place: no rebuild,
// no registration of the caller's memory.
//
// `stats_like` selects whose statistics the lane reports: the sequential
// lane's (run_howard_seq, solve.cpp:43: sums over regions) or the
// data-parallel lane's (run_howard_par, solve.cpp:86: maximum over the
// concurrently iterating regions). The optimal mean and cycle are the same.
//
// Compiled against the reference headers by oracle/Makefile (target
// `integration`) and exercised by tests/test_integration_cpp.py.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "ocm_b200.h"
#include "ocm/graph.hpp"
#include "ocm/rational.hpp"
#include "ocm/solve.hpp"

namespace ocm {

inline Solution run_howard_b200(const Graph& g, const SolveOptions& opt,
                                Algo stats_like = Algo::HowardSeq, int device = 0) {
    ocm_solve_options o{};
    o.algo = stats_like == Algo::HowardPar ? OCM_ALGO_HOWARD_PAR : OCM_ALGO_HOWARD;
    o.objective = OCM_MINIMIZE; // solve() negated the weights for Maximize
    o.scc = opt.scc == SccStrategy::Off        ? OCM_SCC_OFF
            : opt.scc == SccStrategy::Parallel ? OCM_SCC_PARALLEL
                                               : OCM_SCC_TARJAN;
    o.device = device;
    o.epsilon = opt.epsilon;
    ocm_solution r{};
    std::vector<std::uint32_t> cyc(g.n > 0 ? g.n : 1);
    const int rc = ocm_solve_csr(g.n, g.m, g.fwd_index.data(), g.fwd_target.data(),
                                 g.fwd_weight.data(), &o, &r, cyc.data(),
                                 static_cast<std::uint32_t>(cyc.size()));
    if (rc == OCM_E_INVALID)
        throw std::invalid_argument(ocm_last_error());
    if (rc == OCM_E_LOGIC)
        throw std::logic_error(ocm_last_error());
    if (rc != OCM_OK)
        throw std::runtime_error(std::string("howard-b200: ") + ocm_last_error());
    Solution s;
    s.has_cycle = r.has_cycle != 0;
    s.exact = r.exact != 0;
    if (s.exact)
        s.mu_exact = Rational(r.mu_num, r.mu_den);
    s.mu = r.mu;
    if (s.has_cycle)
        s.cycle_vertices.assign(cyc.begin(), cyc.begin() + r.cycle_len);
    s.stats.outer_iters = r.outer_iters;
    s.stats.spf_passes = r.spf_passes;
    s.stats.launches = r.launches;
    s.stats.fixpoint_iters = r.fixpoint_iters;
    s.stats.regions = r.regions;
    s.stats.trivial_regions = r.trivial_regions;
    return s;
}

} // namespace ocm
