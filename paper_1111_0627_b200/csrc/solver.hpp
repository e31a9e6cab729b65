// Device session of the B200 optimal-cycle-mean solver (policy iteration,
// data-parallel decomposition of the reference's howard-par lane,
// proj/include/ocm/howard_par.hpp). See DESIGN.md for the kernel list.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "../../include/ocm_b200.h"
#include "graph.hpp"

namespace ocmb {

// Host-side split of a graph into solver regions: strongly connected
// components (Tarjan) minus trivial ones, renumbered so every region is a
// contiguous vertex range (ascending original id inside a region, so "least
// vertex of a cycle" is the same under both numberings), with the CSR
// restricted to intra-region edges (relative edge order preserved, so
// "smallest edge id" tie-breaks are unchanged).
struct Prepared {
    std::uint32_t n_orig = 0;
    std::uint32_t N = 0;            // vertices in non-trivial regions
    std::uint32_t R = 0;            // non-trivial regions
    std::uint32_t regions_total = 0;
    std::uint32_t trivial = 0;
    std::uint64_t M = 0;            // intra-region edges
    std::uint32_t max_region = 0;
    bool exact = false;
    bool scc_off = false;
    double no_cycle_above = 0.0;
    std::int64_t max_abs_w = 0;     // exact mode
    std::vector<std::uint32_t> orig;   // N
    std::vector<std::uint32_t> reg;    // N
    std::vector<std::uint32_t> row;    // N+1
    std::vector<std::uint32_t> tgt;    // M
    std::vector<double> w;             // M (already sign-flipped for maximize)
};

Prepared prepare(const Graph& g, const ocm_solve_options& opt);

struct DeviceState; // defined in solver.cu

class Session {
  public:
    Session(const Graph& g, const ocm_solve_options& opt);
    ~Session();
    void solve(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);
    void values(std::int64_t* key_num, std::int64_t* lam_num, std::int64_t* lam_den, double* fval,
                std::uint32_t* succ_vertex);
    void* stream() const;

  private:
    template <class M> void run(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);
    ocm_solve_options opt_;
    Prepared prep_;
    double prep_ms_ = 0.0;
    std::uint64_t h2d_bytes_ = 0;
    std::unique_ptr<DeviceState> d_;
    bool solved_ = false;
    int k_hint_ = 8;               // doubling rounds needed last iteration
    std::uint32_t stamp_base_ = 0; // mark stamps stay unique across solves
};

} // namespace ocmb
