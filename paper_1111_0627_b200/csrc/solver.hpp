// Device session of the B200 optimal-cycle-mean solver (policy iteration,
// data-parallel decomposition of the reference's howard-par lane,
// proj/include/ocm/howard_par.hpp). See DESIGN.md for the kernel list.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

#include "../../include/ocm_b200.h"
#include "gen.hpp"
#include "graph.hpp"
#include "prepinfo.hpp"

namespace ocmb {

struct DeviceState; // devcommon.cuh

class Session {
  public:
    Session(const Graph& g, const ocm_solve_options& opt);
    // graph generated directly in HBM (gen_dev.cu)
    Session(const GenSpec& spec, const ocm_solve_options& opt);
    ~Session();
    void solve(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);
    void values(std::int64_t* key_num, std::int64_t* lam_num, std::int64_t* lam_den, double* fval,
                std::uint32_t* succ_vertex);
    void* stream() const;

    std::uint32_t n() const { return prep_.n; }

  private:
    void init(const std::function<void(DeviceState&)>& prepare);
    template <class M> void run(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);
    ocm_solve_options opt_;
    PrepInfo prep_;
    double prep_ms_ = 0.0;
    std::uint64_t h2d_bytes_ = 0;
    std::unique_ptr<DeviceState> d_;
    bool solved_ = false;
    int grid_exact_ = 0, grid_float_ = 0; // cooperative grid of k_solve<exact / float>
};

} // namespace ocmb
