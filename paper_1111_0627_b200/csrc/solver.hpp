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

constexpr std::uint32_t kTraceCap = 4096; // lambda trace entries kept per solve

class Session {
  public:
    // rank/world > 1: a shard of the sharded lane; the rank
    // improves the policy of vertices [rank*chunk, (rank+1)*chunk) only.
    Session(const Graph& g, const ocm_solve_options& opt, std::uint32_t rank = 0,
            std::uint32_t world = 1);
    // a host CSR in the caller's memory (e.g. the reference's ocm::Graph)
    Session(const HostCsr& g, const ocm_solve_options& opt, std::uint32_t rank = 0,
            std::uint32_t world = 1);
    // graph generated directly in HBM (gen_dev.cu)
    Session(const GenSpec& spec, const ocm_solve_options& opt, std::uint32_t rank = 0,
            std::uint32_t world = 1);
    ~Session();
    void solve(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);
    void certify(ocm_certificate* out);
    void values(std::int64_t* key_num, std::int64_t* lam_num, std::int64_t* lam_den, double* fval,
                std::uint32_t* succ_vertex);
    void* stream() const;
    void keys_wide(std::int64_t* hi, std::uint64_t* lo);
    void lambda_trace(std::int64_t* num, std::int64_t* den, double* f, std::uint32_t cap,
                      std::uint32_t* len);
    void iter_trace(std::uint32_t it, std::uint32_t* succ_e, std::int64_t* key, double* fval);
    bool wide() const { return mode_ == 2; }

    std::uint32_t n() const { return prep_.n; }

    // Sharded lane: one launch up to the next exchange point (true when the
    // solve finished), the device buffers the host exchanges between
    // launches, and the result of the finished solve.
    bool shard_step();
    void shard_buffers(ocm_shard_buffers* b) const;
    void shard_finish(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);
    // Fused sharded lane: exchange buffer descriptors (device pointers + IPC
    // handles), map the peers', then one launch per solve per rank.
    void shard_peer_info(ocm_shard_peer* out) const;
    void shard_connect(const ocm_shard_peer* peers, std::uint32_t world, bool ipc);
    void fused_launch();
    void fused_finish(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);

  private:
    void init(const std::function<void(DeviceState&)>& prepare);
    template <class M> float launch(int mode);
    template <class M> void launch_async(int mode);
    float launch_wait();
    template <class M> void collect(ocm_solution* out, std::uint32_t* cycle_buf, std::uint32_t cap);
    ocm_solve_options opt_;
    PrepInfo prep_;
    double prep_ms_ = 0.0;
    std::uint64_t h2d_bytes_ = 0;
    std::unique_ptr<DeviceState> d_;
    bool solved_ = false;
    int grid_ = 0; // cooperative grid of the session's k_solve instantiation
    int gi_ = 0;   // its improvement group width (index into 1, 2, 4, 8)
    std::uint32_t rank_ = 0, world_ = 1, chunk_ = 0;
    void build_blocked_edges();
    void choose_hubs();
    std::size_t dyn_smem_bytes() const;
    void alloc_wide();
    void promote_wide();
    int mode_ = 1; // k_solve arithmetic: 0 float, 1 exact (64-bit keys), 2 wide exact (128-bit)
    int krow() const; // solve_fn row: mode_, or 3 for the exact lane with 3 doubling steps per pass
    std::size_t hot_bytes_ = 0;    // dynamic shared memory of the staged hub table
    double hot_coverage_ = 0.0;    // share of intra-region edges into the staged hubs
    bool shard_started_ = false;
    bool connected_ = false; // fused sharded lane: peers mapped
    bool fused_broken_ = false; // a cross-rank barrier timed out (epochs out of step)
    double solve_ms_ = 0.0;   // event time of the current solve's launches
    std::uint64_t d2h_ = 0;   // device->host bytes of the current solve
    unsigned launches_ = 0;   // launches of the current solve
};

} // namespace ocmb
