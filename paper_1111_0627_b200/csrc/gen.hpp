// Seeded synthetic graph generators (benchmark workloads). The counter hash
// is bit-identical to oracle/ocm_oracle.c so checkers see the same graphs.
#pragma once

#include <cstdint>
#include <vector>

#include "graph.hpp"

namespace ocmb {

// Every vertex gets exactly `deg` out-edges (edge i of v has id v*deg+i);
// targets uniform over [0, n), integer weights uniform in [wlo, whi].
Graph generate_uniform(std::uint32_t n, std::uint32_t deg, std::int32_t wlo, std::int32_t whi,
                       std::uint64_t seed);

} // namespace ocmb

namespace ocmb {

// Composite state spaces of interleaved client state machines
// (proj/include/ocm/model_gen.hpp): one vertex per reachable composite state
// numbered in breadth-first discovery order (clients, then transitions, in
// declaration order), one edge per enabled transition with its cost.
struct ScenarioTransition {
    std::uint32_t from = 0, to = 0;
    std::int64_t cost = 0;
    bool acquires = false; // enabled only while the server is free
    bool releases = false; // enabled only for the current holder
};

struct Scenario {
    std::uint32_t states = 0;
    std::vector<ScenarioTransition> transitions;
    bool uses_server = false;
};

// model_gen.hpp:67 generate_model. Throws std::invalid_argument on
// malformed scenarios and std::length_error past max_states (the
// reference's bound is kMaxModelStates = 5'000'000).
Graph generate_model(const Scenario& sc, std::uint32_t clients, std::uint64_t max_states);

} // namespace ocmb
