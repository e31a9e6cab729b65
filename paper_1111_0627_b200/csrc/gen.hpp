// Seeded synthetic graph generators (benchmark workloads). The counter hash
// is bit-identical to oracle/ocm_oracle.c so checkers see the same graphs.
#pragma once

#include <cstdint>

#include "graph.hpp"

namespace ocmb {

// Every vertex gets exactly `deg` out-edges (edge i of v has id v*deg+i);
// targets uniform over [0, n), integer weights uniform in [wlo, whi].
Graph generate_uniform(std::uint32_t n, std::uint32_t deg, std::int32_t wlo, std::int32_t whi,
                       std::uint64_t seed);

} // namespace ocmb
