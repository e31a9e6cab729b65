// Summary of the device-side region split, shared by host and device code.
#pragma once

#include <cstdint>

namespace ocmb {

// Summary of the device-side region split (prep.cu).
struct PrepInfo {
    std::uint32_t n = 0;            // vertices (device arrays are indexed by original id)
    std::uint32_t R = 0;            // non-trivial regions; trivial vertices carry region R
    std::uint32_t regions_total = 0;
    std::uint32_t trivial = 0;
    std::uint64_t M = 0;            // intra-region edges
    std::uint32_t max_region = 0;
    bool exact = false;
    bool wide = false;              // exact lane with 128-bit keys and 64-bit weights
    bool scc_off = false;
    double no_cycle_above = 0.0;
    long long max_abs_w = 0;
    std::uint64_t h2d_bytes = 0;
    double scc_ms = 0.0;
};

} // namespace ocmb
