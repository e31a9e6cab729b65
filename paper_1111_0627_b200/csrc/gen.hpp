// Seeded synthetic graph generators (benchmark workloads). The counter hash
// is bit-identical to oracle/ocm_oracle.c so checkers see the same graphs.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#include "graph.hpp"

namespace ocmb {

// Every vertex gets exactly `deg` out-edges (edge i of v has id v*deg+i);
// targets uniform over [0, n), integer weights uniform in [wlo, whi].
Graph generate_uniform(std::uint32_t n, std::uint32_t deg, std::int32_t wlo, std::int32_t whi,
                       std::uint64_t seed);

// Power-law out-degrees: deg(v) = min(dmax, floor(dmin / sqrt(u_v))), u_v
// uniform in (0, 1] -- P(deg > d) = (dmin/d)^2, the tail exponent 3 of
// preferential attachment -- with targets uniform over [0, n) and integer
// weights uniform in [wlo, whi]. Only IEEE-exact operations (sqrt, divide)
// touch floating point, so host and device generate identical graphs.
Graph generate_powerlaw(std::uint32_t n, std::uint32_t dmin, std::uint32_t dmax, std::int32_t wlo,
                        std::int32_t whi, std::uint64_t seed);

// Power-law in- and out-degrees ("hub" graphs): out-degrees as
// generate_powerlaw; the target of edge e is x = floor(n * u^2) (u uniform
// in (0, 1]) scattered over the vertex ids by the bijection
// x -> (x * A + B) mod n, so vertex rank r receives in-degree ~ r^(-1/2):
// P(in-degree > d) ~ d^(-2), the same tail exponent 3 as the out-degrees,
// with the hubs spread across the id space (not the low ids). Exactly
// rounded double multiplies only, so host and device agree bit for bit.
Graph generate_powerlaw_hubs(std::uint32_t n, std::uint32_t dmin, std::uint32_t dmax,
                             std::int32_t wlo, std::int32_t whi, std::uint64_t seed);
// The same with targets floor(n * u^8): in-degree tail P(in > d) ~ d^(-8/7),
// density exponent ~2.14 -- the web graphs' in-degree law; a few hundred
// hubs receive a quarter of the edges ("powerlaw-web").
Graph generate_powerlaw_web(std::uint32_t n, std::uint32_t dmin, std::uint32_t dmax,
                            std::int32_t wlo, std::int32_t whi, std::uint64_t seed);

// Generator description shared by the host generators and the device ones
// (gen_dev.cu) that write the CSR straight into HBM.
struct GenSpec {
    int kind = 0; // 0 uniform, 1 power-law out-degree, 2 + hub in-degrees (u^2), 3 web-like (u^8)
    std::uint32_t n = 0;
    std::uint32_t deg = 8; // uniform: out-degree; power-law: dmin
    std::uint32_t dmax = 0; // power-law cap
    std::int32_t wlo = 1, whi = 100;
    std::uint64_t seed = 1;
};

Graph generate(const GenSpec& g);

// Shared counter hash (bit-identical to oracle/ocm_oracle.c and gen_dev.cu).
inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline std::uint64_t hash2(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) {
    return splitmix64(splitmix64(seed ^ (stream * 0xd1342543de82ef95ull)) + i);
}
// deg(v) of the power-law generator.
inline std::uint32_t powerlaw_degree(std::uint64_t seed, std::uint32_t v, std::uint32_t dmin,
                                     std::uint32_t dmax) {
    const double u = double((hash2(seed, 3, v) >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double d = double(dmin) / std::sqrt(u);
    return d >= double(dmax) ? dmax : static_cast<std::uint32_t>(d);
}

// Target scatter of generate_powerlaw_hubs: multiplier and offset of the
// bijection x -> (x * A + B) mod n.
constexpr std::uint64_t kHubMul = 2654435761ull; // prime, so coprime to every n != it
inline std::uint64_t hub_mul(std::uint32_t n) { return n % kHubMul == 0 ? 1 : kHubMul % n; }
inline std::uint64_t hub_add(std::uint64_t seed, std::uint32_t n) { return hash2(seed, 4, 0) % n; }
inline std::uint32_t hub_target(std::uint64_t h, std::uint32_t n, std::uint64_t mul,
                                std::uint64_t add, int squarings = 1) {
    const double u = double((h >> 11) + 1) * (1.0 / 9007199254740992.0);
    double f = u;
    for (int i = 0; i < squarings; ++i)
        f = f * f;
    double x = double(n) * f;
    std::uint64_t r = static_cast<std::uint64_t>(x);
    if (r >= n)
        r = n - 1;
    return static_cast<std::uint32_t>((r * mul + add) % n);
}

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
