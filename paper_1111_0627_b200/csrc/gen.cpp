#include "gen.hpp"

#include <stdexcept>
#include <thread>
#include <vector>

namespace ocmb {

namespace {

inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

inline std::uint64_t hash2(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) {
    return splitmix64(splitmix64(seed ^ (stream * 0xd1342543de82ef95ull)) + i);
}

} // namespace

Graph generate_uniform(std::uint32_t n, std::uint32_t deg, std::int32_t wlo, std::int32_t whi,
                       std::uint64_t seed) {
    if (n == 0 || deg == 0 || whi < wlo)
        throw std::invalid_argument("generate_uniform: need n > 0, deg > 0, wlo <= whi");
    const std::uint64_t m = std::uint64_t(n) * deg;
    if (m >= 0xffffffffull)
        throw std::invalid_argument("generate_uniform: edge count exceeds the 32-bit id space");
    Graph g;
    g.n = n;
    g.m = m;
    g.integer_exact = true;
    g.fwd_index.resize(std::size_t(n) + 1);
    g.fwd_target.resize(m);
    g.fwd_weight.resize(m);
    const std::uint64_t span = std::uint64_t(std::int64_t(whi) - wlo + 1);
    unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            const std::uint64_t lo = m * t / T, hi = m * (t + 1) / T;
            for (std::uint64_t e = lo; e < hi; ++e) {
                g.fwd_target[e] = static_cast<Vertex>(hash2(seed, 1, e) % n);
                g.fwd_weight[e] = double(wlo + std::int64_t(hash2(seed, 2, e) % span));
            }
        });
    for (auto& th : pool)
        th.join();
    for (std::uint32_t v = 0; v <= n; ++v)
        g.fwd_index[v] = std::uint64_t(v) * deg;
    return g;
}

} // namespace ocmb
