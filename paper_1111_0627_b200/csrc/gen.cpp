#include "gen.hpp"

#include <cmath>
#include <algorithm>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace ocmb {

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

namespace {

Graph powerlaw_graph(std::uint32_t n, std::uint32_t dmin, std::uint32_t dmax, std::int32_t wlo,
                     std::int32_t whi, std::uint64_t seed, int hubs) {
    if (n == 0 || dmin == 0 || dmax < dmin || whi < wlo)
        throw std::invalid_argument("generate_powerlaw: need n > 0, 0 < dmin <= dmax, wlo <= whi");
    Graph g;
    g.n = n;
    g.integer_exact = true;
    g.fwd_index.resize(std::size_t(n) + 1);
    g.fwd_index[0] = 0;
    for (std::uint32_t v = 0; v < n; ++v)
        g.fwd_index[v + 1] = g.fwd_index[v] + powerlaw_degree(seed, v, dmin, dmax);
    const std::uint64_t m = g.fwd_index[n];
    if (m >= 0xffffffffull)
        throw std::invalid_argument("generate_powerlaw: edge count exceeds the 32-bit id space");
    g.m = m;
    g.fwd_target.resize(m);
    g.fwd_weight.resize(m);
    const std::uint64_t span = std::uint64_t(std::int64_t(whi) - wlo + 1);
    const std::uint64_t mul = hub_mul(n), add = hub_add(seed, n);
    unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            const std::uint64_t lo = m * t / T, hi = m * (t + 1) / T;
            for (std::uint64_t e = lo; e < hi; ++e) {
                g.fwd_target[e] = hubs ? hub_target(hash2(seed, 1, e), n, mul, add, hubs)
                                       : static_cast<Vertex>(hash2(seed, 1, e) % n);
                g.fwd_weight[e] = double(wlo + std::int64_t(hash2(seed, 2, e) % span));
            }
        });
    for (auto& th : pool)
        th.join();
    return g;
}

} // namespace

Graph generate_powerlaw(std::uint32_t n, std::uint32_t dmin, std::uint32_t dmax, std::int32_t wlo,
                        std::int32_t whi, std::uint64_t seed) {
    return powerlaw_graph(n, dmin, dmax, wlo, whi, seed, 0);
}

Graph generate_powerlaw_hubs(std::uint32_t n, std::uint32_t dmin, std::uint32_t dmax,
                             std::int32_t wlo, std::int32_t whi, std::uint64_t seed) {
    return powerlaw_graph(n, dmin, dmax, wlo, whi, seed, 1);
}

Graph generate_powerlaw_web(std::uint32_t n, std::uint32_t dmin, std::uint32_t dmax,
                            std::int32_t wlo, std::int32_t whi, std::uint64_t seed) {
    return powerlaw_graph(n, dmin, dmax, wlo, whi, seed, 3);
}

Graph generate(const GenSpec& s) {
    if (s.kind == 0)
        return generate_uniform(s.n, s.deg, s.wlo, s.whi, s.seed);
    if (s.kind == 1)
        return generate_powerlaw(s.n, s.deg, s.dmax, s.wlo, s.whi, s.seed);
    if (s.kind == 2)
        return generate_powerlaw_hubs(s.n, s.deg, s.dmax, s.wlo, s.whi, s.seed);
    if (s.kind == 3)
        return generate_powerlaw_web(s.n, s.deg, s.dmax, s.wlo, s.whi, s.seed);
    throw std::invalid_argument("unknown generator kind");
}

} // namespace ocmb

namespace ocmb {

namespace {

// Open-addressing map from packed composite state to vertex id.
class StateIndex {
  public:
    explicit StateIndex(std::size_t hint) { rehash(std::max<std::size_t>(1024, hint * 2)); }
    // returns (id, inserted)
    std::pair<std::uint32_t, bool> intern(std::uint64_t key, std::uint32_t fresh_id) {
        if ((size_ + 1) * 2 > cap_)
            rehash(cap_ * 2);
        std::size_t h = mix(key) & (cap_ - 1);
        for (;;) {
            if (ids_[h] == kEmpty) {
                keys_[h] = key;
                ids_[h] = fresh_id;
                ++size_;
                return {fresh_id, true};
            }
            if (keys_[h] == key)
                return {ids_[h], false};
            h = (h + 1) & (cap_ - 1);
        }
    }

  private:
    static constexpr std::uint32_t kEmpty = 0xffffffffu;
    static std::size_t mix(std::uint64_t x) {
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdull;
        x ^= x >> 33;
        return static_cast<std::size_t>(x);
    }
    void rehash(std::size_t cap) {
        std::vector<std::uint64_t> ok = std::move(keys_);
        std::vector<std::uint32_t> oi = std::move(ids_);
        cap_ = 1;
        while (cap_ < cap)
            cap_ <<= 1;
        keys_.assign(cap_, 0);
        ids_.assign(cap_, kEmpty);
        size_ = 0;
        for (std::size_t i = 0; i < oi.size(); ++i)
            if (oi[i] != kEmpty)
                intern(ok[i], oi[i]);
    }
    std::vector<std::uint64_t> keys_;
    std::vector<std::uint32_t> ids_;
    std::size_t cap_ = 0, size_ = 0;
};

std::uint32_t bits_for(std::uint64_t values) {
    std::uint32_t b = 0;
    while (b < 64 && (std::uint64_t(1) << b) < values)
        ++b;
    return b;
}

} // namespace

Graph generate_model(const Scenario& sc, std::uint32_t clients, std::uint64_t max_states) {
    if (sc.states == 0 || clients == 0)
        throw std::invalid_argument("model needs at least one state and one client");
    for (const auto& t : sc.transitions) {
        if (t.from >= sc.states || t.to >= sc.states)
            throw std::invalid_argument("scenario transition references a missing state");
        if ((t.acquires || t.releases) && !sc.uses_server)
            throw std::invalid_argument("server transition in a server-free scenario");
    }
    const std::uint32_t cb = std::max(bits_for(sc.states), 1u);
    const std::uint32_t ob = sc.uses_server ? bits_for(std::uint64_t(clients) + 1) : 0;
    if (std::uint64_t(cb) * clients + ob > 64)
        throw std::invalid_argument("composite state does not fit in 64 bits");
    const std::uint64_t cmask = (std::uint64_t(1) << cb) - 1;
    const std::uint64_t oshift = std::uint64_t(clients) * cb;
    const std::uint64_t omask = ob ? (((std::uint64_t(1) << ob) - 1) << oshift) : 0;
    const std::uint64_t cap = std::min<std::uint64_t>(max_states, 0xfffffffeull);

    // transitions grouped by source local state, declaration order kept
    std::vector<std::vector<ScenarioTransition>> by_from(sc.states);
    for (const auto& t : sc.transitions)
        by_from[t.from].push_back(t);

    Graph g;
    g.integer_exact = true;
    std::vector<std::uint64_t> state; // id -> packed state (the BFS queue)
    StateIndex index(1 << 16);
    state.push_back(0); // all clients in state 0, server free
    index.intern(0, 0);
    g.fwd_index.push_back(0);
    bool exact = true;
    for (std::size_t u = 0; u < state.size(); ++u) {
        const std::uint64_t s = state[u];
        const std::uint64_t owner = ob ? (s & omask) >> oshift : 0;
        for (std::uint32_t i = 0; i < clients; ++i) {
            const std::uint64_t shift = std::uint64_t(i) * cb;
            const std::uint32_t loc = static_cast<std::uint32_t>((s >> shift) & cmask);
            for (const auto& t : by_from[loc]) {
                if (t.acquires && owner != 0)
                    continue;
                if (t.releases && owner != i + 1)
                    continue;
                std::uint64_t ns = (s & ~(cmask << shift)) | (std::uint64_t(t.to) << shift);
                if (t.acquires)
                    ns = (ns & ~omask) | (std::uint64_t(i + 1) << oshift);
                if (t.releases)
                    ns &= ~omask;
                const auto [id, fresh] = index.intern(ns, static_cast<std::uint32_t>(state.size()));
                if (fresh) {
                    if (state.size() + 1 > cap)
                        throw std::length_error("state space exceeds " + std::to_string(max_states) +
                                                " states");
                    state.push_back(ns);
                }
                g.fwd_target.push_back(id);
                const double w = static_cast<double>(t.cost);
                exact = exact && static_cast<std::int64_t>(w) == t.cost &&
                        std::fabs(w) < 9007199254740992.0;
                g.fwd_weight.push_back(w);
            }
        }
        g.fwd_index.push_back(g.fwd_target.size());
    }
    g.n = static_cast<Vertex>(state.size());
    g.m = g.fwd_target.size();
    g.integer_exact = exact;
    return g;
}

} // namespace ocmb
