// Host-side graph layer of the B200 optimal-cycle-mean solver.
//
// Mirrors the reference's graph vocabulary (proj/include/ocm/graph.hpp) so the
// C-ABI can stand in for its entry points: edge ids are CSR positions grouped
// by source with input order preserved (graph.hpp:7), multi-edges and
// self-loops are allowed, and integer_exact is set when every weight is an
// integer below 2^53 (graph.hpp:43). Only what the solver path needs is kept:
// the backward CSR is built on the device when a kernel needs it.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ocmb {

using Vertex = std::uint32_t;
constexpr Vertex kNoVertex = 0xffffffffu;

struct Graph {
    Vertex n = 0;
    std::uint64_t m = 0;
    std::vector<std::uint64_t> fwd_index; // n+1
    std::vector<Vertex> fwd_target;       // m
    std::vector<double> fwd_weight;       // m
    bool integer_exact = false;
};

// Parse errors carry "<source>:<line>: <message>" like the reference's
// ParseError (proj/include/ocm/graph_io.hpp:27).
class ParseError : public std::runtime_error {
  public:
    ParseError(const std::string& src, int line, const std::string& what)
        : std::runtime_error(src + ":" + std::to_string(line) + ": " + what), line_(line) {}
    int line() const { return line_; }

  private:
    int line_;
};

// A host CSR the device path uploads from: either this library's Graph
// (64-bit offsets, registered/pinned by the C-ABI) or the reference's own
// ocm::Graph arrays handed over as they are (32-bit EdgeId offsets,
// graph.hpp:21/38-41; pageable memory, staged). `validated` = the arrays
// come from build_graph (endpoints, finiteness and exactness already known);
// otherwise the device checks them before preparing.
struct HostCsr {
    Vertex n = 0;
    std::uint64_t m = 0;
    const std::uint64_t* index64 = nullptr;
    const std::uint32_t* index32 = nullptr;
    const Vertex* target = nullptr;
    const double* weight = nullptr;
    bool integer_exact = false;
    bool validated = false;
};

inline HostCsr csr_view(const Graph& g) {
    HostCsr h;
    h.n = g.n;
    h.m = g.m;
    h.index64 = g.fwd_index.data();
    h.target = g.fwd_target.data();
    h.weight = g.fwd_weight.data();
    h.integer_exact = g.integer_exact;
    h.validated = true;
    return h;
}

// proj/include/ocm/graph.hpp:76 build_graph. Throws std::invalid_argument on
// out-of-range endpoints or non-finite weights (same messages).
Graph build_graph(Vertex n, std::uint64_t m, const Vertex* src, const Vertex* dst,
                  const double* w);

// proj/include/ocm/graph_io.hpp:41 parse_graph_text / :45 read_graph_file.
Graph parse_graph_text(const char* text, std::size_t len, const std::string& source);
Graph read_graph_file(const std::string& path);

// Edge list in CSR order (fwd_source implied by fwd_index).
void graph_edges(const Graph& g, Vertex* src, Vertex* dst, double* w);

} // namespace ocmb
