// Device-side synthetic graph generation: the CSR of a GenSpec is written
// straight into HBM (no host copy, no upload), bit-identical to the host
// generators in gen.cpp, then handed to the region split (prep.cu).

#include <cub/cub.cuh>

#include <functional>
#include <stdexcept>

#include "../../include/ocm_b200.h"
#include "devcommon.cuh"
#include "gen.hpp"

namespace ocmb {

void device_prepare_csr(std::uint32_t n, std::uint64_t m, DBuf<std::uint32_t>& row,
                        DBuf<std::uint32_t>& tgt, DBuf<double>& w, int exactness,
                        const ocm_solve_options& opt, DeviceState& d, PrepInfo& info,
                        cudaEvent_t w_ready = nullptr,
                        const std::function<void()>& w_host_done = nullptr);

namespace {

__device__ __forceinline__ std::uint64_t d_splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// hash2(seed, stream, i) = splitmix64(splitmix64(seed ^ stream*C) + i); the
// inner term is a per-stream constant computed on the host.
__device__ __forceinline__ std::uint64_t d_hash(std::uint64_t stream_key, std::uint64_t i) {
    return d_splitmix64(stream_key + i);
}

__global__ void kg_uniform_row(std::uint32_t n, std::uint32_t deg, std::uint32_t* row) {
    for (std::size_t v = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x; v <= n;
         v += std::size_t(gridDim.x) * blockDim.x)
        row[v] = static_cast<std::uint32_t>(v * deg);
}

__global__ void kg_powerlaw_deg(std::uint32_t n, std::uint64_t k3, std::uint32_t dmin, std::uint32_t dmax,
                                std::uint32_t* deg) {
    for (std::size_t v = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x; v <= n;
         v += std::size_t(gridDim.x) * blockDim.x) {
        if (v == n) {
            deg[v] = 0;
            continue;
        }
        const double u = double((d_hash(k3, v) >> 11) + 1) * (1.0 / 9007199254740992.0);
        const double dd = __ddiv_rn(double(dmin), __dsqrt_rn(u));
        deg[v] = dd >= double(dmax) ? dmax : static_cast<std::uint32_t>(dd);
    }
}

// hub_target (gen.hpp) with explicitly rounded multiplies
__device__ __forceinline__ std::uint32_t d_hub_target(std::uint64_t h, std::uint32_t n,
                                                      std::uint64_t mul, std::uint64_t add,
                                                      int squarings) {
    const double u = __dmul_rn(double((h >> 11) + 1), 1.0 / 9007199254740992.0);
    double f = u;
    for (int i = 0; i < squarings; ++i)
        f = __dmul_rn(f, f);
    const double x = __dmul_rn(double(n), f);
    std::uint64_t r = static_cast<std::uint64_t>(x);
    if (r >= n)
        r = n - 1;
    return static_cast<std::uint32_t>((r * mul + add) % n);
}

__global__ void kg_edges(std::uint64_t m, std::uint32_t n, std::uint64_t k1, std::uint64_t k2,
                         std::int32_t wlo, std::uint64_t span, std::uint32_t* tgt, double* w,
                         std::uint64_t hub_mul, std::uint64_t hub_add, int squarings) {
    for (std::uint64_t e = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; e < m;
         e += std::uint64_t(gridDim.x) * blockDim.x) {
        tgt[e] = squarings ? d_hub_target(d_hash(k1, e), n, hub_mul, hub_add, squarings)
                         : static_cast<std::uint32_t>(d_hash(k1, e) % n);
        w[e] = double(wlo + static_cast<std::int64_t>(d_hash(k2, e) % span));
    }
}

std::uint64_t stream_key(std::uint64_t seed, std::uint64_t stream) {
    return splitmix64(seed ^ (stream * 0xd1342543de82ef95ull));
}

} // namespace

// Generates spec's CSR on the device and runs the region split on it.
void device_generate_prepare(const GenSpec& spec, const ocm_solve_options& opt, DeviceState& d,
                             PrepInfo& info) {
    cudaStream_t s = d.stream;
    const std::uint32_t n = spec.n;
    if (n == 0 || spec.deg == 0 || spec.whi < spec.wlo || (spec.kind != 0 && spec.dmax < spec.deg))
        throw std::invalid_argument("generator: need n > 0, degree > 0, wlo <= whi (dmin <= dmax)");
    DBuf<std::uint32_t> row, tgt;
    DBuf<double> w;
    row.alloc(std::size_t(n) + 1, s);
    const int g = grid_for(std::size_t(n) + 1, d.sms);
    std::uint64_t m = 0;
    if (spec.kind == 0) {
        m = std::uint64_t(n) * spec.deg;
        if (m >= 0xffffffffull)
            throw std::invalid_argument("generate_uniform: edge count exceeds the 32-bit id space");
        kg_uniform_row<<<g, kBlock, 0, s>>>(n, spec.deg, row.p);
    } else if (spec.kind >= 1 && spec.kind <= 3) {
        DBuf<std::uint32_t> deg;
        deg.alloc(std::size_t(n) + 1, s);
        kg_powerlaw_deg<<<g, kBlock, 0, s>>>(n, stream_key(spec.seed, 3), spec.deg, spec.dmax, deg.p);
        // 64-bit total first: the 32-bit offsets must not wrap
        DBuf<unsigned long long> tot;
        tot.alloc(1, s);
        std::size_t bytes = 0;
        CK(cub::DeviceReduce::Sum(nullptr, bytes, deg.p, tot.p, std::size_t(n) + 1, s));
        DBuf<unsigned char> tmp;
        tmp.alloc(bytes, s);
        CK(cub::DeviceReduce::Sum(tmp.p, bytes, deg.p, tot.p, std::size_t(n) + 1, s));
        unsigned long long mm = 0;
        CK(cudaMemcpyAsync(&mm, tot.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (mm >= 0xffffffffull)
            throw std::invalid_argument("generate_powerlaw: edge count exceeds the 32-bit id space");
        m = mm;
        bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg.p, row.p, std::size_t(n) + 1, s));
        DBuf<unsigned char> tmp2;
        tmp2.alloc(bytes, s);
        CK(cub::DeviceScan::ExclusiveSum(tmp2.p, bytes, deg.p, row.p, std::size_t(n) + 1, s));
    } else {
        throw std::invalid_argument("unknown generator kind");
    }
    tgt.alloc(std::max<std::uint64_t>(m, 1), s);
    w.alloc(std::max<std::uint64_t>(m, 1), s);
    const std::uint64_t span = std::uint64_t(std::int64_t(spec.whi) - spec.wlo + 1);
    kg_edges<<<grid_for(m, d.sms, 32), kBlock, 0, s>>>(m, n, stream_key(spec.seed, 1),
                                                         stream_key(spec.seed, 2), spec.wlo, span,
                                                         tgt.p, w.p,
                                                         hub_mul(n), hub_add(spec.seed, n),
                                                         spec.kind == 2 ? 1 : spec.kind == 3 ? 3 : 0);
    CK(cudaGetLastError());
    device_prepare_csr(n, m, row, tgt, w, 1, opt, d, info);
}

} // namespace ocmb
