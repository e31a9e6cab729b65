// Exception types that the C-ABI maps onto OCM_E_* codes (see include/ocm_b200.h).
#pragma once

#include <stdexcept>

namespace ocmb {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RangeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct UnsupportedError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

} // namespace ocmb
