// Time-fused kernel with the peer-memory scatter epilogue (fused all-to-all back to the time
// slabs); a separate translation unit only for parallel compilation.
#include "fd_time_impl.cuh"

namespace stiga {
namespace gpu {

cudaError_t dispatch_time_scatter(const Tiling& t, const ModeGeom& g, const double* X, const double* Jt,
                                  const double* J, const ArrowParams& ap, cudaStream_t st, int* occ,
                                  const Scatter* sc) {
    return dispatch_time_v<true>(t, g, X, nullptr, Jt, J, ap, st, occ, sc);
}

}  // namespace gpu
}  // namespace stiga
