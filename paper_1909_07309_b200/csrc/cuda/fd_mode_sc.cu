// Dense mode products with the peer-memory scatter epilogue (the fused all-to-all of the
// time-sharded apply); a separate translation unit only for parallel compilation.
#include "fd_mode_impl.cuh"

namespace stiga {
namespace gpu {

cudaError_t dispatch_mode_scatter(const Tiling& t, const ModeGeom& g, const double* X, const double* J,
                                  cudaStream_t st, int* occ, const Scatter* sc) {
    return dispatch_mode_v<false, true>(t, g, X, nullptr, J, nullptr, nullptr, st, occ, sc);
}

}  // namespace gpu
}  // namespace stiga
