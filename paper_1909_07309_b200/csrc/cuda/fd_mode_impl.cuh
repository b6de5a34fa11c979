// Dense mode-product kernel template and its launch dispatch (instantiated per variant in
// fd_mode.cu: plain and D^-1/2 pre-scaled; fd_mode_sc.cu: peer-memory scatter epilogue).
#pragma once
#include "fd_common.cuh"

namespace stiga {
namespace gpu {
namespace {

// PS: Y = (I (x) J (x) I)(pre .* X) -- the D^-1/2 pre-scale of the apply fused into the first forward
// mode product: each fiber chunk's D^-1/2 chunk is staged beside it by the same cp.async pattern
// and B fragments are scaled as they are read (two DMULs per k-step on the FP64 pipe, against the
// separate 24 B/DoF HBM pass of scale_kernel).
template <int MI, int WN, bool PS, bool SC, int WM = 1>
__global__ void __launch_bounds__(32 * WM * WN)
    mode_product_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                        const double* __restrict__ post, const double* __restrict__ pre, const __grid_constant__ Scatter sc) {
    using SH = Shape<MI, WM, WN, PS>;
    extern __shared__ __align__(16) double smem[];
    const int rb = blockIdx.x % a.RB;  // row blocks of one fiber tile are adjacent -> X tile reused from L2
    const long long c0 = static_cast<long long>(blockIdx.x / a.RB) * SH::BN;
    const double* Jg = J + static_cast<size_t>(rb) * SH::MPB * a.Kp;
    Prod p = make_prod<SH>(a, c0, X, Jg);
    if constexpr (PS) p.dg = pre + (p.xg - X);
    double acc[SH::MI][SH::NI][2];
    zero_acc<SH>(acc);
    gemm<SH, true>(a, smem, p, X, nullptr, false, rb * MI * WM, acc);
    if constexpr (SC) store_acc_scatter<SH>(a, acc, c0, rb * MI * WM, sc);
    else store_acc<SH>(a, acc, c0, rb * MI * WM, Y, post);
}


template <int MI, int WN, bool PS, bool SC, int WM = 1>
cudaError_t launch_mode_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, cudaStream_t st, int* occ, const Scatter* sc) {
    auto k = mode_product_kernel<MI, WN, PS, SC, WM>;
    const size_t smem = PS ? prescale_smem(t) : t.smem;
    if (occ) {
        *occ = occupancy(k, 32 * WM * WN, smem);
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN * t.RB;
    k<<<static_cast<unsigned>(blocks), 32 * WM * WN, smem, st>>>(make_args(t, g), X, Y, J, post, pre,
                                                                 sc ? *sc : Scatter{});
    return cudaGetLastError();
}

template <bool PS, bool SC, int WN>
cudaError_t dispatch_mode_wn(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                             const double* post, const double* pre, cudaStream_t st, int* occ, const Scatter* sc) {
#define STIGA_CALL_MODE(M) launch_mode_t<M, WN, PS, SC>(t, g, X, Y, J, post, pre, st, occ, sc)
    STIGA_MI_SWITCH(t.MI, STIGA_CALL_MODE)
#undef STIGA_CALL_MODE
}

// WM = 2 (two warp rows over the row block, one fiber tile): plain products only (no pre-scale, no
// scatter epilogue), MI <= 8.
template <int WN>
cudaError_t dispatch_mode_wm2(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                              const double* post, cudaStream_t st, int* occ) {
    switch (t.MI) {
        case 1: return launch_mode_t<1, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        case 2: return launch_mode_t<2, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        case 3: return launch_mode_t<3, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        case 4: return launch_mode_t<4, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        case 5: return launch_mode_t<5, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        case 6: return launch_mode_t<6, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        case 7: return launch_mode_t<7, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        case 8: return launch_mode_t<8, WN, false, false, 2>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
        default: return cudaErrorInvalidValue;
    }
}

template <bool PS, bool SC>
cudaError_t dispatch_mode_v(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                            const double* post, const double* pre, cudaStream_t st, int* occ, const Scatter* sc) {
    if constexpr (!PS && !SC) {
        if (t.WM == 2) {
            if (t.WN == 4) return dispatch_mode_wm2<4>(t, g, X, Y, J, post, st, occ);
            if (t.WN == 2) return dispatch_mode_wm2<2>(t, g, X, Y, J, post, st, occ);
            return cudaErrorInvalidValue;
        }
    }
    if (t.WM != 1) return cudaErrorInvalidValue;
    if (t.WN == 4) return dispatch_mode_wn<PS, SC, 4>(t, g, X, Y, J, post, pre, st, occ, sc);
    if (t.WN == 2) return dispatch_mode_wn<PS, SC, 2>(t, g, X, Y, J, post, pre, st, occ, sc);
    return cudaErrorInvalidValue;
}

}  // namespace
}  // namespace gpu
}  // namespace stiga
