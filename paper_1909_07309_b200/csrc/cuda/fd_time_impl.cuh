// Time-fused kernel template (U_t^T -> block-arrowhead solve -> U_t per spatial-index tile) and
// its launch dispatch (fd_time.cu: plain epilogue; fd_time_sc.cu: peer-memory scatter epilogue).
#pragma once
#include "fd_common.cuh"

namespace stiga {
namespace gpu {
namespace {

template <int MI, int WM, int WN, bool SC>
__global__ void __launch_bounds__(32 * WM * WN)
    time_fused_kernel(KArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ Jt,
                      const double* __restrict__ J, ArrowParams ap, const __grid_constant__ Scatter sc) {
    using SH = Shape<MI, WM, WN>;
    extern __shared__ __align__(16) double smem[];
    double* Zs = smem;                                               // Zrows x LDX, resident
    double* stages = smem + static_cast<size_t>(a.Zrows) * SH::LDX;  // nstage x stage
    double* cs = stages + static_cast<size_t>(a.nstage) * SH::STAGE;    // 7 x (n_t/2 + 1) pair constants
    double* ccol = cs + 7 * arrow_np(ap);                               // 3 x BN column constants
    double* red = ccol + 3 * SH::BN;                                    // WM = 3 only: 6 x BN Schur partial sums
    const long long c0 = static_cast<long long>(blockIdx.x) * SH::BN;
    stage_arrow_consts(ap, cs);  // visible after the GEMM's first barrier
    stage_column_consts(ap, c0, a.geo.ncols, SH::BN, ccol);
    Prod p = make_prod<SH>(a, c0, X, Jt);
    double acc[SH::MI][SH::NI][2];
    zero_acc<SH>(acc);
    gemm<SH, true>(a, stages, p, X, nullptr, false, 0, acc);  // Z = U_t^T x
    // Z -> smem (rows < Kp; padded rows are exact zeros because the padded J rows are zero)
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int wm = warp % WM, wn = warp / WM;
        const int g = lane >> 2, t = lane & 3;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
            const int row = (wm * MI + mi) * 8 + g;
            if (row < a.Zrows) {
#pragma unroll
                for (int ni = 0; ni < SH::NI; ++ni) {
                    const int col = (wn * SH::NI + ni) * 8 + 2 * t;
                    Zs[row * SH::LDX + col] = acc[mi][ni][0];
                    Zs[row * SH::LDX + col + 1] = acc[mi][ni][1];
                }
            }
        }
    }
    __syncthreads();  // Z visible; every warp is done with the GEMM-1 stages
    // U_t chunks stream in while the arrowhead runs
    p.jg = J + (p.jg - Jt);
    {
        const int nchunks = (a.Kp + kBK - 1) / kBK;
        const unsigned st0 = smem_u32(stages);
        for (int s = 0; s < a.nstage - 1; ++s) {
            if (s < nchunks) issue_chunk<SH>(a, p, st0 + 8u * s * SH::STAGE, s, false, X);
            cp_commit();
        }
    }
    if (!(ap.debug & 1)) arrowhead_tile<SH>(a, Zs, c0, ap, cs, ccol, red);
    __syncthreads();
    zero_acc<SH>(acc);
    gemm<SH, false>(a, stages, p, X, Zs, true, 0, acc);  // y = U_t z
    if constexpr (SC) store_acc_scatter<SH>(a, acc, c0, 0, sc);
    else store_acc<SH>(a, acc, c0, 0, Y, nullptr);
}


template <int MI, int WM, int WN, bool SC>
cudaError_t launch_time_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                          const double* J, const ArrowParams& ap, cudaStream_t st, int* occ, const Scatter* sc) {
    auto k = time_fused_kernel<MI, WM, WN, SC>;
    if (occ) {
        *occ = occupancy(k, 32 * WM * WN, t.smem);
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem));
    if (e != cudaSuccess) return e;
    const long long blocks = (g.ncols + t.BN - 1) / t.BN;
    k<<<static_cast<unsigned>(blocks), 32 * WM * WN, t.smem, st>>>(make_args(t, g), X, Y, Jt, J, ap,
                                                                     sc ? *sc : Scatter{});
    return cudaGetLastError();
}

template <bool SC, int WM, int WN>
cudaError_t dispatch_time_w(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                            const double* J, const ArrowParams& ap, cudaStream_t st, int* occ, const Scatter* sc) {
#define STIGA_CALL_TIME(M) launch_time_t<M, WM, WN, SC>(t, g, X, Y, Jt, J, ap, st, occ, sc)
    STIGA_MI_SWITCH(t.MI, STIGA_CALL_TIME)
#undef STIGA_CALL_TIME
}

template <bool SC>
cudaError_t dispatch_time_v(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                            const double* J, const ArrowParams& ap, cudaStream_t st, int* occ, const Scatter* sc) {
    if (t.WN == 2) {
        if (t.WM == 1) return dispatch_time_w<SC, 1, 2>(t, g, X, Y, Jt, J, ap, st, occ, sc);
        if (t.WM == 2) return dispatch_time_w<SC, 2, 2>(t, g, X, Y, Jt, J, ap, st, occ, sc);
        if (t.WM == 3) return dispatch_time_w<SC, 3, 2>(t, g, X, Y, Jt, J, ap, st, occ, sc);
        if (t.WM == 4) return dispatch_time_w<SC, 4, 2>(t, g, X, Y, Jt, J, ap, st, occ, sc);
    } else if (t.WN == 4) {
        if (t.WM == 1) return dispatch_time_w<SC, 1, 4>(t, g, X, Y, Jt, J, ap, st, occ, sc);
        if (t.WM == 2) return dispatch_time_w<SC, 2, 4>(t, g, X, Y, Jt, J, ap, st, occ, sc);
        if (t.WM == 3) return dispatch_time_w<SC, 3, 4>(t, g, X, Y, Jt, J, ap, st, occ, sc);
    }
    return cudaErrorInvalidValue;
}

}  // namespace
}  // namespace gpu
}  // namespace stiga
