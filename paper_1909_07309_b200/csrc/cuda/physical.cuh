// Physical (geometry-mapped) spatial stiffness / mass on the device, stored in a tensor "stencil"
// format, and the space-time system mat-vec y = M_s X W_t^T + K_s X M_t^T built on them.
//
// Replaces SpaceTimeSystem's A_ (solver.cpp:58-70 with assemble_spatial_physical,
// assembly.cpp:151-268): the reference assembles K_s, M_s through Eigen triplets (~131 GB at config 4);
// here one CTA per element computes the (p+1)^d x (p+1)^d local matrices by Gauss quadrature with the
// spline geometry evaluated in-kernel, and adds them into per-row arrays of the (2p+1)^d possible
// neighbours (the tensor B-spline sparsity pattern), so A x is a stencil SpMM over all time slices.
#pragma once

#include <cuda_runtime.h>

#include "aux_kernels.cuh"

namespace stiga {
namespace gpu {

/// Analytic coefficient fields of the problem catalog (geometry.hpp make_problem), evaluated on the
/// device at physical points.
enum FieldKind : int { kFieldOne = 0, kFieldSeparableNu = 1, kFieldDeformedKappa = 2, kFieldDeformedC = 3 };

struct PhysicalDesc {
    int d = 0;
    int p = 0, q = 0;              // spline degree and Gauss points per element (q = p+1)
    int n_el = 0;                  // elements per direction (uniform open knots)
    int n = 0;                     // active functions per direction (both ends dropped)
    // geometry: uniform open knot vectors of degree pg with neg elements per direction, control
    // points (prod(neg+pg) x d, column-major) on the device
    int pg = 1, neg = 1;
    const double* cp = nullptr;
    long long ncp = 0;
    int nu_kind = kFieldOne, gamma_kind = kFieldOne;
    // per direction 1D tables (same in every direction): Gauss nodes / weights of all elements
    // (n_el*q), active-basis values / derivatives (n_el*q x (p+1)) and the first active index
    const double* qnode = nullptr;
    const double* qweight = nullptr;
    const double* bval = nullptr;
    const double* bder = nullptr;
    const int* bfirst = nullptr;
};

/// Stencil-format assembly: Kst / Mst hold (2p+1)^d offset planes of N_s doubles (zeroed by the
/// caller); entry [o][i] couples row i with the neighbour at offset o = sum_l (j_l - i_l + p)(2p+1)^l.
cudaError_t launch_physical_assembly(const PhysicalDesc& desc, double* Kst, double* Mst, cudaStream_t st);

/// MX = M_s X and KX = K_s X, X / MX / KX (N_s x n_t) colex (space fastest), on the FP64 tensor cores.
cudaError_t launch_stencil_apply2(const PhysicalDesc& desc, const double* Mst, const double* Kst, const double* X,
                                  double* MX, double* KX, long long n_t, cudaStream_t st);

/// Diagonal entries of the two stencils (the centre offset), N_s each.
cudaError_t launch_stencil_diag(const PhysicalDesc& desc, const double* Kst, const double* Mst, double* dK, double* dM,
                                cudaStream_t st);

}  // namespace gpu
}  // namespace stiga
