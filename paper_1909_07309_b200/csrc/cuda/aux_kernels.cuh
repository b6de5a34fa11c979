// Banded Kronecker passes (system mat-vec), GMRES vector kernels and the FP64 peak probe.
#pragma once

#include <cuda_runtime.h>

#include "fd_kernels.cuh"

namespace stiga {
namespace gpu {

/// Banded 1D factor in row band storage: band[i*(2p+1) + (j-i+p)] = F(i,j) for |i-j| <= p.
struct Band {
    const double* band = nullptr;  // device pointer, nullptr = absent
    int p = 0;
};

/// One banded mode pass over a colex tensor (geometry as ModeGeom with n == m):
///   out0 = A in0 + B in1 (+ beta0 * out0_old)      out1 = C in0 + D in1
/// Any of A..D may be absent; out1 may be null.  in1 may be null if B and D are absent.
cudaError_t launch_banded_pass(const ModeGeom& g, const double* in0, const double* in1, double* out0, double* out1,
                               Band A, Band B, Band C, Band D, double beta0, cudaStream_t st);

/// Time-banded pass on a slab of ntl time slices starting at global slice t0 (colex, N_s fastest):
/// y = A a + B b with A, B the global n_t x n_t bands; a, b hold slices [t0 - hl, ...) (the halo
/// of p slices on each side that exists).
cudaError_t launch_time_band_slab(long long Ns, int nt, long long t0, long long ntl, int hl, const double* a,
                                  const double* b, double* y, Band A, Band B, cudaStream_t st);

/// Deterministic dot product: partials (grid-sized) then a single-block finish into *d_result.
cudaError_t launch_dot(const double* x, const double* y, long long n, double* d_partials, double* d_result,
                       cudaStream_t st);
int dot_partials_size();
/// Batched dots d_out[j] = V[j] . w (j < k <= 64; deterministic two-level reduction; d_partials of
/// multidot_partials_size() doubles) and the batched update w += sum_j coefs[j] V[j] (host coefs).
int multidot_partials_size();
cudaError_t launch_multidot(const double* const* V, int k, const double* w, long long n, double* d_partials,
                            double* d_out, cudaStream_t st);
cudaError_t launch_multiaxpy(const double* coefs, const double* const* V, int k, double* w, long long n,
                             cudaStream_t st);
/// MGS step: w -= (*d_h) * v, then *d_result = dot(vn, w) (vn == nullptr: dot(w, w)); bit-identical
/// to launch_axpy(-h) followed by launch_dot.
cudaError_t launch_axpy_dot(const double* d_h, const double* v, double* w, const double* vn, long long n,
                            double* d_partials, double* d_result, cudaStream_t st);
/// y = y + alpha x
cudaError_t launch_axpy(double alpha, const double* x, double* y, long long n, cudaStream_t st);
/// y = alpha x
cudaError_t launch_scal(double alpha, const double* x, double* y, long long n, cudaStream_t st);
/// z = x - y
cudaError_t launch_sub(const double* x, const double* y, double* z, long long n, cudaStream_t st);

/// FP64 throughput probe (DMMA m8n8k4 and dependent-chain DFMA), TFLOP/s.
cudaError_t fp64_peak_probe(double ms, double* tf_dmma, double* tf_dfma);

}  // namespace gpu
}  // namespace stiga
