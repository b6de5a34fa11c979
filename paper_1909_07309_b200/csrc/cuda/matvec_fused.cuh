// Fused sum-factorized space-time system mat-vec kernels (matvec_fused.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace stiga {
namespace gpu {

constexpr int kMaxFusedP = 6;  // half-bandwidth limit of the fused kernels (p <= 6)

/// Modes 0 and 1 of the colex tensor (n0, n1, R): a2 = (M1 (x) M0) x, b2 = (K1 (x) M0 + M1 (x) K0) x
/// (mode 1 applied first; distinct-mode Kronecker factors commute).
/// m0/k0 (n0 rows) and m1/k1 (n1 rows): row band storage widened to 2P+1 taps.
cudaError_t launch_plane2(int n0, int n1, long long R, int P, const double* x, double* a2, double* b2,
                          const double* m0, const double* k0, const double* m1, const double* k1, cudaStream_t st);
size_t plane2_smem_bytes(int n0, int P);

/// Time pass (mode2 = false: fields (Lc, T)) or mode 2 + time pass (mode2 = true: fields (Lc, n2, T)):
///   [a3 = M2 a, b3 = K2 a + M2 b]   y(t) = sum_t' cw(t')[t - t' + P] a3(t') + cm(t')[t - t' + P] b3(t')
/// a, b hold the global time slices [ti0, ti0 + nti), y the slices [to0, to0 + nto) (inside the input
/// range); cw / cm are the band COLUMNS (nt x (2P+1)) of gamma W_t and nu M_t.
cudaError_t launch_stream(bool mode2, long long Lc, int n2, int nt, int ti0, int nti, int to0, int nto, int P,
                          const double* a, const double* b, double* y, const double* m2, const double* k2,
                          const double* cw, const double* cm, cudaStream_t st);

}  // namespace gpu
}  // namespace stiga
