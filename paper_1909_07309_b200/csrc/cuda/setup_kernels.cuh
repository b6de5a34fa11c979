// Device half of the preconditioner setup: the O(N) pieces of
// ExtendedFDPreconditioner::setup (fdsolve.cpp:91-136, 145-151) and the geometry scaling
// D = diag(A) / diag(A~) of make_geometry_preconditioner (solver.cpp:138-142, kronop.cpp:117-131).
// Every kernel evaluates each entry with the host's operation sequence in correctly rounded
// __d*_rn arithmetic (no FMA contraction), so the results are bit-identical to the host loops.
#pragma once

#include <cuda_runtime.h>

namespace stiga {
namespace gpu {

constexpr int kSetupMaxDim = 4;

/// Per-pair constants of the Schur diagonal, computed on the host exactly as fdsolve.cpp:114-129
/// writes them: c = gamma^2/nu lambda_j^2, c1sq = (gamma/nu lambda_j)^2 / nu, ga2 = g_a^2, gb2 = g_b^2.
struct SchurArgs {
    int d = 0;
    int n[kSetupMaxDim] = {0, 0, 0, 0};
    const double* lam[kSetupMaxDim] = {};  // per-direction eigenvalues in the device (fiber) order
    int npairs = 0;
    const double* pc = nullptr;    // npairs x 4: c, c1sq, ga2, gb2
    double gs = 0.0;               // gamma * sigma
    double nu = 0.0, gg = 0.0;     // nu, gamma * gamma
    double cz = 0.0;               // zero block: gamma^2 g_z^2 / nu (0 without a zero block)
    int zero_block = 0;
};

/// S^-1 over the spatial index in the device order; *flag |= 1 for a non-positive Lambda_s entry,
/// |= 2 for a zero Schur entry (the reference's runtime_errors, fdsolve.cpp:100-102, 134-135).
cudaError_t launch_schur_inv(const SchurArgs& a, long long Ns, double* S_inv, int* flag, cudaStream_t st);

/// out = 1 / sqrt(D); *flag |= 1 for a non-positive entry (fdsolve.cpp:145-151).
cudaError_t launch_dinv_sqrt(const double* D, double* out, long long n, int* flag, cudaStream_t st);

/// diag of a Kronecker-sum operator: out[i] = sum_t c_t prod_l diag_{t,l}[i_l] (kronop.cpp:117-131,
/// product built first factor first, terms accumulated in order).  diags: nterms x D device pointers
/// (host array), dims: D sizes (first fastest).  With `num` set the kernel writes out[i] = num[i] / diag[i]
/// instead (D = diag(A) / diag(A~); num may alias out).
cudaError_t launch_kron_diag(int D, const int* dims, int nterms, const double* coeffs, const double* const* diags,
                             const double* num, double* out, long long n, cudaStream_t st);

/// Physical system diagonal diag(M_s) (x) diag(W_t) + diag(K_s) (x) diag(M_t) (solver.cpp:67-70):
/// out[t Ns + i] = dM[i] W[t] + dK[i] M[t]; with `den` set, out = (that) / den.
cudaError_t launch_physical_diag(const double* dM, const double* dK, const double* W, const double* M, long long Ns,
                                 int nt, const double* den, double* out, cudaStream_t st);

}  // namespace gpu
}  // namespace stiga
