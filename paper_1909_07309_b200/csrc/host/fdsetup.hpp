// Host half of ExtendedFDPreconditioner::setup (/root/reference/proj/core/src/fdsolve.cpp:67-153).
// Produces every factor the device apply needs; the device never sees Eigen-shaped objects.
#pragma once

#include <vector>

#include "assembly.hpp"
#include "pencil.hpp"

namespace stiga {

struct FDFactors {
    int d = 0;
    std::vector<int> n;             // spatial sizes n_1..n_d
    int n_t = 0;
    std::vector<DenseMatrix> U;     // U_l, K_l U_l = M_l U_l Lambda_l, U_l^T M_l U_l = I
    std::vector<Vector> lambda;     // Lambda_l ascending
    TimeFactorization time;         // U_t, lambda_j (pairs), zero_count, g, sigma
    double gamma = 0.0, nu = 0.0;
    Vector S_inv;                   // inverse diagonal Schur complement, N_s (fdsolve.cpp:121-136)
    Vector d_inv_sqrt;              // D^-1/2 (N_dof) or empty (fdsolve.cpp:145-151)
    Index n_s_total = 0, n_dof = 0;
};

/// Throws std::invalid_argument / std::runtime_error exactly where the reference does.
/// `scaling` (length N_dof) may be null.
FDFactors fd_setup(const std::vector<DenseMatrix>& space_K, const std::vector<DenseMatrix>& space_M,
                   const DenseMatrix& Wt, const DenseMatrix& Mt, double gamma, double nu,
                   const double* scaling);

/// Kronecker-sum spatial eigenvalues Lambda_s, left-to-right adds (fdsolve.cpp:91-99).
Vector kron_sum_eigenvalues(const std::vector<Vector>& lambda);

} // namespace stiga
