// Host half of ExtendedFDPreconditioner::setup (/root/reference/proj/core/src/fdsolve.cpp:67-153).
// Produces every factor the device apply needs; the device never sees Eigen-shaped objects.
#pragma once

#include <vector>

#include "assembly.hpp"
#include "pencil.hpp"

namespace stiga {

/// Centrosymmetric split of one spatial direction (DESIGN.md §5 "Folded products"): when
/// J K_l J = K_l and J M_l J = M_l (J = exchange matrix), the eigenbasis is built as
/// U = Q blockdiag(W_e, W_o) from the two half-size pencils, so every eigenvector is exactly
/// symmetric or skew and the device applies U / U^T with half the FLOPs.  The exported U_l /
/// Lambda_l stay in ascending eigenvalue order; the device uses the folded order [even; odd].
struct FoldBasis {
    bool on = false;
    int h = 0, F = 0;                 // n = h + F, F = h + (n mod 2)
    DenseMatrix We, Wo;               // F x F, h x h (M_e / M_o-orthonormal eigenvectors)
    std::vector<int> dev_order;       // dev_order[f] = ascending index of folded position f
};

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
    std::vector<FoldBasis> fold;    // per spatial direction

    /// Device-order views: eigenvalues / eigenvectors of direction l in the order the device uses
    /// (folded order for a split direction), and S^-1 over the device order of all directions.
    Vector lambda_dev(int l) const;
    DenseMatrix U_dev(int l) const;
    Vector S_inv_dev() const;
};

/// Symmetry + centrosymmetry test: |A(i,j) - A(n-1-i,n-1-j)|, |A(i,j) - A(j,i)| <= rtol * max|A|.
bool centrosymmetric(const DenseMatrix& A, double rtol);
/// Folded matrices of a split direction, row-major zero-padded (Mp x Kp) each, stacked:
/// forward = [A_e; A_o] (applies U^T), backward = [A_p; A_q] (applies U); fold_kernels.cu.
std::vector<double> fold_matrices(const FoldBasis& fb, bool forward, int Mp, int Kp);

/// Throws std::invalid_argument / std::runtime_error exactly where the reference does.
/// `scaling` (length N_dof) may be null.  host_schur = false leaves Lambda_s / S_inv (and their
/// positivity / singularity checks) to the device setup (cuda/setup_kernels.cu): S_inv stays empty.
FDFactors fd_setup(const std::vector<DenseMatrix>& space_K, const std::vector<DenseMatrix>& space_M,
                   const DenseMatrix& Wt, const DenseMatrix& Mt, double gamma, double nu,
                   const double* scaling, bool host_schur = true);

/// Kronecker-sum spatial eigenvalues Lambda_s, left-to-right adds (fdsolve.cpp:91-99).
Vector kron_sum_eigenvalues(const std::vector<Vector>& lambda);

} // namespace stiga
