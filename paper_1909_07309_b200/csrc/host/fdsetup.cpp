// Host half of the extended-FD setup; follows /root/reference/proj/core/src/fdsolve.cpp:67-153.
#include "fdsetup.hpp"

#include <cmath>
#include <stdexcept>

namespace stiga {

Vector kron_sum_eigenvalues(const std::vector<Vector>& lambda) {
    Vector lam_s(1, 0.0);
    for (const Vector& lam_l : lambda) {
        Vector next(lam_s.size() * lam_l.size());
        for (size_t j = 0; j < lam_l.size(); ++j)
            for (size_t i = 0; i < lam_s.size(); ++i) next[j * lam_s.size() + i] = lam_s[i] + lam_l[j];
        lam_s.swap(next);
    }
    return lam_s;
}

FDFactors fd_setup(const std::vector<DenseMatrix>& space_K, const std::vector<DenseMatrix>& space_M,
                   const DenseMatrix& Wt, const DenseMatrix& Mt, double gamma, double nu,
                   const double* scaling) {
    if (gamma <= 0.0) throw std::invalid_argument("ExtendedFDPreconditioner: gamma must be positive");
    if (nu <= 0.0) throw std::invalid_argument("ExtendedFDPreconditioner: nu must be positive");
    if (space_K.size() != space_M.size() || space_K.empty())
        throw std::invalid_argument("ExtendedFDPreconditioner: per-direction matrices mismatch");
    FDFactors F;
    F.d = static_cast<int>(space_K.size());
    Index n_s = 1;
    for (int l = 0; l < F.d; ++l) {
        DenseMatrix U;
        Vector lam;
        spd_generalized_eig(space_K[l], space_M[l], U, lam);
        F.n.push_back(static_cast<int>(lam.size()));
        F.U.push_back(std::move(U));
        F.lambda.push_back(std::move(lam));
        n_s *= F.n.back();
    }
    F.time = time_factorization(Wt, Mt);
    F.n_t = static_cast<int>(F.time.size());
    F.n_s_total = n_s;
    F.n_dof = n_s * F.n_t;
    F.gamma = gamma;
    F.nu = nu;

    const Vector lam_s = kron_sum_eigenvalues(F.lambda);
    for (double v : lam_s)
        if (v <= 0.0)
            throw std::runtime_error("ExtendedFDPreconditioner: spatial eigenvalues not positive "
                                     "(stiffness pencil not positive definite)");
    Vector lam_inv(lam_s.size());
    for (size_t s = 0; s < lam_s.size(); ++s) lam_inv[s] = 1.0 / lam_s[s];

    // S = gamma sigma + nu Lambda_s + sum_j gamma^2 (g_a^2 Pd_j + g_b^2 R_j^-1) [+ zero block]
    // with R_j^-1 = 1 / (nu Lambda_s + (gamma^2/nu) lambda_j^2 Lambda_s^-1)   (fdsolve.cpp:114-136)
    const int npairs = static_cast<int>(F.time.lambda.size());
    const int nt = F.n_t;
    Vector S(lam_s.size());
    for (size_t s = 0; s < lam_s.size(); ++s) S[s] = gamma * F.time.sigma + nu * lam_s[s];
    for (int j = 0; j < npairs; ++j) {
        const double lam = F.time.lambda[j];
        const double c = gamma * gamma / nu * lam * lam;
        const double ga = F.time.g[2 * j], gb = F.time.g[2 * j + 1];
        const double c1 = gamma / nu * lam;
        for (size_t s = 0; s < lam_s.size(); ++s) {
            const double rinv = 1.0 / (nu * lam_s[s] + c * lam_inv[s]);
            const double Pd = lam_inv[s] / nu - (c1 * c1 / nu) * (lam_inv[s] * lam_inv[s] * rinv);
            S[s] += gamma * gamma * (ga * ga * Pd + gb * gb * rinv);
        }
    }
    if (F.time.zero_count) {
        const double gz = F.time.g[nt - 2];
        const double cz = gamma * gamma * gz * gz / nu;
        for (size_t s = 0; s < lam_s.size(); ++s) S[s] += cz * lam_inv[s];
    }
    F.S_inv.resize(S.size());
    for (size_t s = 0; s < S.size(); ++s) {
        if (std::fabs(S[s]) == 0.0)
            throw std::runtime_error("ExtendedFDPreconditioner: singular Schur complement");
        F.S_inv[s] = 1.0 / S[s];
    }

    if (scaling) {
        F.d_inv_sqrt.resize(static_cast<size_t>(F.n_dof));
        for (Index i = 0; i < F.n_dof; ++i)
            if (!(scaling[i] > 0.0))
                throw std::invalid_argument("ExtendedFDPreconditioner: scaling must be strictly positive");
        for (Index i = 0; i < F.n_dof; ++i) F.d_inv_sqrt[i] = 1.0 / std::sqrt(scaling[i]);
    }
    return F;
}

} // namespace stiga
