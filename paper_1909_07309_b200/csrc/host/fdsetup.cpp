// Host half of the extended-FD setup; follows /root/reference/proj/core/src/fdsolve.cpp:67-153.
#include "fdsetup.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
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

bool centrosymmetric(const DenseMatrix& A, double rtol) {
    const Index n = A.rows;
    if (A.cols != n || n < 2) return false;
    double amax = 0.0, dmax = 0.0;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            amax = std::max(amax, std::fabs(A(i, j)));
            dmax = std::max(dmax, std::fabs(A(i, j) - A(n - 1 - i, n - 1 - j)));
            dmax = std::max(dmax, std::fabs(A(i, j) - A(j, i)));
        }
    return amax > 0.0 && dmax <= rtol * amax;
}

namespace {

// Q^T A Q for Q = [(e_i + e_{n-1-i})/sqrt2 (i < h), e_h (n odd), (e_i - e_{n-1-i})/sqrt2 (i < h)],
// symmetrised over the four mirrored entries (A is centrosymmetric only to rounding).
void fold_blocks(const DenseMatrix& A, int h, int F, DenseMatrix& E, DenseMatrix& O) {
    const Index n = A.rows;
    const double r2 = std::sqrt(2.0);
    E = DenseMatrix(F, F);
    O = DenseMatrix(h, h);
    auto a = [&](Index i, Index j) { return 0.5 * (A(i, j) + A(j, i)); };
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < h; ++i) {
            const double s = a(i, j), c = a(i, n - 1 - j), r = a(n - 1 - i, j), t = a(n - 1 - i, n - 1 - j);
            E(i, j) = 0.5 * ((s + t) + (c + r));
            O(i, j) = 0.5 * ((s + t) - (c + r));
        }
    if (F > h) {
        for (int i = 0; i < h; ++i) E(i, h) = E(h, i) = (a(i, h) + a(n - 1 - i, h)) / r2;
        E(h, h) = A(h, h);
    }
}

// Split eigenbasis of a centrosymmetric SPD pencil: U (n x n) in folded column order [even; odd]
// with eigenvalues lam_fold; fb receives the half-size bases.
void split_eig(const DenseMatrix& K, const DenseMatrix& M, FoldBasis& fb, DenseMatrix& U, Vector& lam_fold) {
    const Index n = K.rows;
    fb.h = static_cast<int>(n / 2);
    fb.F = static_cast<int>(n) - fb.h;
    DenseMatrix Ke, Ko, Me, Mo;
    fold_blocks(K, fb.h, fb.F, Ke, Ko);
    fold_blocks(M, fb.h, fb.F, Me, Mo);
    Vector le, lo;
    spd_generalized_eig(Ke, Me, fb.We, le);
    if (fb.h > 0) spd_generalized_eig(Ko, Mo, fb.Wo, lo);
    const double r2 = std::sqrt(2.0);
    U = DenseMatrix(n, n);
    for (int c = 0; c < fb.F; ++c) {
        for (int i = 0; i < fb.h; ++i) U(i, c) = U(n - 1 - i, c) = fb.We(i, c) / r2;
        if (fb.F > fb.h) U(fb.h, c) = fb.We(fb.h, c);
    }
    for (int c = 0; c < fb.h; ++c)
        for (int i = 0; i < fb.h; ++i) {
            U(i, fb.F + c) = fb.Wo(i, c) / r2;
            U(n - 1 - i, fb.F + c) = -fb.Wo(i, c) / r2;
        }
    lam_fold = le;
    lam_fold.insert(lam_fold.end(), lo.begin(), lo.end());
}

// Rayleigh-quotient refinement of the spatial eigenvalues: lambda_k = u_k^T K u_k / u_k^T M u_k with
// long-double accumulation.  A backward-stable eigensolver returns lambda_k to an absolute error of
// ~eps * lambda_max, i.e. a relative error of eps * lambda_max / lambda_min for the smallest (smoothest)
// modes -- 1e-11 at n ~ 257 -- and those modes dominate the FD output.  The quotient of an
// eigenvector accurate to delta is accurate to ~delta^2 * lambda_max, so the refined eigenvalues are
// accurate to rounding and independent of the eigensolver.
void refine_eigenvalues(const DenseMatrix& K, const DenseMatrix& M, const DenseMatrix& U, Vector& lam) {
    const Index n = K.rows;
    std::vector<long double> ku(n), mu(n);
    for (Index k = 0; k < U.cols; ++k) {
        const double* u = U.col(k);
        for (Index i = 0; i < n; ++i) ku[i] = mu[i] = 0.0L;
        for (Index j = 0; j < n; ++j) {
            const long double uj = u[j];
            if (uj == 0.0L) continue;
            const double* kc = K.col(j);
            const double* mc = M.col(j);
            for (Index i = 0; i < n; ++i) {
                ku[i] += static_cast<long double>(kc[i]) * uj;
                mu[i] += static_cast<long double>(mc[i]) * uj;
            }
        }
        long double num = 0.0L, den = 0.0L;
        for (Index i = 0; i < n; ++i) {
            num += static_cast<long double>(u[i]) * ku[i];
            den += static_cast<long double>(u[i]) * mu[i];
        }
        if (den > 0.0L) lam[k] = static_cast<double>(num / den);
    }
}

}  // namespace

std::vector<double> fold_matrices(const FoldBasis& fb, bool forward, int Mp, int Kp) {
    const int h = fb.h, F = fb.F;
    if (Mp < F || Kp < F) throw std::runtime_error("internal: folded matrix padding too small");
    std::vector<double> out(2 * static_cast<size_t>(Mp) * Kp, 0.0);
    double* A1 = out.data();
    double* A2 = out.data() + static_cast<size_t>(Mp) * Kp;
    const double r2 = std::sqrt(2.0);
    for (int r = 0; r < F; ++r)
        for (int k = 0; k < F; ++k) {
            if (forward) {  // A_e[r][k] (U^T, even rows), A_o[r][k] (odd rows)
                A1[r * Kp + k] = k < h ? fb.We(k, r) / r2 : 0.5 * fb.We(k, r);
                if (r < h && k < h) A2[r * Kp + k] = fb.Wo(k, r) / r2;
            } else {        // A_p[i][c], A_q[i][c] (U: p = A_p y_e, q = A_q y_o)
                A1[r * Kp + k] = r < h ? fb.We(r, k) / r2 : fb.We(r, k);
                if (r < h && k < h) A2[r * Kp + k] = fb.Wo(r, k) / r2;
            }
        }
    return out;
}

Vector FDFactors::lambda_dev(int l) const {
    if (!fold[l].on) return lambda[l];
    Vector v(lambda[l].size());
    for (size_t f = 0; f < v.size(); ++f) v[f] = lambda[l][fold[l].dev_order[f]];
    return v;
}

DenseMatrix FDFactors::U_dev(int l) const {
    if (!fold[l].on) return U[l];
    const DenseMatrix& A = U[l];
    DenseMatrix B(A.rows, A.cols);
    for (Index f = 0; f < A.cols; ++f)
        for (Index i = 0; i < A.rows; ++i) B(i, f) = A(i, fold[l].dev_order[f]);
    return B;
}

Vector FDFactors::S_inv_dev() const {
    bool any = false;
    for (const auto& fb : fold) any = any || fb.on;
    if (!any) return S_inv;
    Vector out(S_inv.size());
    std::vector<Index> stride(d, 1);
    for (int l = 1; l < d; ++l) stride[l] = stride[l - 1] * n[l - 1];
    for (Index s = 0; s < static_cast<Index>(S_inv.size()); ++s) {
        Index rem = s, sa = 0;
        for (int l = 0; l < d; ++l) {
            const Index f = rem % n[l];
            rem /= n[l];
            sa += stride[l] * (fold[l].on ? fold[l].dev_order[f] : f);
        }
        out[s] = S_inv[sa];
    }
    return out;
}

FDFactors fd_setup(const std::vector<DenseMatrix>& space_K, const std::vector<DenseMatrix>& space_M,
                   const DenseMatrix& Wt, const DenseMatrix& Mt, double gamma, double nu,
                   const double* scaling, bool host_schur) {
    if (gamma <= 0.0) throw std::invalid_argument("ExtendedFDPreconditioner: gamma must be positive");
    if (nu <= 0.0) throw std::invalid_argument("ExtendedFDPreconditioner: nu must be positive");
    if (space_K.size() != space_M.size() || space_K.empty())
        throw std::invalid_argument("ExtendedFDPreconditioner: per-direction matrices mismatch");
    FDFactors F;
    F.d = static_cast<int>(space_K.size());
    Index n_s = 1;
    static const bool no_fold = std::getenv("STIGA_NO_FOLD") != nullptr;
    for (int l = 0; l < F.d; ++l) {
        DenseMatrix U;
        Vector lam;
        FoldBasis fb;
        // exact mirror symmetry only: splitting a pencil that is centrosymmetric merely to rounding
        // would perturb the preconditioner by ~1e-12 relative (measured), so such inputs keep the
        // dense eigenbasis
        if (!no_fold && space_K[l].rows >= 2 && centrosymmetric(space_K[l], 0.0) &&
            centrosymmetric(space_M[l], 0.0)) {
            DenseMatrix Uf;
            Vector lf;
            split_eig(space_K[l], space_M[l], fb, Uf, lf);
            // exported order: ascending eigenvalues, as spd_generalized_eig returns them
            const int nl = static_cast<int>(lf.size());
            std::vector<int> asc(nl);
            for (int i = 0; i < nl; ++i) asc[i] = i;
            std::stable_sort(asc.begin(), asc.end(), [&](int a, int b) { return lf[a] < lf[b]; });
            U = DenseMatrix(nl, nl);
            lam.resize(nl);
            fb.dev_order.assign(nl, 0);
            for (int k = 0; k < nl; ++k) {
                lam[k] = lf[asc[k]];
                for (int i = 0; i < nl; ++i) U(i, k) = Uf(i, asc[k]);
                fb.dev_order[asc[k]] = k;
            }
            fb.on = true;
        } else {
            spd_generalized_eig(space_K[l], space_M[l], U, lam);
        }
        refine_eigenvalues(space_K[l], space_M[l], U, lam);  // lambda_dev() reads these through dev_order
        F.n.push_back(static_cast<int>(lam.size()));
        F.U.push_back(std::move(U));
        F.lambda.push_back(std::move(lam));
        F.fold.push_back(std::move(fb));
        n_s *= F.n.back();
    }
    F.time = time_factorization(Wt, Mt);
    F.n_t = static_cast<int>(F.time.size());
    F.n_s_total = n_s;
    F.n_dof = n_s * F.n_t;
    F.gamma = gamma;
    F.nu = nu;

    if (!host_schur) {  // Lambda_s, S^-1 and their checks on the device (capi.cpp fd_build)
        if (scaling) {
            F.d_inv_sqrt.resize(static_cast<size_t>(F.n_dof));
            for (Index i = 0; i < F.n_dof; ++i)
                if (!(scaling[i] > 0.0))
                    throw std::invalid_argument("ExtendedFDPreconditioner: scaling must be strictly positive");
            for (Index i = 0; i < F.n_dof; ++i) F.d_inv_sqrt[i] = 1.0 / std::sqrt(scaling[i]);
        }
        return F;
    }
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
