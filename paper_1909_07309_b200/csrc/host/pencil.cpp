// Host-side pencil factorizations; follows /root/reference/proj/core/src/pencil.cpp:12-165.
// Eigen's GeneralizedSelfAdjointEigenSolver / SelfAdjointEigenSolver / LLT / SimplicialLLT are
// replaced by the Cholesky + Householder/QL routines of linalg.cpp.  The eigenvector bases may
// differ from Eigen's by signs/rotations inside clusters; the FD apply is invariant to that.
#include "pencil.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace stiga {

void spd_generalized_eig(const DenseMatrix& K, const DenseMatrix& M, DenseMatrix& U, Vector& lambda) {
    if (K.rows != K.cols || M.rows != M.cols || K.rows != M.rows)
        throw std::invalid_argument("spd_generalized_eig: shape mismatch");
    DenseMatrix L;
    if (!cholesky(M, L)) throw std::runtime_error("spd_generalized_eig: mass matrix not SPD");
    // C = L^-1 K L^-T
    DenseMatrix C = K;
    trsm_lower(L, C);
    C = C.transpose();
    trsm_lower(L, C);
    DenseMatrix Q;
    sym_eig(C, lambda, Q);
    trsm_lower_t(L, Q);  // U = L^-T Q  ->  U^T M U = I
    U = std::move(Q);
}

namespace {

// Pairs (v, q) with S q = lam v, S v = -lam q from the real symmetric embedding
// E = [[0, -S], [S, 0]] of the Hermitian iS (E [x; y] = lam [x; y] <=> S x = lam y, -S y = lam x;
// q = sqrt(2) x, v = sqrt(2) y).  Every positive eigenvalue of E is double (z and Jz, J [x; y] = [-y; x]).
// Pairs are built by pivoted Gram-Schmidt over each cluster's J-invariant eigenspace, and every new z
// and Jz is orthogonalised against ALL accepted vectors (two passes): distinct pairs closer than the
// eigensolver can separate (p = 4, n_el = 64: gaps ~1e-8 relative) then stay exactly orthonormal, and
// their residual mixing perturbs U^T W U only by gap x mixing ~ eps.  DESIGN.md §3.3.
void embedding_pairs(const DenseMatrix& S, double zero_tol_mu, std::vector<double>& lam_out, std::vector<Vector>& cols) {
    const Index n = S.rows;
    DenseMatrix E(2 * n, 2 * n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            E(i, n + j) = -S(i, j);
            E(n + i, j) = S(i, j);
        }
    Vector w;
    DenseMatrix V;
    sym_eig(E, w, V);
    const double lam_tol = std::sqrt(zero_tol_mu);
    const double lam_max = std::max(w[2 * n - 1], 1.0);
    std::vector<std::vector<Index>> clusters;
    for (Index k = 0; k < 2 * n; ++k) {
        if (!(w[k] > lam_tol)) continue;
        if (clusters.empty() || w[k] - w[clusters.back().back()] > 1e-8 * lam_max) clusters.emplace_back();
        clusters.back().push_back(k);
    }
    struct Pair { double lam; Vector v, q; };
    std::vector<Pair> pairs;
    std::vector<Vector> basis;  // every accepted z and Jz, across clusters
    const double r2 = std::sqrt(2.0);
    auto project = [&](Vector& r) {
        for (int pass = 0; pass < 2; ++pass)
            for (const Vector& b : basis) {
                const double c = dot(b, r);
                for (Index i = 0; i < 2 * n; ++i) r[i] -= c * b[i];
            }
    };
    auto normalize = [](Vector& r) {
        const double nr = norm2(r);
        for (double& x : r) x /= nr;
    };
    for (const auto& cl : clusters) {
        for (size_t m = 0; m < cl.size() / 2; ++m) {
            Vector best;
            double bnorm = -1.0;
            for (Index k : cl) {
                Vector r(V.col(k), V.col(k) + 2 * n);
                project(r);
                const double nr = norm2(r);
                if (nr > bnorm) {
                    bnorm = nr;
                    best = r;
                }
            }
            for (double& x : best) x /= bnorm;
            project(best);
            normalize(best);
            basis.push_back(best);
            Vector jz(2 * n);
            for (Index i = 0; i < n; ++i) {
                jz[i] = -best[n + i];
                jz[n + i] = best[i];
            }
            project(jz);
            normalize(jz);
            basis.push_back(jz);
            const Vector Ez = matvec(E, best);
            Pair P;
            P.lam = dot(best, Ez);
            P.q.resize(n);
            P.v.resize(n);
            for (Index i = 0; i < n; ++i) {
                P.q[i] = r2 * best[i];
                P.v[i] = r2 * best[n + i];
            }
            pairs.push_back(std::move(P));
        }
    }
    std::stable_sort(pairs.begin(), pairs.end(), [](const Pair& a, const Pair& b) { return a.lam < b.lam; });
    lam_out.clear();
    cols.clear();
    for (auto& P : pairs) {
        lam_out.push_back(P.lam);
        cols.push_back(std::move(P.v));
        cols.push_back(std::move(P.q));
    }
}

}  // namespace

SkewPencilEig skew_pencil_eig(const DenseMatrix& W, const DenseMatrix& M) {
    const Index n = W.rows;
    if (W.cols != n || M.rows != n || M.cols != n) throw std::invalid_argument("skew_pencil_eig: shape mismatch");
    SkewPencilEig out;
    if (n == 0) return out;
    double wmax = 0.0, asym = 0.0;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            wmax = std::max(wmax, std::fabs(W(i, j)));
            asym = std::max(asym, std::fabs(W(i, j) + W(j, i)));
        }
    if (asym > 1e-13 * std::max(wmax, 1.0))
        throw std::runtime_error("skew_pencil_eig: matrix is not skew-symmetric (assembly bug)");
    DenseMatrix L;
    if (!cholesky(M, L)) throw std::runtime_error("skew_pencil_eig: mass matrix not SPD");
    // S = L^-1 W L^-T, skew-symmetrized (pencil.cpp:41-44)
    DenseMatrix S = W;
    trsm_lower(L, S);
    S = S.transpose();
    trsm_lower(L, S);
    S = S.transpose();
    for (Index j = 0; j < n; ++j)
        for (Index i = j; i < n; ++i) {
            const double a = 0.5 * (S(i, j) - S(j, i));
            S(i, j) = a;
            S(j, i) = -a;
        }
    const DenseMatrix C = matmul_tn(S, S);
    Vector mu;
    DenseMatrix Q;
    sym_eig(C, mu, Q);
    for (double& m : mu) m = std::max(m, 0.0);
    const double mu_max = std::max(mu[n - 1], 1.0);
    const double zero_tol = 1e-12 * mu_max;

    // Pairs from the Hermitian embedding (deliberate deviation): the reference's walk
    // over the eigenvectors of S^T S (pencil.cpp:54-87) squares the conditioning (U^T M U - I = 1e-8 at
    // p = 4, n_el = 64) and fails outright on config 2; S^T S only seeds the zero columns here.
    std::vector<Vector> zero_cols, pair_cols;
    embedding_pairs(S, zero_tol, out.lambda, pair_cols);
    const Index nz = n - static_cast<Index>(pair_cols.size());
    Index n_small = 0;
    for (Index k = 0; k < n; ++k) n_small += mu[k] <= zero_tol ? 1 : 0;
    if (nz < 0 || nz > n_small + 1) throw std::runtime_error("skew_pencil_eig: eigenvalue pairing failed");
    for (Index k = 0; k < nz; ++k) {  // null vectors of S, orthogonal to every pair column (two passes)
        Vector q(Q.col(k), Q.col(k) + n);
        for (int pass = 0; pass < 2; ++pass) {
            for (const auto& c : pair_cols) {
                const double cq = dot(c, q);
                for (Index i = 0; i < n; ++i) q[i] -= cq * c[i];
            }
            for (const auto& c : zero_cols) {
                const double cq = dot(c, q);
                for (Index i = 0; i < n; ++i) q[i] -= cq * c[i];
            }
        }
        const double nq = norm2(q);
        for (double& x : q) x /= nq;
        zero_cols.push_back(std::move(q));
    }
    out.zero_count = static_cast<int>(nz);
    DenseMatrix Ublk(n, n);
    Index c = 0;
    for (const auto& col : pair_cols) std::copy(col.begin(), col.end(), Ublk.col(c++));
    for (const auto& col : zero_cols) std::copy(col.begin(), col.end(), Ublk.col(c++));
    trsm_lower_t(L, Ublk);  // U = L^-T Ublk (pencil.cpp:93)
    out.U = std::move(Ublk);
    return out;
}

TimeFactorization time_factorization(const DenseMatrix& W, const DenseMatrix& M) {
    const Index n = W.rows;
    if (M.rows != n || n < 1) throw std::invalid_argument("time_factorization: shape mismatch");
    TimeFactorization out;
    out.U = DenseMatrix(n, n);
    out.g.assign(n - 1, 0.0);
    out.r.assign(n - 1, 0.0);
    if (n == 1) {  // pencil.cpp:124-130
        out.rho = 1.0 / std::sqrt(M(0, 0));
        out.U(0, 0) = out.rho;
        out.sigma = out.rho * W(0, 0) * out.rho;
        return out;
    }
    const DenseMatrix W0 = W.block(0, 0, n - 1, n - 1);
    const DenseMatrix M0 = M.block(0, 0, n - 1, n - 1);
    Vector w(n - 1), m(n - 1);
    for (Index i = 0; i < n - 1; ++i) {
        w[i] = W(i, n - 1);
        m[i] = M(i, n - 1);
    }
    SkewPencilEig skew = skew_pencil_eig(W0, M0);
    out.lambda = skew.lambda;
    out.zero_count = skew.zero_count;

    // M0 v = -m by Cholesky (pencil.cpp:141-146)
    DenseMatrix L;
    if (!cholesky(M0, L)) throw std::runtime_error("time_factorization: leading time mass block not SPD");
    DenseMatrix v(n - 1, 1);
    for (Index i = 0; i < n - 1; ++i) v(i, 0) = -m[i];
    trsm_lower(L, v);
    trsm_lower_t(L, v);

    Vector q(n);
    for (Index i = 0; i < n - 1; ++i) q[i] = v(i, 0);
    q[n - 1] = 1.0;
    const double s = std::sqrt(dot(q, matvec(M, q)));
    for (Index i = 0; i < n - 1; ++i) out.r[i] = v(i, 0) / s;
    out.rho = 1.0 / s;

    for (Index j = 0; j < n - 1; ++j)
        for (Index i = 0; i < n - 1; ++i) out.U(i, j) = skew.U(i, j);
    for (Index i = 0; i < n - 1; ++i) out.U(i, n - 1) = out.r[i];
    out.U(n - 1, n - 1) = out.rho;

    Vector t = matvec(W0, out.r);
    for (Index i = 0; i < n - 1; ++i) t[i] += w[i] * out.rho;
    out.g = matvec_t(skew.U, t);  // g = U_blk^T (W0 r + w rho)
    Vector rr(out.r);
    rr.push_back(out.rho);
    out.sigma = dot(rr, matvec(W, rr));
    return out;
}

} // namespace stiga
