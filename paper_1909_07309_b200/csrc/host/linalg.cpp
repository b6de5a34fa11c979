// Host dense linear algebra used by the FD setup (see linalg.hpp).
#include "linalg.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <numeric>

namespace stiga {

DenseMatrix DenseMatrix::transpose() const {
    DenseMatrix t(cols, rows);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) t(j, i) = (*this)(i, j);
    return t;
}

DenseMatrix DenseMatrix::block(Index r0, Index c0, Index nr, Index nc) const {
    DenseMatrix b(nr, nc);
    for (Index j = 0; j < nc; ++j)
        for (Index i = 0; i < nr; ++i) b(i, j) = (*this)(r0 + i, c0 + j);
    return b;
}

DenseMatrix matmul(const DenseMatrix& A, const DenseMatrix& B) {
    if (A.cols != B.rows) throw std::invalid_argument("matmul: shape mismatch");
    DenseMatrix C(A.rows, B.cols);
    for (Index j = 0; j < B.cols; ++j)
        for (Index k = 0; k < A.cols; ++k) {
            const double b = B(k, j);
            if (b == 0.0) continue;
            const double* a = A.col(k);
            double* c = C.col(j);
            for (Index i = 0; i < A.rows; ++i) c[i] += a[i] * b;
        }
    return C;
}

DenseMatrix matmul_tn(const DenseMatrix& A, const DenseMatrix& B) {
    if (A.rows != B.rows) throw std::invalid_argument("matmul_tn: shape mismatch");
    DenseMatrix C(A.cols, B.cols);
    for (Index j = 0; j < B.cols; ++j)
        for (Index i = 0; i < A.cols; ++i) {
            const double* a = A.col(i);
            const double* b = B.col(j);
            double s = 0.0;
            for (Index k = 0; k < A.rows; ++k) s += a[k] * b[k];
            C(i, j) = s;
        }
    return C;
}

Vector matvec(const DenseMatrix& A, const Vector& x) {
    Vector y(static_cast<size_t>(A.rows), 0.0);
    for (Index k = 0; k < A.cols; ++k) {
        const double* a = A.col(k);
        for (Index i = 0; i < A.rows; ++i) y[i] += a[i] * x[k];
    }
    return y;
}

Vector matvec_t(const DenseMatrix& A, const Vector& x) {
    Vector y(static_cast<size_t>(A.cols), 0.0);
    for (Index j = 0; j < A.cols; ++j) {
        const double* a = A.col(j);
        double s = 0.0;
        for (Index i = 0; i < A.rows; ++i) s += a[i] * x[i];
        y[j] = s;
    }
    return y;
}

double dot(const Vector& x, const Vector& y) {
    double s = 0.0;
    for (size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
    return s;
}

double norm2(const Vector& x) { return std::sqrt(dot(x, x)); }

bool cholesky(const DenseMatrix& A, DenseMatrix& L) {
    const Index n = A.rows;
    L = DenseMatrix(n, n);
    for (Index j = 0; j < n; ++j) {
        double s = A(j, j);
        for (Index k = 0; k < j; ++k) s -= L(j, k) * L(j, k);
        if (!(s > 0.0)) return false;
        const double ljj = std::sqrt(s);
        L(j, j) = ljj;
        for (Index i = j + 1; i < n; ++i) {
            double t = A(i, j);
            for (Index k = 0; k < j; ++k) t -= L(i, k) * L(j, k);
            L(i, j) = t / ljj;
        }
    }
    return true;
}

void trsm_lower(const DenseMatrix& L, DenseMatrix& B) {
    const Index n = L.rows;
    for (Index c = 0; c < B.cols; ++c) {
        double* b = B.col(c);
        for (Index i = 0; i < n; ++i) {
            double s = b[i];
            for (Index k = 0; k < i; ++k) s -= L(i, k) * b[k];
            b[i] = s / L(i, i);
        }
    }
}

void trsm_lower_t(const DenseMatrix& L, DenseMatrix& B) {
    const Index n = L.rows;
    for (Index c = 0; c < B.cols; ++c) {
        double* b = B.col(c);
        for (Index i = n - 1; i >= 0; --i) {
            double s = b[i];
            for (Index k = i + 1; k < n; ++k) s -= L(k, i) * b[k];
            b[i] = s / L(i, i);
        }
    }
}

// Householder reduction of the symmetric matrix T (in place) to tridiagonal form,
// Q accumulating the reflectors so that A = Q T Q^T.
static void tridiagonalize(DenseMatrix& T, DenseMatrix& Q, Vector& diag, Vector& off) {
    const Index n = T.rows;
    Q = DenseMatrix::identity(n);
    Vector v(n), p(n), w(n);
    for (Index k = 0; k + 2 < n; ++k) {
        const Index m = n - k - 1;  // length of the column below the diagonal
        double alpha = 0.0;
        for (Index i = 0; i < m; ++i) alpha += T(k + 1 + i, k) * T(k + 1 + i, k);
        alpha = std::sqrt(alpha);
        if (alpha == 0.0) continue;
        const double x0 = T(k + 1, k);
        const double beta = (x0 >= 0.0) ? -alpha : alpha;  // target value
        // v = x - beta e1, tau = 2 / (v^T v)
        for (Index i = 0; i < m; ++i) v[i] = T(k + 1 + i, k);
        v[0] -= beta;
        double vtv = 0.0;
        for (Index i = 0; i < m; ++i) vtv += v[i] * v[i];
        if (vtv == 0.0) continue;
        const double tau = 2.0 / vtv;
        // p = tau * T22 v
        for (Index i = 0; i < m; ++i) {
            double s = 0.0;
            for (Index j = 0; j < m; ++j) s += T(k + 1 + i, k + 1 + j) * v[j];
            p[i] = tau * s;
        }
        double pv = 0.0;
        for (Index i = 0; i < m; ++i) pv += p[i] * v[i];
        const double half = 0.5 * tau * pv;
        for (Index i = 0; i < m; ++i) w[i] = p[i] - half * v[i];
        for (Index j = 0; j < m; ++j)
            for (Index i = 0; i < m; ++i)
                T(k + 1 + i, k + 1 + j) -= v[i] * w[j] + w[i] * v[j];
        T(k + 1, k) = beta;
        T(k, k + 1) = beta;
        for (Index i = 1; i < m; ++i) {
            T(k + 1 + i, k) = 0.0;
            T(k, k + 1 + i) = 0.0;
        }
        // Q <- Q H with H = I - tau v v^T acting on rows/cols k+1..n-1
        for (Index r = 0; r < n; ++r) {
            double s = 0.0;
            for (Index i = 0; i < m; ++i) s += Q(r, k + 1 + i) * v[i];
            s *= tau;
            for (Index i = 0; i < m; ++i) Q(r, k + 1 + i) -= s * v[i];
        }
    }
    diag.assign(n, 0.0);
    off.assign(n, 0.0);
    for (Index i = 0; i < n; ++i) diag[i] = T(i, i);
    for (Index i = 0; i + 1 < n; ++i) off[i] = T(i + 1, i);
}

// Implicit-shift QL on the symmetric tridiagonal (d, e) with e[i] = T(i+1,i),
// rotating the columns of Z.
static void tridiagonal_ql(Vector& d, Vector& e, DenseMatrix& Z) {
    const Index n = static_cast<Index>(d.size());
    if (n == 0) return;
    e[n - 1] = 0.0;
    for (Index l = 0; l < n; ++l) {
        int iter = 0;
        while (true) {
            Index m = l;
            for (; m < n - 1; ++m) {
                const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= DBL_EPSILON * dd) break;
            }
            if (m == l) break;
            if (++iter > 100) throw std::runtime_error("sym_eig: QL iteration did not converge");
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
            double s = 1.0, c = 1.0, p = 0.0;
            bool deflated = false;
            for (Index i = m - 1; i >= l; --i) {
                const double f = s * e[i];
                const double b = c * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {
                    d[i + 1] -= p;
                    e[m] = 0.0;
                    deflated = true;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - p;
                r = (d[i] - g) * s + 2.0 * c * b;
                p = s * r;
                d[i + 1] = g + p;
                g = c * r - b;
                double* zi = Z.col(i);
                double* zi1 = Z.col(i + 1);
                for (Index k = 0; k < n; ++k) {
                    const double t = zi1[k];
                    zi1[k] = s * zi[k] + c * t;
                    zi[k] = c * zi[k] - s * t;
                }
            }
            if (deflated) continue;
            d[l] -= p;
            e[l] = g;
            e[m] = 0.0;
        }
    }
}

namespace {
thread_local SymEigFn g_sym_eig_backend = nullptr;
}

SymEigFn set_sym_eig_backend(SymEigFn fn) {
    const SymEigFn prev = g_sym_eig_backend;
    g_sym_eig_backend = fn;
    return prev;
}

void sym_eig(const DenseMatrix& A, Vector& w, DenseMatrix& Q) {
    const Index n = A.rows;
    if (A.cols != n) throw std::invalid_argument("sym_eig: matrix not square");
    if (g_sym_eig_backend) {
        g_sym_eig_backend(A, w, Q);
        return;
    }
    DenseMatrix T = A;
    // symmetrize defensively (the callers pass symmetric matrices)
    for (Index j = 0; j < n; ++j)
        for (Index i = j + 1; i < n; ++i) {
            const double s = 0.5 * (T(i, j) + T(j, i));
            T(i, j) = s;
            T(j, i) = s;
        }
    DenseMatrix Z;
    Vector d, e;
    tridiagonalize(T, Z, d, e);
    tridiagonal_ql(d, e, Z);
    std::vector<Index> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](Index a, Index b) { return d[a] < d[b]; });
    w.resize(n);
    Q = DenseMatrix(n, n);
    for (Index j = 0; j < n; ++j) {
        w[j] = d[order[j]];
        const double* src = Z.col(order[j]);
        std::copy(src, src + n, Q.col(j));
    }
}

} // namespace stiga
