// Eigen-free dense linear algebra for the host-side setup of the FD preconditioner.
// Replaces the Eigen calls of the reference (types.hpp:8-11, pencil.cpp:15-16,36,47,143,
// bspline.cpp:162): column-major dense matrices, Cholesky, triangular solves and a
// symmetric eigensolver (Householder tridiagonalisation + implicit-shift QL).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace stiga {

using Index = std::int64_t;
using Vector = std::vector<double>;

/// Column-major dense matrix (the reference's DenseMatrix = Eigen::MatrixXd).
struct DenseMatrix {
    Index rows = 0, cols = 0;
    std::vector<double> a;

    DenseMatrix() = default;
    DenseMatrix(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
    static DenseMatrix identity(Index n) {
        DenseMatrix m(n, n);
        for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + rows * j)]; }
    double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + rows * j)]; }
    double* col(Index j) { return a.data() + rows * j; }
    const double* col(Index j) const { return a.data() + rows * j; }
    DenseMatrix transpose() const;
    DenseMatrix block(Index r0, Index c0, Index nr, Index nc) const;
};

DenseMatrix matmul(const DenseMatrix& A, const DenseMatrix& B);          // A * B
DenseMatrix matmul_tn(const DenseMatrix& A, const DenseMatrix& B);       // A^T * B
Vector matvec(const DenseMatrix& A, const Vector& x);                    // A * x
Vector matvec_t(const DenseMatrix& A, const Vector& x);                  // A^T * x
double dot(const Vector& x, const Vector& y);
double norm2(const Vector& x);

/// Lower Cholesky factor L (A = L L^T).  Returns false if A is not SPD.
bool cholesky(const DenseMatrix& A, DenseMatrix& L);
/// Solve L X = B in place (L lower triangular).
void trsm_lower(const DenseMatrix& L, DenseMatrix& B);
/// Solve L^T X = B in place (L lower triangular).
void trsm_lower_t(const DenseMatrix& L, DenseMatrix& B);

/// Symmetric eigendecomposition A = Q diag(w) Q^T, eigenvalues ascending.
/// Throws std::runtime_error if the QL iteration does not converge.
void sym_eig(const DenseMatrix& A, Vector& w, DenseMatrix& Q);

/// Alternative symmetric eigensolver for sym_eig on the calling thread (nullptr: the host
/// Householder + QL).  Used by the setup's cuSOLVER backend (host/eig_device.cpp) through
/// ScopedSymEig; same contract: ascending w, orthonormal columns of Q.
using SymEigFn = void (*)(const DenseMatrix& A, Vector& w, DenseMatrix& Q);
SymEigFn set_sym_eig_backend(SymEigFn fn);
struct ScopedSymEig {
    SymEigFn prev;
    explicit ScopedSymEig(SymEigFn fn) : prev(set_sym_eig_backend(fn)) {}
    ~ScopedSymEig() { set_sym_eig_backend(prev); }
};

} // namespace stiga
